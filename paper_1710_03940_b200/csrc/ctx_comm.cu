// Collectives of the multi-rank solve: NCCL (loaded with dlopen) or the
// in-process fabric used to test several ranks on one device.
#include "ctx_impl.cuh"

Nccl g_nccl;

// ---------------------------------------------------------------------------
// communication (no-ops on a single rank)

static int nccl_check(dfl_ctx *ctx, int rc, const char *what) {
    if (rc != 0) {
        ctx->err = std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(rc) : "nccl error");
        return DFL_E_COMM;
    }
    return DFL_OK;
}

// allgather of `count` doubles per rank into recv[q * count] (send may alias
// recv + rank * count)
int comm_allgather(dfl_ctx *ctx, const double *send, double *recv, size_t count) {
    if (ctx->comm) return nccl_check(ctx, g_nccl.AllGather(send, recv, count, ncclDouble_, ctx->comm, ctx->st), "ncclAllGather");
    dfl_fabric *f = ctx->fab;
    CK(cudaStreamSynchronize(ctx->st));
    f->pub[ctx->rank] = send;
    f->barrier();
    for (int q = 0; q < ctx->nranks; ++q) {
        double *dst = recv + (size_t)q * count;
        if (f->pub[q] != dst) CK(cudaMemcpyAsync(dst, f->pub[q], count * sizeof(double), cudaMemcpyDefault, ctx->st));
    }
    CK(cudaStreamSynchronize(ctx->st));
    f->barrier();
    return DFL_OK;
}

// fill the ghost part v[n .. n+n_ghost) from the neighbours (runtime.py:246-271)
// pack on ctx->st; the NCCL transfers run on `xs` (ctx->st, or the comm
// stream when the operator overlaps them with its interior rows)
int halo(dfl_ctx *ctx, double *v, cudaStream_t xs) {
    if (!multi(ctx) || (ctx->nbr.empty() && !ctx->fab)) return DFL_OK;
    if (!xs) xs = ctx->st;
    if (ctx->nsend > 0) {
        launch_k(ctx->st, k_gather, (unsigned)cdiv(ctx->nsend, kBlock), kBlock, 0, v, ctx->send_idx, ctx->nsend,
                                                                              ctx->sendbuf);
        ctx->launches++;
    }
    if (xs != ctx->st && !ctx->fab) {
        CK(cudaEventRecord(ctx->ev_packed, ctx->st));
        CK(cudaStreamWaitEvent(xs, ctx->ev_packed, 0));
    }
    if (ctx->fab) {  // every rank takes part in the barriers, neighbours or not
        dfl_fabric *f = ctx->fab;
        CK(cudaStreamSynchronize(ctx->st));
        f->pub[ctx->rank] = ctx->sendbuf;
        f->barrier();
        int64_t ro = 0;
        for (size_t qi = 0; qi < ctx->nbr.size(); ++qi) {
            const dfl_ctx *peer = f->ctxs[ctx->nbr[qi]];
            int64_t off = 0, cnt = -1;
            for (size_t j = 0; j < peer->nbr.size(); ++j) {
                if (peer->nbr[j] == ctx->rank) {
                    cnt = peer->send_cnt[j];
                    break;
                }
                off += peer->send_cnt[j];
            }
            if (cnt != ctx->recv_cnt[qi]) {
                ctx->err = "halo plan mismatch between ranks";
                f->barrier();
                return DFL_E_COMM;
            }
            if (cnt > 0)
                CK(cudaMemcpyAsync(v + ctx->n + ro, f->pub[ctx->nbr[qi]] + off, cnt * sizeof(double), cudaMemcpyDefault,
                                   ctx->st));
            ro += ctx->recv_cnt[qi];
        }
        CK(cudaStreamSynchronize(ctx->st));
        f->barrier();
        return DFL_OK;
    }
    RC(nccl_check(ctx, g_nccl.GroupStart(), "ncclGroupStart"));
    int64_t so = 0, ro = 0;
    for (size_t q = 0; q < ctx->nbr.size(); ++q) {
        if (ctx->send_cnt[q] > 0)
            RC(nccl_check(ctx, g_nccl.Send(ctx->sendbuf + so, ctx->send_cnt[q], ncclDouble_, ctx->nbr[q], ctx->comm, xs),
                          "ncclSend"));
        if (ctx->recv_cnt[q] > 0)
            RC(nccl_check(ctx, g_nccl.Recv(v + ctx->n + ro, ctx->recv_cnt[q], ncclDouble_, ctx->nbr[q], ctx->comm, xs),
                          "ncclRecv"));
        so += ctx->send_cnt[q];
        ro += ctx->recv_cnt[q];
    }
    RC(nccl_check(ctx, g_nccl.GroupEnd(), "ncclGroupEnd"));
    return DFL_OK;
}

// Z' v partials -> t (global numbering) -> t2 = E^-1 t on every rank
int zt_to_t2(dfl_ctx *ctx, const KState *st, int need_refresh, bool from_op) {
    const int64_t *sub_tiles = ctx->sub_tiles;
    if (!multi(ctx)) {
        launch_k(ctx->st, k_zt_finish, ctx->nsub * ctx->k, 1024, 0, ctx->zt_part, sub_tiles, ctx->nsub, ctx->k,
                                                             ctx->tvec, 0, ctx->inexact ? nullptr : ctx->Einv,
                                                             ctx->K, ctx->t2, st, need_refresh, ctx->ticket,
                                                             from_op && ctx->split ? ctx->sub_btiles : nullptr,
                                                             ctx->ntiles);
        ctx->launches++;
        if (ctx->inexact) {
            launch_k(ctx->st, k_egmres, 1, 256, 0, ctx->Edense, (int)ctx->K, ctx->tvec, ctx->t2, ctx->coarse_tol,
                                             ctx->egm_scr, st, need_refresh);
            ctx->launches++;
        }
        return DFL_OK;
    }
    // local entries into a padded slot, allgather, unpack, solve
    const int64_t slot = (int64_t)ctx->max_nsub * ctx->k;
    double *mine = ctx->tgather + (int64_t)ctx->rank * slot;
    launch_k(ctx->st, k_zt_finish, ctx->nsub * ctx->k, 1024, 0, ctx->zt_part, sub_tiles, ctx->nsub, ctx->k, mine, 0,
                                                         nullptr, ctx->K, nullptr, st, need_refresh, ctx->ticket,
                                                         from_op && ctx->split ? ctx->sub_btiles : nullptr,
                                                         ctx->ntiles);
    RC(comm_allgather(ctx, mine, ctx->tgather, slot));
    // unpack rank slots into t: rank q owns a contiguous subdomain range
    int64_t pos = 0;
    for (int q = 0; q < ctx->nranks; ++q) {
        const int64_t cnt = (int64_t)ctx->rank_nsub[q] * ctx->k;
        if (cnt > 0) CK(cudaMemcpyAsync(ctx->tvec + pos, ctx->tgather + q * slot, cnt * sizeof(double),
                                        cudaMemcpyDeviceToDevice, ctx->st));
        pos += cnt;
    }
    if (ctx->inexact)
        launch_k(ctx->st, k_egmres, 1, 256, 0, ctx->Edense, (int)ctx->K, ctx->tvec, ctx->t2, ctx->coarse_tol, ctx->egm_scr,
                                         st, need_refresh);
    else
        launch_k(ctx->st, k_esolve, 1, 256, 0, ctx->Einv, ctx->K, ctx->tvec, ctx->t2, st, need_refresh);
    ctx->launches += 2;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// reductions across ranks: returns the pointer the scalar kernel reads
int rank_scalar(dfl_ctx *ctx, const double *part, int64_t nparts, int slot, const double **gath) {
    *gath = nullptr;
    if (!multi(ctx)) return DFL_OK;
    launch_k(ctx->st, k_reduce, 1, 1024, 0, part, nparts, ctx->scal + slot);
    ctx->launches++;
    RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
    *gath = ctx->sgather;
    return DFL_OK;
}

extern "C" {

int dfl_nccl_unique_id(void *id) {
    std::string err;
    if (!g_nccl.load(err)) {
        dfl::set_setup_error(err);
        return DFL_E_COMM;
    }
    int rc = g_nccl.GetUniqueId(static_cast<NcclId *>(id));
    if (rc != 0) {
        dfl::set_setup_error(std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(rc));
        return DFL_E_COMM;
    }
    return DFL_OK;
}

int dfl_ctx_set_comm(dfl_ctx *ctx, int nranks, int rank, const void *id) {
    if (!ctx) return DFL_E_STATE;
    if (nranks < 1 || rank < 0 || rank >= nranks) {
        ctx->err = "bad rank / world size";
        return DFL_E_PARTITION;
    }
    ctx->nranks = nranks;
    ctx->rank = rank;
    // a 1-rank NCCL communicator exercises the multi-rank code path on one GPU
    const char *fc = getenv("DFL_FORCE_COMM");
    if (nranks == 1 && !(fc && fc[0] == '1')) return DFL_OK;
    if (!g_nccl.load(ctx->err)) return DFL_E_COMM;
    CK(cudaSetDevice(ctx->device));
    NcclId nid;
    std::memcpy(&nid, id, sizeof nid);
    return nccl_check(ctx, g_nccl.CommInitRank(&ctx->comm, nranks, nid, rank), "ncclCommInitRank");
}

int dfl_fabric_create(int nranks, dfl_fabric **out) {
    if (!out || nranks < 1) return DFL_E_STATE;
    auto *f = new dfl_fabric;
    f->nranks = nranks;
    f->ctxs.assign(nranks, nullptr);
    f->pub.assign(nranks, nullptr);
    *out = f;
    return DFL_OK;
}

void dfl_fabric_destroy(dfl_fabric *f) { delete f; }

int dfl_ctx_set_fabric(dfl_ctx *ctx, dfl_fabric *f, int rank) {
    if (!ctx || !f || rank < 0 || rank >= f->nranks) return DFL_E_STATE;
    ctx->fab = f;
    ctx->nranks = f->nranks;
    ctx->rank = rank;
    f->ctxs[rank] = ctx;
    return DFL_OK;
}

}  // extern "C"
