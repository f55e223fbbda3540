// Collectives of the multi-rank solve: NCCL (loaded with dlopen) or the
// in-process fabric used to test several ranks on one device.
#include <functional>
#include <thread>

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

static int dropped(dfl_ctx *ctx) {
    ctx->err = "a participant dropped out: the collective did not complete within " +
               std::to_string(ctx->fab ? ctx->fab->timeout_s : ctx->comm_timeout_s) + " s";
    return DFL_E_COMM;
}

static double comm_timeout_default() {
    const char *t = getenv("DFL_COMM_TIMEOUT");
    return t ? atof(t) : 300.0;
}

static int comm_poll(dfl_ctx *ctx, const std::function<cudaError_t()> &query) {
    if (ctx->comm_dead) {
        ctx->err = "the communicator was aborted after an earlier failure";
        return DFL_E_COMM;
    }
    if (!ctx->comm) {
        for (;;) {  // no NCCL: plain wait
            const cudaError_t q = query();
            if (q == cudaSuccess) return DFL_OK;
            if (q != cudaErrorNotReady) CK(q);
            std::this_thread::yield();
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (long spin = 0;; ++spin) {
        const cudaError_t q = query();
        if (q == cudaSuccess) return DFL_OK;
        if (q != cudaErrorNotReady) CK(q);
        if ((spin & 255) == 0) {
            int aerr = 0;
            if (g_nccl.CommGetAsyncError && g_nccl.CommGetAsyncError(ctx->comm, &aerr) == 0 && aerr != 0 &&
                aerr != 7 /* ncclInProgress */) {
                ctx->err = std::string("NCCL asynchronous error: ") + g_nccl.GetErrorString(aerr) +
                           " (a participant dropped out?)";
                if (g_nccl.CommAbort) g_nccl.CommAbort(ctx->comm);
                ctx->comm = nullptr;
                ctx->comm_dead = true;
                return DFL_E_COMM;
            }
            const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (el > ctx->comm_timeout_s) {
                if (g_nccl.CommAbort) g_nccl.CommAbort(ctx->comm);
                ctx->comm = nullptr;
                ctx->comm_dead = true;
                return dropped(ctx);
            }
            if (spin > 4096) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
}

int comm_wait(dfl_ctx *ctx, cudaStream_t s) {
    if (!ctx->comm && !ctx->comm_dead) {
        CK(cudaStreamSynchronize(s));
        return DFL_OK;
    }
    return comm_poll(ctx, [s] { return cudaStreamQuery(s); });
}

int comm_wait_event(dfl_ctx *ctx, cudaEvent_t e) {
    if (!ctx->comm && !ctx->comm_dead) {
        CK(cudaEventSynchronize(e));
        return DFL_OK;
    }
    return comm_poll(ctx, [e] { return cudaEventQuery(e); });
}

// allgather of `count` doubles per rank into recv[q * count] (send may alias
// recv + rank * count)
int comm_allgather(dfl_ctx *ctx, const double *send, double *recv, size_t count) {
    if (ctx->comm_dead) return comm_wait(ctx, ctx->st);
    if (ctx->comm) return nccl_check(ctx, g_nccl.AllGather(send, recv, count, ncclDouble_, ctx->comm, ctx->st), "ncclAllGather");
    dfl_fabric *f = ctx->fab;
    CK(cudaStreamSynchronize(ctx->st));
    f->pub[ctx->rank] = send;
    if (!f->barrier()) return dropped(ctx);
    for (int q = 0; q < ctx->nranks; ++q) {
        double *dst = recv + (size_t)q * count;
        if (f->pub[q] != dst) CK(cudaMemcpyAsync(dst, f->pub[q], count * sizeof(double), cudaMemcpyDefault, ctx->st));
    }
    CK(cudaStreamSynchronize(ctx->st));
    if (!f->barrier()) return dropped(ctx);
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
        if (!f->barrier()) return dropped(ctx);
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
        if (!f->barrier()) return dropped(ctx);
        return DFL_OK;
    }
    if (ctx->comm_dead) return comm_wait(ctx, ctx->st);
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
int zt_to_t2(dfl_ctx *ctx, const KState *st, int need_refresh, bool from_op, const double *extra_part,
             int64_t extra_n, KState *fold) {
    const int64_t *sub_tiles = ctx->sub_tiles;
    if (!multi(ctx)) {
        launch_k(ctx->st, k_zt_finish, dim3(ctx->zt_chunks, ctx->nsub), 256, 0, ctx->zt_part, sub_tiles, ctx->nsub,
                 ctx->k, ctx->tvec, 0, ctx->inexact ? nullptr : ctx->Einv, ctx->K, ctx->t2, st, need_refresh,
                 ctx->ticket, ctx->zt_scratch, from_op && ctx->split ? ctx->sub_btiles : nullptr, ctx->ntiles,
                 (const double *)nullptr, (int64_t)0, (double *)nullptr);
        ctx->launches++;
        if (ctx->inexact) {
            launch_k(ctx->st, k_egmres, 1, 256, 0, ctx->Edense, (int)ctx->K, ctx->tvec, ctx->t2, ctx->coarse_tol,
                                             ctx->egm_scr, st, need_refresh);
            ctx->launches++;
        }
        return DFL_OK;
    }
    // local entries into a padded slot (+ the caller's extra scalar: CG's
    // rank-local p.w), allgather, unpack, solve
    const int64_t slot = (int64_t)ctx->max_nsub * ctx->k + 1;
    double *mine = ctx->tgather + (int64_t)ctx->rank * slot;
    // the finish kernel's last block also sums the caller's partials into the slot's last entry
    launch_k(ctx->st, k_zt_finish, dim3(ctx->zt_chunks, ctx->nsub), 256, 0, ctx->zt_part, sub_tiles, ctx->nsub,
             ctx->k, mine, 0, nullptr, ctx->K, nullptr, st, need_refresh, ctx->ticket, ctx->zt_scratch,
             from_op && ctx->split ? ctx->sub_btiles : nullptr, ctx->ntiles, extra_part, extra_n,
             extra_part ? mine + slot - 1 : nullptr);
    RC(comm_allgather(ctx, mine, ctx->tgather, slot));
    // unpack the rank slots into t (rank q owns a contiguous subdomain range),
    // t2 = E^-1 t and (CG) the folded p.q, in one single-block kernel
    launch_k(ctx->st, k_unpack, 1, 256, 0, (const double *)ctx->tgather, ctx->nranks, slot,
             (const int64_t *)ctx->rank_cnt_d, ctx->tvec, ctx->inexact ? nullptr : (const double *)ctx->Einv, ctx->K,
             ctx->t2, st, need_refresh, ctx->inexact ? nullptr : fold);
    ctx->launches += 2;
    if (ctx->inexact) {
        launch_k(ctx->st, k_egmres, 1, 256, 0, ctx->Edense, (int)ctx->K, ctx->tvec, ctx->t2, ctx->coarse_tol,
                 ctx->egm_scr, st, need_refresh);
        ctx->launches++;
    }
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
    ctx->comm_timeout_s = comm_timeout_default();
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

int dfl_fabric_set_timeout(dfl_fabric *f, double seconds) {
    if (!f || !(seconds > 0.0)) return DFL_E_STATE;
    std::lock_guard<std::mutex> lk(f->mu);
    f->timeout_s = seconds;
    return DFL_OK;
}

int dfl_ctx_set_fabric(dfl_ctx *ctx, dfl_fabric *f, int rank) {
    if (!ctx || !f || rank < 0 || rank >= f->nranks) return DFL_E_STATE;
    ctx->fab = f;
    ctx->nranks = f->nranks;
    ctx->rank = rank;
    f->ctxs[rank] = ctx;
    return DFL_OK;
}

}  // extern "C"
