// Device context of one rank: uploads the host setup products into
// device-resident layouts and runs the solve phase (deflation.py:254-312)
// entirely on the GPU.  The Krylov loop is a CUDA graph with a device-side
// while-conditional, so a whole CG solve is a handful of launches and no
// host round trip per iteration (single rank); with several ranks the loop is
// host-driven with NCCL collectives between kernels.
#include <map>
#include <mutex>
#include "ctx_impl.cuh"

// format / launch switches (read once per context creation; the A/B record
// of every layout and launch variant that was measured and dropped is in
// profiles/r01/README.md and profiles/r02/README.md)
bool g_use_code = true;       // DFL_NO_CODE=1: no stencil-coded ELL
bool g_use_class = true;      // DFL_NO_CLASS=1: no row-class coded matrices
bool g_use_pcode = true;      // DFL_NO_PCODE=1: no delta/value-coded rows (P)
bool g_no_sell = false;       // DFL_NO_SELL=1: long-row matrices as CSR-vector instead of SELL
bool g_pdl = true;            // DFL_NO_PDL=1: plain launches instead of programmatic dependent launch
bool g_nccl_graph = false;    // DFL_NCCL_GRAPH=1: several NCCL ranks replay the captured CG body
bool g_use_zdict = true;      // DFL_NO_ZDICT=1: Z / AZ columns read dense instead of dictionary-coded
int g_sm_count = 148;

static int stage_in(dfl_ctx *ctx, double *dst, const double *src, int ptr_kind) {
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * ctx->n,
                       ptr_kind == DFL_PTR_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->st));
    return DFL_OK;
}

static int stage_out(dfl_ctx *ctx, double *dst, const double *src, int ptr_kind) {
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * ctx->n,
                       ptr_kind == DFL_PTR_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->st));
    RC(comm_wait(ctx, ctx->st));
    return DFL_OK;
}

int ready(dfl_ctx *ctx) {
    if (!ctx) return DFL_E_STATE;
    if (!ctx->finalized) {
        ctx->err = "context not finalized";
        return DFL_E_STATE;
    }
    CK(cudaSetDevice(ctx->device));
    return DFL_OK;
}

static int rank_dot(dfl_ctx *ctx, const double *a, const double *b, double *out) {
    const unsigned nb = (unsigned)std::min<int64_t>(std::max<int64_t>(1, ctx->nblk), 4 * 148);
    launch_k(ctx->st, k_dot, nb, kBlock, 0, a, b, ctx->n, ctx->dpart, nullptr);
    launch_k(ctx->st, k_reduce, 1, 1024, 0, ctx->dpart, nb, ctx->scal);
    ctx->launches += 2;
    if (multi(ctx)) {
        RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
        launch_k(ctx->st, k_rank_sum, 1, 32, 0, ctx->sgather, ctx->nranks, 8, 1, ctx->scal + 1);
        ctx->launches++;
        CK(cudaMemcpyAsync(out, ctx->scal + 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    } else {
        CK(cudaMemcpyAsync(out, ctx->scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    }
    RC(comm_wait(ctx, ctx->st));
    return DFL_OK;
}


// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char *dfl_breakdown_string(int code) {
    switch (code) {
        case DFL_BRK_NONE: return "";
        case DFL_BRK_CURVATURE: return "non-positive curvature p'Ap";
        case DFL_BRK_RZ: return "preconditioned residual product degenerated";
        case DFL_BRK_RHO: return "rho degenerated in the BiCG stage";
        case DFL_BRK_SHADOW: return "shadow product degenerated in the BiCG stage";
        case DFL_BRK_MR: return "minimal-residual basis degenerated";
        case DFL_BRK_OMEGA: return "stabilization weight vanished";
        default: return "unknown breakdown";
    }
}

int dfl_ctx_create(int device, dfl_ctx **out) {
    if (!out) return DFL_E_STATE;
    *out = nullptr;
    auto *ctx = new dfl_ctx;
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_state, sizeof(KState));
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) g_sm_count = ctx->sm_count;
    if (e == cudaSuccess) {
        auto on = [](const char *name) {
            const char *v = getenv(name);
            return v && v[0] == '1';
        };
        g_use_code = !on("DFL_NO_CODE");
        g_use_class = !on("DFL_NO_CLASS");
        g_use_pcode = !on("DFL_NO_PCODE");
        g_no_sell = on("DFL_NO_SELL");
        g_pdl = !on("DFL_NO_PDL");
        g_nccl_graph = on("DFL_NCCL_GRAPH");
        g_use_zdict = !on("DFL_NO_ZDICT");
    }
    if (e != cudaSuccess) {
        dfl::set_setup_error(std::string("CUDA context creation failed: ") + cudaGetErrorString(e));
        delete ctx;
        return DFL_E_CUDA;
    }
    *out = ctx;
    return DFL_OK;
}

void dfl_ctx_destroy(dfl_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->st) cudaStreamSynchronize(ctx->st);
    if (ctx->loop_exec) cudaGraphExecDestroy(ctx->loop_exec);
    if (ctx->solve_exec) cudaGraphExecDestroy(ctx->solve_exec);
    if (ctx->bg_exec) cudaGraphExecDestroy(ctx->bg_exec);
    for (auto &e : ctx->body_exec)
        if (e) cudaGraphExecDestroy(e);
    if (ctx->h_state2) cudaFreeHost(ctx->h_state2);
    for (cudaEvent_t e : ctx->ev_it)
        if (e) cudaEventDestroy(e);
    if (ctx->h_bstate) cudaFreeHost(ctx->h_bstate);
    for (void *p : ctx->allocs) cudaFree(p);
    if (ctx->h_state) cudaFreeHost(ctx->h_state);
    if (ctx->h_dots) cudaFreeHost(ctx->h_dots);
    if (ctx->h_gm) cudaFreeHost(ctx->h_gm);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->comm) g_nccl.CommDestroy(ctx->comm);
    if (ctx->st2) cudaStreamDestroy(ctx->st2);
    if (ctx->st_copy) cudaStreamDestroy(ctx->st_copy);
    if (ctx->st_if) cudaStreamDestroy(ctx->st_if);
    if (ctx->ev_packed) cudaEventDestroy(ctx->ev_packed);
    if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
    if (ctx->st) cudaStreamDestroy(ctx->st);
    delete ctx;
}

const char *dfl_last_error(const dfl_ctx *ctx) { return ctx ? ctx->err.c_str() : dfl::setup_error(); }

int64_t dfl_ctx_device_bytes(const dfl_ctx *ctx) { return ctx ? ctx->bytes : 0; }

int dfl_ctx_set_operator(dfl_ctx *ctx, const dfl_csr *A, int32_t nsub, const int64_t *sub_offsets, int32_t nnbr,
                         const int32_t *nbr_rank, const int64_t *recv_counts, const int64_t *send_counts,
                         const int64_t *send_idx) {
    if (!ctx || !A || nsub < 1 || !sub_offsets) return DFL_E_STATE;
    CK(cudaSetDevice(ctx->device));
    if (sub_offsets[0] != 0 || sub_offsets[nsub] != A->nrows) {
        ctx->err = "subdomain offsets do not span the operator rows";
        return DFL_E_PARTITION;
    }
    for (int s = 0; s < nsub; ++s)
        if (sub_offsets[s + 1] <= sub_offsets[s]) {
            ctx->err = "empty subdomain";
            return DFL_E_PARTITION;
        }
    ctx->n = A->nrows;
    ctx->n_ghost = A->ncols - A->nrows;
    if (ctx->n_ghost < 0) {
        ctx->err = "operator has fewer columns than rows";
        return DFL_E_DIMENSION;
    }
    ctx->nsub = nsub;
    ctx->sub_off.assign(sub_offsets, sub_offsets + nsub + 1);
    HostRows h{A->nrows, A->ncols, A->row_ptr, A->col_idx, A->values};
    // the operator: row-class coded when it has few distinct rows (structured
    // grids; 1 byte per row instead of 12 per entry), else uniform ELL (at the
    // HBM roofline); FMT_CODE only pays off for the V-cycle kernels with longer
    // epilogues (profiles/r01).  A rank with ghost columns splits the
    // operator: the rows with ghost columns (the boundary pass, k_op_bnd, after
    // the halo) go into a matrix of their own, Abnd (ELL / CSR, one row per
    // boundary slot), and are emptied in Aop, so the interior rows -- which
    // run while the halo is in flight -- keep the class-coded layout.
    //
    // Several subdomains in one context: the rows coupling to another
    // subdomain have irregular column offsets under a box ordering (300^3 as
    // 2x2x2 boxes), so the whole operator does not class-code; they take the
    // same boundary pass (here with no halo), the rest stays class-coded.
    const char *no_ov = getenv("DFL_NO_OVERLAP");
    const bool overlap_ok = !(no_ov && no_ov[0] == '1');
    std::vector<int> rowsub((size_t)A->nrows);
    for (int s = 0; s < nsub; ++s)
        for (int64_t i = sub_offsets[s]; i < sub_offsets[s + 1]; ++i) rowsub[(size_t)i] = s;
    bool cross_rule = false;  // boundary rows also = rows coupling to another subdomain
    auto is_bnd = [&](int64_t i) {
        const int s = rowsub[(size_t)i];
        for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; ++e) {
            const int64_t c = A->col_idx[e];
            if (c >= A->nrows) return true;
            if (cross_rule && (c < sub_offsets[s] || c >= sub_offsets[s + 1])) return true;
        }
        return false;
    };
    //
    // Rows of rare classes (a matrix with more than kMaxClass distinct
    // non-dominant rows, e.g. jump coefficients: 242 distinct rows, the 64
    // most frequent cover 99.8% of them) take the boundary pass too.
    bool will_split = multi(ctx) && A->ncols > A->nrows && overlap_ok;
    bool full_class = false, full_uploaded = false;
    if (!will_split && overlap_ok && g_use_class) {
        RC(upload_matrix(ctx, h, ctx->Aop, ctx->sub_off, nullptr, true, nullptr, nullptr, false, false, true));
        full_uploaded = true;
        full_class = ctx->Aop.fmt == FMT_CLASS;
        if (!full_class && nsub > 1) will_split = true;  // retry with the coupling rows apart
    }
    if (will_split && nsub > 1) cross_rule = true;
    std::vector<uint8_t> exc;
    auto is_bnd2 = [&](int64_t i) { return (!exc.empty() && exc[(size_t)i]) || is_bnd(i); };
    std::vector<int64_t> ib_ptr, bb_ptr, bb_col;
    std::vector<double> bb_val;
    // interior copy (boundary rows emptied: skipped by the interior pass) +
    // the boundary rows' own matrix; true if the interior class-codes
    auto build_split = [&](bool &interior_class) -> int {
        ib_ptr.assign(A->nrows + 1, 0);
        bb_ptr.assign(1, 0);
        bb_col.clear();
        bb_val.clear();
        for (int64_t i = 0; i < A->nrows; ++i) {
            if (is_bnd2(i)) {
                for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; ++e) {
                    bb_col.push_back(A->col_idx[e]);
                    bb_val.push_back(A->values[e]);
                }
                bb_ptr.push_back((int64_t)bb_col.size());
                ib_ptr[i + 1] = ib_ptr[i];
            } else {
                ib_ptr[i + 1] = ib_ptr[i] + (A->row_ptr[i + 1] - A->row_ptr[i]);
            }
        }
        std::vector<int64_t> icol((size_t)ib_ptr[A->nrows]);
        std::vector<double> ival((size_t)ib_ptr[A->nrows]);
        for (int64_t i = 0, q = 0; i < A->nrows; ++i)
            if (ib_ptr[i + 1] > ib_ptr[i])
                for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; ++e, ++q) {
                    icol[q] = A->col_idx[e];
                    ival[q] = A->values[e];
                }
        HostRows hi{A->nrows, A->ncols, ib_ptr.data(), icol.data(), ival.data()};
        RC(upload_matrix(ctx, hi, ctx->Aop, ctx->sub_off, nullptr, true, nullptr, nullptr, false, false, true));
        const int64_t nb = (int64_t)bb_ptr.size() - 1;
        HostRows hb{nb, A->ncols, bb_ptr.data(), bb_col.data(), bb_val.data()};
        RC(upload_matrix(ctx, hb, ctx->Abnd, {0, nb}, nullptr, true, nullptr, nullptr, false, false, false));
        interior_class = ctx->Aop.fmt == FMT_CLASS;
        return DFL_OK;
    };
    if (!full_class) {
        bool interior_class = false;
        if (will_split) RC(build_split(interior_class));
        if (!interior_class && overlap_ok && g_use_class) {
            // second attempt: the rows of rare classes into the boundary pass as well
            exc = class_exceptions(h, [&](int64_t i) { return is_bnd(i); });
            if (!exc.empty()) {
                will_split = true;
                RC(build_split(interior_class));
            }
        }
        if (will_split && !multi(ctx) && !interior_class) {
            // one context: the split only pays when the interior class-codes
            will_split = false;
            exc.clear();
            RC(upload_matrix(ctx, h, ctx->Aop, ctx->sub_off, nullptr, true, nullptr, nullptr, false, false, true));
        } else if (!will_split && !full_uploaded) {
            RC(upload_matrix(ctx, h, ctx->Aop, ctx->sub_off, nullptr, true, nullptr, nullptr, false, false, true));
        }
    }
    if (getenv("DFL_SETUP_VERBOSE"))
        fprintf(stderr, "dfl: operator fmt %d (class %d), split %d, exception rows %lld, boundary rows %lld\n",
                ctx->Aop.fmt, (int)full_class, (int)will_split,
                (long long)std::count(exc.begin(), exc.end(), (uint8_t)1), (long long)(bb_ptr.empty() ? 0 : bb_ptr.size() - 1));
    ctx->op_nnz = A->row_ptr[A->nrows] - A->row_ptr[0];
    int64_t nrecv = 0;
    ctx->nbr.clear();
    ctx->recv_cnt.clear();
    ctx->send_cnt.clear();
    ctx->nsend = 0;
    for (int q = 0; q < nnbr; ++q) {
        ctx->nbr.push_back(nbr_rank[q]);
        ctx->recv_cnt.push_back(recv_counts[q]);
        ctx->send_cnt.push_back(send_counts[q]);
        nrecv += recv_counts[q];
        ctx->nsend += send_counts[q];
    }
    if (nrecv != ctx->n_ghost) {
        ctx->err = "halo plan receives " + std::to_string(nrecv) + " values for " + std::to_string(ctx->n_ghost) +
                   " ghost columns";
        return DFL_E_COMM;
    }
    if (ctx->nsend > 0) {
        std::vector<int> si(send_idx, send_idx + ctx->nsend);
        for (int v : si)
            if (v < 0 || v >= ctx->n) {
                ctx->err = "halo send index out of range";
                return DFL_E_COMM;
            }
        RC(upload(ctx, &ctx->send_idx, si.data(), ctx->nsend));
        RC(dalloc(ctx, &ctx->sendbuf, ctx->nsend));
    }
    // boundary rows (ghost columns; with several subdomains also the rows
    // coupling to another one): second pass of the operator
    ctx->split = false;
    if (will_split) {
        std::vector<uint8_t> flag(ctx->n, 0);
        std::vector<int> rows, bs, bc;
        std::vector<int64_t> sbt{0};
        for (int s = 0; s < nsub; ++s) {
            const size_t first = rows.size();
            for (int64_t i = sub_offsets[s]; i < sub_offsets[s + 1]; ++i)
                if (is_bnd2(i)) {
                    flag[i] = 1;
                    rows.push_back((int)i);
                }
            for (size_t j = first; j < rows.size(); j += kBlock) {
                bs.push_back((int)j);
                bc.push_back((int)std::min<size_t>(kBlock, rows.size() - j));
            }
            sbt.push_back((int64_t)bs.size());
        }
        ctx->nbtiles = (int64_t)bs.size();
        RC(upload(ctx, &ctx->bflag, flag.data(), ctx->n));
        RC(upload(ctx, &ctx->brows, rows.data(), (int64_t)rows.size()));
        RC(upload(ctx, &ctx->bstart, bs.data(), (int64_t)bs.size()));
        RC(upload(ctx, &ctx->bcnt, bc.data(), (int64_t)bc.size()));
        RC(upload(ctx, &ctx->sub_btiles, sbt.data(), (int64_t)sbt.size()));
        if (!ctx->st2) {
            CK(cudaStreamCreateWithFlags(&ctx->st2, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ctx->ev_packed, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
        }
        ctx->split = true;
    }
    ctx->pending.assign(nsub, nullptr);
    ctx->pending_set.assign(nsub, 0);
    ctx->have_op = true;
    ctx->finalized = false;
    return DFL_OK;
}

int dfl_ctx_add_hierarchy(dfl_ctx *ctx, int32_t sub, const dfl_hier *h) {
    if (!ctx || !h) return DFL_E_STATE;
    if (!ctx->have_op || sub < 0 || sub >= ctx->nsub) {
        ctx->err = "hierarchy for an unknown subdomain (set the operator first)";
        return DFL_E_STATE;
    }
    const dfl::Hierarchy &src = *h->sp;
    if (sub > 0 && src.relax != ctx->relax) {
        ctx->err = "all subdomains must use the same relaxation";
        return DFL_E_CONFIG;
    }
    ctx->relax = src.relax;
    ctx->pending[sub] = h->sp;
    ctx->pending_set[sub] = 1;
    return DFL_OK;
}

// Lossless dictionary coding of dense per-row columns (the Z and AZ columns
// of the hot loop): every column's distinct values (by bit pattern) go to a
// table, each row stores one uint16 index per column, `stride` indices per
// row (row-major, one vector load).  Linear deflation on a grid has a few
// hundred distinct values per column (coordinates repeat along the other
// axes), so 2 bytes replace 8 per value.  Returns false (caller keeps the
// dense columns) if a column has more than 65536 distinct values.
static bool dict_code(const double *cols, int ncol, int64_t n, int stride, std::vector<uint16_t> &codes,
                      std::vector<double> &tab, int *off) {
    constexpr int kBits = 17;
    constexpr uint64_t kSlots = 1ull << kBits;  // load factor <= 1/2 at 65536 values
    codes.assign((size_t)n * stride, 0);
    tab.clear();
    std::vector<uint64_t> key(kSlots);
    std::vector<int32_t> idx(kSlots);
    for (int c = 0; c < ncol; ++c) {
        off[c] = (int)tab.size();
        std::fill(idx.begin(), idx.end(), -1);
        int cnt = 0;
        const double *col = cols + (size_t)c * n;
        for (int64_t i = 0; i < n; ++i) {
            uint64_t b;
            std::memcpy(&b, col + i, 8);
            uint64_t h = (b * 0x9E3779B97F4A7C15ull) >> (64 - kBits);
            while (idx[h] >= 0 && key[h] != b) h = (h + 1) & (kSlots - 1);
            if (idx[h] < 0) {
                if (cnt == 65536) return false;
                key[h] = b;
                idx[h] = cnt++;
                tab.push_back(col[i]);
            }
            codes[(size_t)i * stride + c] = (uint16_t)idx[h];
        }
    }
    return true;
}

static int code_stride(int ncol) { return ncol <= 1 ? 1 : ncol <= 2 ? 2 : ncol <= 4 ? 4 : 8; }

int dfl_ctx_set_deflation(dfl_ctx *ctx, int32_t k, const double *zcols, const dfl_csr *AZ, int64_t K,
                          const double *Einv, int32_t first_sub) {
    if (!ctx || !AZ || !Einv) return DFL_E_STATE;
    if (!ctx->have_op) {
        ctx->err = "set the operator before the deflation basis";
        return DFL_E_STATE;
    }
    if (k < 1 || k > kKmax || K % k != 0 || AZ->nrows != ctx->n || AZ->ncols != K) {
        ctx->err = "inconsistent deflation dimensions";
        return DFL_E_DIMENSION;
    }
    CK(cudaSetDevice(ctx->device));
    ctx->k = k;
    ctx->K = K;
    ctx->first_sub = first_sub;
    const int m = (int)(K / k);
    ctx->rank_nsub.assign(ctx->nranks, 0);
    for (int q = 0; q < ctx->nranks; ++q) ctx->rank_nsub[q] = m / ctx->nranks + (q < m % ctx->nranks ? 1 : 0);
    ctx->max_nsub = *std::max_element(ctx->rank_nsub.begin(), ctx->rank_nsub.end());
    {
        std::vector<int64_t> rc(ctx->nranks);
        for (int q = 0; q < ctx->nranks; ++q) rc[q] = (int64_t)ctx->rank_nsub[q] * k;
        RC(upload(ctx, &ctx->rank_cnt_d, rc.data(), (int64_t)ctx->nranks));
    }
    if (ctx->rank_nsub[ctx->rank] != ctx->nsub) {
        ctx->err = "rank owns " + std::to_string(ctx->nsub) + " subdomains, placement expects " +
                   std::to_string(ctx->rank_nsub[ctx->rank]);
        return DFL_E_PARTITION;
    }
    // Z columns 1..k-1, column-major for coalesced loads
    std::vector<double> zc((size_t)std::max(1, k - 1) * ctx->n, 0.0);
    for (int c = 1; c < k; ++c)
        for (int64_t i = 0; i < ctx->n; ++i) zc[(size_t)(c - 1) * ctx->n + i] = zcols[i * (k - 1) + (c - 1)];
    RC(upload(ctx, &ctx->zcols, zc.data(), (int64_t)zc.size()));
    // AZ: own-subdomain block dense (k x n), the other entries as an extras CSR
    // (kernels.cuh, ProjArgs); column order inside a row is preserved
    const int64_t n = ctx->n;
    std::vector<double> azd((size_t)k * n, 0.0);
    std::vector<int> xptr(n + 1, 0), xcol;
    std::vector<double> xval;
    for (int s = 0; s < ctx->nsub; ++s) {
        const int64_t own0 = (int64_t)(first_sub + s) * k;
        for (int64_t i = ctx->sub_off[s]; i < ctx->sub_off[s + 1]; ++i) {
            for (int64_t e = AZ->row_ptr[i]; e < AZ->row_ptr[i + 1]; ++e) {
                const int64_t c = AZ->col_idx[e];
                if (c >= own0 && c < own0 + k) {
                    azd[(size_t)(c - own0) * n + i] = AZ->values[e];
                } else {
                    xcol.push_back((int)c);
                    xval.push_back(AZ->values[e]);
                }
            }
            xptr[i + 1] = (int)xcol.size();
        }
    }
    ctx->az_nnz = AZ->row_ptr[n];
    ctx->ax_nnz = (int64_t)xcol.size();
    RC(upload(ctx, &ctx->azd, azd.data(), (int64_t)azd.size()));
    ctx->zcode = nullptr;
    ctx->acode = nullptr;
    if (g_use_zdict && n > 0) {
        std::vector<uint16_t> codes;
        std::vector<double> tab;
        // row stride code_stride(k) (the operator kernel's Z'y width NV: a
        // compile-time stride there), columns 1..k-1 in its first k-1 slots
        if (k > 1 && dict_code(zc.data(), k - 1, n, code_stride(k), codes, tab, ctx->ztab_off)) {
            ctx->zs = code_stride(k);
            RC(upload(ctx, &ctx->zcode, codes.data(), (int64_t)codes.size()));
            RC(upload(ctx, &ctx->ztab, tab.data(), (int64_t)tab.size()));
            ctx->ztab_n = (int64_t)tab.size();
        }
        if (dict_code(azd.data(), k, n, code_stride(k), codes, tab, ctx->atab_off)) {
            RC(upload(ctx, &ctx->acode, codes.data(), (int64_t)codes.size()));
            RC(upload(ctx, &ctx->atab, tab.data(), (int64_t)tab.size()));
            ctx->atab_n = (int64_t)tab.size();
        }
    }
    if (ctx->ax_nnz > 0) {
        RC(upload(ctx, &ctx->ax_ptr, xptr.data(), n + 1));
        std::vector<uint8_t> xf((size_t)n, 0);
        for (int64_t i = 0; i < n; ++i) xf[(size_t)i] = xptr[i + 1] > xptr[i] ? 1 : 0;
        RC(upload(ctx, &ctx->ax_flag, xf.data(), n));
        RC(upload(ctx, &ctx->ax_col, xcol.data(), ctx->ax_nnz));
        RC(upload(ctx, &ctx->ax_val, xval.data(), ctx->ax_nnz));
    }
    if (!ctx->sub_off_d) RC(upload(ctx, &ctx->sub_off_d, ctx->sub_off.data(), (int64_t)ctx->sub_off.size()));
    RC(upload(ctx, &ctx->Einv, Einv, K * K));
    RC(dalloc(ctx, &ctx->tvec, K));
    RC(dalloc(ctx, &ctx->t2, K));
    RC(dalloc(ctx, &ctx->tgather, (int64_t)ctx->nranks * (ctx->max_nsub * k + 1)));  // + the p.w slot of CG
    ctx->deflation = true;
    return DFL_OK;
}

int dfl_ctx_set_inexact(dfl_ctx *ctx, const double *E, double coarse_tol) {
    if (!ctx || !ctx->deflation) {
        if (ctx) ctx->err = "set the deflation basis before the inexact coarse solve";
        return DFL_E_STATE;
    }
    if (E == nullptr) {
        ctx->inexact = false;
        return DFL_OK;
    }
    CK(cudaSetDevice(ctx->device));
    const int64_t K = ctx->K;
    if (K > 1024) {
        ctx->err = "inexact coarse solve supports K <= 1024";
        return DFL_E_DIMENSION;
    }
    if (!ctx->Edense) {
        RC(dalloc(ctx, &ctx->Edense, K * K));
        RC(dalloc(ctx, &ctx->egm_scr, 2 * (K + 1) * K + 8 * (K + 1)));
    }
    CK(cudaMemcpy(ctx->Edense, E, sizeof(double) * K * K, cudaMemcpyHostToDevice));
    ctx->coarse_tol = coarse_tol;
    ctx->inexact = true;
    return DFL_OK;
}

int dfl_ctx_finalize(dfl_ctx *ctx) {
    dfl::NvtxRange nv("dfl.upload");
    if (!ctx) return DFL_E_STATE;
    if (!ctx->have_op) {
        ctx->err = "no operator uploaded";
        return DFL_E_STATE;
    }
    for (int s = 0; s < ctx->nsub; ++s)
        if (!ctx->pending_set[s]) {
            ctx->err = "missing hierarchy for subdomain " + std::to_string(s);
            return DFL_E_STATE;
        }
    CK(cudaSetDevice(ctx->device));
    // graphs captured against the previous buffers (a context finalized again)
    if (ctx->solve_exec) cudaGraphExecDestroy(ctx->solve_exec), ctx->solve_exec = nullptr, ctx->solve_key.clear();
    if (ctx->loop_exec) cudaGraphExecDestroy(ctx->loop_exec), ctx->loop_exec = nullptr, ctx->loop_key = -1;
    if (ctx->bg_exec) cudaGraphExecDestroy(ctx->bg_exec), ctx->bg_exec = nullptr, ctx->bg_key = -1;
    for (auto &e : ctx->body_exec)
        if (e) cudaGraphExecDestroy(e), e = nullptr;
    ctx->body_key = -1;
    RC(build_groups(ctx));
    ctx->pending.clear();
    ctx->pending.shrink_to_fit();
    RC(build_tiles(ctx));
    const int64_t nx = ctx->n + ctx->n_ghost;
    RC(dalloc(ctx, &ctx->b, ctx->n));
    RC(dalloc(ctx, &ctx->bp, ctx->n));
    RC(dalloc(ctx, &ctx->x, nx));
    RC(dalloc(ctx, &ctx->xin, nx));
    RC(dalloc(ctx, &ctx->p, nx));
    RC(dalloc(ctx, &ctx->r, ctx->n));
    RC(dalloc(ctx, &ctx->z, ctx->n));
    RC(dalloc(ctx, &ctx->w, ctx->n));
    RC(dalloc(ctx, &ctx->tmp, ctx->n));
    RC(dalloc(ctx, &ctx->yout, ctx->n));
    ctx->nblk = cdiv(ctx->n, kBlock);
    {
        // one full wave of the grid-stride vector kernels (the smallest residency among them)
        const int occ = std::min({occupancy(k_project<0, 4>), occupancy(k_project<1, 4>),
                                  occupancy(k_cg_update), occupancy(k_cg_p), occupancy(k_dot)});
        ctx->vgrid = std::max<int64_t>(1, std::min<int64_t>(ctx->nblk, (int64_t)occ * ctx->sm_count));
    }
    int64_t vparts = 0;
    for (auto &g : ctx->groups)
        vparts += g.lv.empty() ? std::max<int64_t>(1, std::min<int64_t>(cdiv(g.row1 - g.row0, kBlock), 64))
                               : parts_for(g.lv[0].A);
    // partial-sum scratch: one slot per block of the row kernels, or 3 per
    // block of the multi-dot kernels (grid <= 4 * SMs)
    const int64_t dslots = std::max({ctx->nblk, vparts, kDotStride * std::max<int64_t>(ctx->nblk, 4 * ctx->sm_count)});
    RC(dalloc(ctx, &ctx->dpart, dslots + 64));
    RC(dalloc(ctx, &ctx->zt_part, (ctx->ntiles + ctx->nbtiles) * kKmax + 64));
    // ~512 tiles per k_zt_finish block: enough blocks that the partial reads
    // of a 10^6-row subdomain are spread over the GPU, few enough that the
    // last block's chunk sum stays short
    ctx->zt_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(kZtMaxChunks, ctx->ntiles / std::max(1, ctx->nsub) / 512));
    RC(dalloc(ctx, &ctx->zt_scratch, (int64_t)ctx->nsub * kKmax * kZtMaxChunks + 64));
    RC(dalloc(ctx, &ctx->scal, 16));
    RC(dalloc(ctx, &ctx->sgather, (int64_t)8 * ctx->nranks));
    RC(dalloc(ctx, &ctx->state, 1));
    CK(cudaMallocHost(&ctx->h_dots, 16 * sizeof(double)));
    RC(dalloc(ctx, &ctx->ticket, 4));
    CK(cudaMemset(ctx->ticket, 0, 4 * sizeof(unsigned int)));
    CK(cudaMemset(ctx->x, 0, sizeof(double) * nx));
    CK(cudaMemset(ctx->xin, 0, sizeof(double) * nx));
    CK(cudaMemset(ctx->p, 0, sizeof(double) * nx));
    CK(cudaDeviceSynchronize());
    ctx->finalized = true;
    return DFL_OK;
}

int dfl_ctx_wait_stream(dfl_ctx *ctx, void *stream) {
    if (!ctx) return DFL_E_STATE;
    CK(cudaSetDevice(ctx->device));
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, (cudaStream_t)stream));
    const cudaError_t w = cudaStreamWaitEvent(ctx->st, e, 0);
    cudaEventDestroy(e);
    CK(w);
    return DFL_OK;
}

int dfl_solve(dfl_ctx *ctx, const dfl_solve_params *p, const double *b, double *x, int ptr_kind, dfl_report *rep) {
    dfl::NvtxRange nv("dfl.solve");
    RC(ready(ctx));
    if (!p || !rep) return DFL_E_STATE;
    if (p->solver < DFL_SOLVER_CG || p->solver > DFL_SOLVER_FGMRES) {
        ctx->err = "solver must be cg, bicgstab2, gmres or fgmres";
        return DFL_E_CONFIG;
    }
    if (p->deflated && !ctx->deflation) {
        ctx->err = "deflated solve requested but no deflation basis uploaded";
        return DFL_E_STATE;
    }
    std::memset(rep, 0, sizeof *rep);
    ctx->launches = 0;
    cudaEvent_t e_h0, e_h1;
    CK(cudaEventCreate(&e_h0));
    CK(cudaEventCreate(&e_h1));
    CK(cudaEventRecord(e_h0, ctx->st));
    RC(stage_in(ctx, ctx->b, b, ptr_kind));
    if (p->x0_given && !p->deflated) {
        if (!ctx->x0) RC(dalloc(ctx, &ctx->x0, ctx->n));
        RC(stage_in(ctx, ctx->x0, x, ptr_kind));
    }
    CK(cudaEventRecord(ctx->ev0, ctx->st));
    const char *ng = getenv("DFL_NO_GRAPH");
    const bool bicg = p->solver != DFL_SOLVER_CG;  // host-driven solvers
    const bool use_graph = !bicg && !multi(ctx) && !(ng && ng[0] == '1');
    KState bstate{};
    const bool dev_loop = !multi(ctx) && !(ng && ng[0] == '1');  // device-side Krylov loops (single rank)
    {
        dfl::NvtxRange kr("dfl.solve.krylov");
        if (p->solver == DFL_SOLVER_BICGSTAB2) {
            if (dev_loop)
                RC(bicg_solve_graph(ctx, p, bstate));
            else
                RC(bicg_solve_dev(ctx, p, bstate));
            RC(lift_dev(ctx, p));
        } else if (p->solver == DFL_SOLVER_GMRES || p->solver == DFL_SOLVER_FGMRES) {
            RC(gmres_solve_dev(ctx, p, p->solver == DFL_SOLVER_FGMRES, bstate));
            RC(lift_dev(ctx, p));
        } else {
            RC(cg_solve_dev(ctx, p, use_graph));
        }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev1, ctx->st));
    // x goes back on its own stream while the true-residual kernels run on
    // the solve stream (both only read xin)
    if (!ctx->st_copy) CK(cudaStreamCreateWithFlags(&ctx->st_copy, cudaStreamNonBlocking));
    CK(cudaStreamWaitEvent(ctx->st_copy, ctx->ev1, 0));
    CK(cudaMemcpyAsync(x, ctx->xin, sizeof(double) * ctx->n,
                       ptr_kind == DFL_PTR_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->st_copy));
    CK(cudaEventRecord(e_h1, ctx->st_copy));
    CK(cudaMemcpyAsync(ctx->h_state, ctx->state, sizeof(KState), cudaMemcpyDeviceToHost, ctx->st));
    RC(comm_wait(ctx, ctx->st));
    const KState s = bicg ? bstate : *ctx->h_state;
    // true residual ||b - A x|| / ||b|| (deflation.py:293-297; outside the timed span)
    const int64_t solve_launches = ctx->launches;
    double rr = 0.0;
    if (s.bnorm != 0.0) {
        RC(op_apply_dev(ctx, ctx->xin, ctx->tmp, 1, ctx->b, false, nullptr, 0));
        RC(rank_dot(ctx, ctx->tmp, ctx->tmp, &rr));
    }
    RC(comm_wait(ctx, ctx->st_copy));
    float ms_h2d = 0, ms_solve = 0, ms_d2h = 0;
    CK(cudaEventElapsedTime(&ms_h2d, e_h0, ctx->ev0));
    CK(cudaEventElapsedTime(&ms_solve, ctx->ev0, ctx->ev1));
    CK(cudaEventElapsedTime(&ms_d2h, ctx->ev1, e_h1));
    cudaEventDestroy(e_h0);
    cudaEventDestroy(e_h1);
    rep->iterations = s.iters;
    rep->converged = s.converged || (s.resnorm <= s.target);
    if (s.breakdown) rep->converged = 0;
    rep->breakdown = rep->converged ? DFL_BRK_NONE : s.breakdown;
    rep->device_loop = (use_graph || (p->solver == DFL_SOLVER_BICGSTAB2 && dev_loop)) ? 1 : 0;
    rep->bnorm = s.bnorm;
    rep->resnorm = s.resnorm;
    rep->breakdown_value = s.brk_val;
    rep->solve_seconds = ms_solve * 1e-3;
    rep->h2d_seconds = ms_h2d * 1e-3;
    rep->d2h_seconds = ms_d2h * 1e-3;
    rep->kernel_launches = solve_launches + (use_graph ? ctx->body_kernels * std::max(1, s.iters) +
                                                            ctx->if_kernels * (s.iters / std::max(1, p->refresh_every))
                                                      : 0);
    rep->relative_residual = s.bnorm == 0.0 ? 0.0 : std::sqrt(std::max(rr, 0.0)) / s.bnorm;
    return DFL_OK;
}

// pinned host block cache (bytes -> free blocks; live block -> bytes)
static std::mutex g_host_mu;
static std::multimap<int64_t, void *> g_host_free;
static std::map<void *, int64_t> g_host_live;

void *dfl_host_alloc(int64_t bytes) {
    if (bytes <= 0) return nullptr;
    std::lock_guard<std::mutex> lk(g_host_mu);
    void *p = nullptr;
    auto it = g_host_free.find(bytes);
    if (it != g_host_free.end()) {
        p = it->second;
        g_host_free.erase(it);
    } else if (cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    g_host_live[p] = bytes;
    return p;
}

void dfl_host_free(void *ptr) {
    if (!ptr) return;
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host_live.find(ptr);
    if (it == g_host_live.end()) return;
    // keep at most four cached blocks per size
    if (g_host_free.count(it->second) < 4)
        g_host_free.emplace(it->second, ptr);
    else
        cudaFreeHost(ptr);
    g_host_live.erase(it);
}

int dfl_op_apply(dfl_ctx *ctx, const double *x, double *y, int ptr_kind) {
    RC(ready(ctx));
    RC(stage_in(ctx, ctx->xin, x, ptr_kind));
    RC(op_apply_dev(ctx, ctx->xin, ctx->yout, 0, nullptr, false, nullptr, 0));
    return stage_out(ctx, y, ctx->yout, ptr_kind);
}

int dfl_precond_apply(dfl_ctx *ctx, const double *r, double *z, int ptr_kind) {
    RC(ready(ctx));
    RC(stage_in(ctx, ctx->tmp, r, ptr_kind));
    RC(vcycle(ctx, ctx->tmp, ctx->yout, nullptr, nullptr, nullptr));
    return stage_out(ctx, z, ctx->yout, ptr_kind);
}

int dfl_project(dfl_ctx *ctx, const double *r, double *out, int ptr_kind) {
    RC(ready(ctx));
    if (!ctx->deflation) {
        ctx->err = "no deflation basis";
        return DFL_E_STATE;
    }
    RC(stage_in(ctx, ctx->tmp, r, ptr_kind));
    RC(project_dev(ctx, ctx->tmp, ctx->yout, nullptr, 0));
    return stage_out(ctx, out, ctx->yout, ptr_kind);
}

int dfl_coarse_lift(dfl_ctx *ctx, const double *r, double *out, int ptr_kind) {
    RC(ready(ctx));
    if (!ctx->deflation) {
        ctx->err = "no deflation basis";
        return DFL_E_STATE;
    }
    RC(stage_in(ctx, ctx->tmp, r, ptr_kind));
    launch_k(ctx->st, k_zt_vec, (unsigned)ctx->ntiles, kBlock, 0, ctx->tiles, ctx->tmp, ctx->zcols, ctx->n, ctx->k,
             ctx->zt_part, zcode_of(ctx));
    RC(zt_to_t2(ctx, nullptr, 0, false));
    launch_k(ctx->st, k_lift, (unsigned)ctx->ntiles, kBlock, 0, ctx->tiles, ctx->tile_sub, ctx->tmp, ctx->zcols, ctx->n,
             ctx->k, ctx->t2, (int64_t)ctx->first_sub * ctx->k, ctx->yout, 0, zcode_of(ctx));
    return stage_out(ctx, out, ctx->yout, ptr_kind);
}

int dfl_dot(dfl_ctx *ctx, const double *a, const double *b, int ptr_kind, double *out) {
    RC(ready(ctx));
    RC(stage_in(ctx, ctx->tmp, a, ptr_kind));
    RC(stage_in(ctx, ctx->yout, b, ptr_kind));
    return rank_dot(ctx, ctx->tmp, ctx->yout, out);
}

}  // extern "C"
