// CG on the device: the loop body captured as a CUDA graph with a
// device-side while-conditional (single rank) or replayed host-driven.
#include "ctx_impl.cuh"

// ---------------------------------------------------------------------------
// Krylov scalar steps (single block).  With several ranks the per-rank sums
// arrive allgathered in `gath` (stride 8) and are added in rank order, which
// mirrors the ascending-order allreduce of runtime.py:214-219.

__device__ __forceinline__ double scalar_in(const double *part, int64_t nparts, const double *gath, int nranks,
                                            int slot) {
    if (gath == nullptr) return reduce_parts(part, nparts);
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += gath[q * 8 + slot];
    return s;
}

// bnorm = ||b|| (deflation.py:266), atol = tol * bnorm
__global__ void k_cg_start(KState *st, const double *part, int64_t nparts, const double *gath, int nranks,
                           double tol, int maxiter, int refresh) {
    DFL_PDL_ENTRY;
    const double bb = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    KState s{};
    s.bnorm = sqrt(fmax(bb, 0.0));
    s.target = tol * s.bnorm;
    s.maxiter = maxiter;
    s.refresh_every = refresh;
    if (s.bnorm == 0.0) {
        s.done = 1;
        s.converged = 1;
    }
    *st = s;
}

// ||b'|| of the projected rhs: zero -> zero solution; r = b' meets the target
// -> converged at 0 iterations (krylov.py:101-113)
__global__ void k_cg_init_r(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    DFL_PDL_ENTRY;
    if (st->done) return;
    const double bb = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    const double bn = sqrt(fmax(bb, 0.0));
    st->resnorm = bn;
    if (bn == 0.0 || bn <= st->target) {
        st->done = 1;
        st->converged = 1;
    } else if (st->maxiter <= 0) {
        st->done = 1;
    }
}

__global__ void k_cg_init_rz(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    DFL_PDL_ENTRY;
    if (st->done) return;
    const double rz = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x == 0) st->rz = rz;
}

// iters += 1; pAp (krylov.py:119-126); with use_if also the refresh IF condition
__global__ void k_cg_pq(KState *st, const double *part, int64_t nparts, const double *gath, int nranks,
                        int use_if, cudaGraphConditionalHandle hif) {
    DFL_PDL_ENTRY;
    if (st->done) return;
    const double pq = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    cg_step_pq(st, pq);
    if (use_if) cudaGraphSetConditional(hif, (!st->done && st->refresh_now) ? 1u : 0u);
}

// several ranks, deflated: pAp = sum_q (p.w)_q - t . t2 in rank / index order
// (the rank-local p.w sums ride in the last slot of every rank's Z'w slot)
__global__ void k_cg_pq_fold(KState *st, const double *tg, int nranks, int64_t slot, const double *t,
                             const double *t2, int64_t K) {
    DFL_PDL_ENTRY;
    if (st->done || threadIdx.x != 0) return;
    double pw = 0.0;
    for (int q = 0; q < nranks; ++q) pw += tg[(int64_t)q * slot + slot - 1];
    double tt = 0.0;
    for (int64_t j = 0; j < K; ++j) tt += t[j] * t2[j];
    cg_step_pq(st, pw - tt);
}

// resnorm test (krylov.py:132-136)
__global__ void k_cg_rr(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    DFL_PDL_ENTRY;
    if (st->done) return;
    const double rr = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    cg_step_rr(st, rr);
}

// beta (krylov.py:138-143)
__global__ void k_cg_rz(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    DFL_PDL_ENTRY;
    if (st->done) return;
    const double rz = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    cg_step_rz(st, rz);
}

// multi-rank: r.r and r.z arrive in one allgather (slots 0 and 1); the
// convergence test uses r.r exactly as k_cg_rr, then beta as k_cg_rz
__global__ void k_cg_rrz(KState *st, const double *gath, int nranks) {
    DFL_PDL_ENTRY;
    if (st->done || threadIdx.x != 0) return;
    double rr = 0.0, rz = 0.0;
    for (int q = 0; q < nranks; ++q) {
        rr += gath[q * 8 + 0];
        rz += gath[q * 8 + 1];
    }
    st->rr = rr;
    st->resnorm = sqrt(fmax(rr, 0.0));
    if (st->resnorm <= st->target) {
        st->converged = 1;
        st->done = 1;
        return;
    }
    if (rz == 0.0 || !isfinite(rz)) {
        st->breakdown = DFL_BRK_RZ;
        st->brk_val = rz;
        st->done = 1;
        return;
    }
    st->beta = rz / st->rz;
    st->rz = rz;
}

__global__ void k_cg_end(KState *st, cudaGraphConditionalHandle h, int use_cond) {
    DFL_PDL_ENTRY;
    if (threadIdx.x != 0) return;
    if (!st->done && st->iters >= st->maxiter) st->done = 1;
    if (use_cond) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

// ---------------------------------------------------------------------------
// one CG iteration (krylov.py:119-143) on the projected operator.
//
// Body: op (+Z'w partials), Z'w finish + E^-1, project (+p.q), alpha step,
// update (+r.r), convergence step, [refresh], V-cycle (+r.z), beta step,
// p update (+loop condition).  Single rank: with a graph the refresh of
// krylov.py:128-129 is a conditional IF node (no launches on the other 49 of
// 50 iterations).  Several ranks: partials are reduced, allgathered and
// consumed by single-block scalar kernels.
struct CgGraph {
    int use_cond = 0;
    cudaGraphConditionalHandle h = 0;
    int use_if = 0;  // refresh as an IF node
    cudaGraphConditionalHandle hif = 0;
};

// r = b' - project(A x)  (krylov.py:128-129); need_refresh: predicated on st->refresh_now
static int cg_refresh(dfl_ctx *ctx, bool deflated, int need_refresh) {
    KState *st = ctx->state;
    RC(op_apply_dev(ctx, ctx->x, ctx->tmp, 0, nullptr, deflated, st, need_refresh));
    if (deflated) RC(zt_to_t2(ctx, st, need_refresh, true));
    ProjArgs a = proj_args(ctx, ctx->tmp, ctx->r, st);
    if (!deflated) a.azd = nullptr, a.K = 0;
    a.base = ctx->bp;
    a.dotmode = 2;
    a.dot_part = ctx->dpart;
    a.need_refresh = need_refresh;
    launch_project<1>(ctx, a);
    return DFL_OK;
}

static int capture_refresh_if(dfl_ctx *ctx, bool deflated, cudaGraphConditionalHandle hif) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t capg = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(ctx->st, &cs, nullptr, &capg, &deps, &nd));
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hif;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t ifnode;
    CK(cudaGraphAddNode(&ifnode, capg, deps, nd, &ip));
    CK(cudaStreamUpdateCaptureDependencies(ctx->st, &ifnode, 1, cudaStreamSetCaptureDependencies));
    if (!ctx->st_if) CK(cudaStreamCreateWithFlags(&ctx->st_if, cudaStreamNonBlocking));
    cudaStream_t main = ctx->st;
    CK(cudaStreamBeginCaptureToGraph(ctx->st_if, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    ctx->st = ctx->st_if;
    const int64_t before = ctx->launches;
    const int rc = cg_refresh(ctx, deflated, 0);
    ctx->if_kernels = ctx->launches - before;  // run on refresh iterations only
    ctx->launches = before;
    ctx->st = main;
    cudaGraph_t g2 = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(ctx->st_if, &g2);
    RC(rc);
    CK(ce);
    return DFL_OK;
}

// refresh: -1 = decided on the device (IF node / predicated kernels), 0 / 1 =
// the caller knows whether this iteration refreshes (host-driven loops:
// iteration it refreshes iff (it + 1) % refresh_every == 0, krylov.py:128)
static int cg_body(dfl_ctx *ctx, bool deflated, const CgGraph &G, int refresh = -1) {
    KState *st = ctx->state;
    const double *gath;
    const bool single = !multi(ctx);
    // w = A p, Z'w -> t2 ; q = w - AZ t2 ; p.q
    RC(op_apply_dev(ctx, ctx->p, ctx->w, 0, nullptr, deflated, st, 0));
    if (!single && deflated) {
        // several ranks: p.q = p.w - t.E^-1 t (A symmetric: p'AZ t2 = (Z'Ap)'t2),
        // so the rank's p.w rides in the Z'w allgather and the iteration needs
        // two collectives besides the halo (Z'w + p.w, then r.r + r.z).  A
        // separate dot pass measured faster than a fifth value slot in the
        // operator kernel's epilogue (10.9 vs 11.2 ms, 1-rank NCCL, 150^3), and
        // as fast as a warp-sum epilogue next to the Z'y tree (10.02 vs 9.98 ms)
        launch_k(ctx->st, k_dot, (unsigned)ctx->vgrid, kBlock, 0, (const double *)ctx->p, (const double *)ctx->w,
                 ctx->n, ctx->dpart, (const KState *)st);
        ctx->launches++;
        RC(zt_to_t2(ctx, st, 0, true, ctx->dpart, ctx->vgrid, st));
        if (ctx->inexact) {  // t2 from the inner GMRES: fold after it
            const int64_t slot = (int64_t)ctx->max_nsub * ctx->k + 1;
            launch_k(ctx->st, k_cg_pq_fold, 1, 32, 0, st, (const double *)ctx->tgather, ctx->nranks, slot,
                     (const double *)ctx->tvec, (const double *)ctx->t2, ctx->K);
            ctx->launches++;
        }
        ProjArgs a = proj_args(ctx, ctx->w, ctx->w, st);
        launch_project<0>(ctx, a);
    } else {
        if (deflated) RC(zt_to_t2(ctx, st, 0, true));
        ProjArgs a = proj_args(ctx, ctx->w, ctx->w, st);
        if (!deflated) a.azd = nullptr, a.K = 0;
        a.dotmode = 1;
        a.dotv = ctx->p;
        a.dot_part = ctx->dpart;
        launch_project<0>(ctx, a);
        RC(rank_scalar(ctx, ctx->dpart, ctx->vgrid, 0, &gath));
        launch_k(ctx->st, k_cg_pq, 1, 1024, 0, st, ctx->dpart, ctx->vgrid, gath, ctx->nranks, G.use_if, G.hif);
        ctx->launches++;
    }
    // x += alpha p ; r -= alpha q (regular iterations); several ranks: the
    // update's last block also sums r.r into the allgather slot
    launch_k(ctx->st, k_cg_update, (unsigned)ctx->vgrid, kBlock, 0, ctx->x, ctx->r, ctx->p, ctx->w, ctx->n,
             ctx->dpart, (const KState *)st, single ? nullptr : ctx->scal + 0, ctx->ticket + 1);
    ctx->launches++;
    // refresh iterations: r = b' - project(A x)   (krylov.py:128-129)
    if (refresh == 0) {
    } else if (G.use_if) {
        RC(capture_refresh_if(ctx, deflated, G.hif));
    } else {
        RC(cg_refresh(ctx, deflated, 1));
    }
    int64_t np = 0;
    if (!single) {
        // one collective for r.r and r.z: the V-cycle runs before the
        // convergence test (its result is discarded on the last iteration)
        if (refresh != 0) {  // r.r of the refreshed residual (the update skipped its own)
            launch_k(ctx->st, k_reduce, 1, 1024, 0, ctx->dpart, ctx->vgrid, ctx->scal + 0);
            ctx->launches++;
        }
        RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
        launch_k(ctx->st, k_reduce, 1, 1024, 0, ctx->dpart, np, ctx->scal + 1);
        RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
        launch_k(ctx->st, k_cg_rrz, 1, 32, 0, st, ctx->sgather, ctx->nranks);
        ctx->launches += 2;
    } else {
        launch_k(ctx->st, k_cg_rr, 1, 1024, 0, st, ctx->dpart, ctx->vgrid, nullptr, 1);
        ctx->launches++;
        // z = M r, r.z -> beta
        RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
        launch_k(ctx->st, k_cg_rz, 1, 1024, 0, st, ctx->dpart, np, nullptr, 1);
        ctx->launches++;
    }
    launch_k(ctx->st, k_cg_p, (unsigned)ctx->vgrid, kBlock, 0, ctx->p, ctx->z, ctx->n, st, G.use_cond, G.h, G.use_if,
                                                       G.hif);
    ctx->launches++;
    if (!G.use_cond) {
        launch_k(ctx->st, k_cg_end, 1, 32, 0, st, 0, 0);
        ctx->launches++;
    }
    return DFL_OK;
}

// the CG body as plain graphs (several NCCL ranks: no conditional nodes),
// one without and one with the residual refresh
static int build_body_graph(dfl_ctx *ctx, bool deflated) {
    const int key = deflated ? 1 : 0;
    if (ctx->body_exec[0] && ctx->body_key == key) return DFL_OK;
    for (auto &e : ctx->body_exec)
        if (e) {
            cudaGraphExecDestroy(e);
            e = nullptr;
        }
    if (!ctx->h_state2) CK(cudaMallocHost(&ctx->h_state2, 2 * sizeof(KState)));
    for (int q = 0; q < 2; ++q)
        if (!ctx->ev_it[q]) CK(cudaEventCreateWithFlags(&ctx->ev_it[q], cudaEventDisableTiming));
    for (int refresh = 0; refresh < 2; ++refresh) {
        CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
        const int64_t before = ctx->launches;
        int rc = cg_body(ctx, deflated, CgGraph{}, refresh);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(ctx->st, &g);
        if (rc != DFL_OK) return rc;
        CK(ce);
        ctx->body_graph_kernels[refresh] = ctx->launches - before;
        ctx->launches = before;
        CK(cudaGraphInstantiate(&ctx->body_exec[refresh], g, 0));
        cudaGraphDestroy(g);
    }
    ctx->body_key = key;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// the whole solve on the device: b, x in ctx->b / ctx->xin
// x = 0, ||b||, b' = project(b), r, z = M r, p = z (krylov.py:101-117)
static int cg_prologue(dfl_ctx *ctx, const dfl_solve_params *p) {
    KState *st = ctx->state;
    const bool defl = p->deflated != 0;
    const double *gath;
    // x = 0 (y of the deflated system)
    launch_k(ctx->st, k_fill, (unsigned)ctx->nblk, kBlock, 0, ctx->x, 0.0, ctx->n);
    // ||b||
    launch_k(ctx->st, k_dot, (unsigned)ctx->vgrid, kBlock, 0, ctx->b, ctx->b, ctx->n, ctx->dpart, nullptr);
    ctx->launches += 2;
    RC(rank_scalar(ctx, ctx->dpart, ctx->vgrid, 0, &gath));
    launch_k(ctx->st, k_cg_start, 1, 1024, 0, st, ctx->dpart, ctx->vgrid, gath, ctx->nranks, p->tol, p->maxiter,
                                      std::max(1, p->refresh_every));
    ctx->launches++;
    // b' = project(b) and ||b'||^2
    // (without x0 the same kernel also writes r = b')
    const bool x0 = use_x0(ctx, p);
    if (defl) {
        RC(project_dev(ctx, ctx->b, ctx->bp, nullptr, 2, x0 ? nullptr : ctx->r));
    } else {
        ProjArgs a = proj_args(ctx, ctx->b, ctx->bp, nullptr);
        a.azd = nullptr;
        a.K = 0;
        a.dotmode = 2;
        a.dot_part = ctx->dpart;
        a.out2 = x0 ? nullptr : ctx->r;
        launch_project<0>(ctx, a);
    }
    if (x0) {  // x = x0 (unless b = 0), r = b - A x0 and ||r|| (krylov.py:108-109)
        launch_k(ctx->st, k_copy_live, (unsigned)ctx->nblk, kBlock, 0, ctx->x, (const double *)ctx->x0, ctx->n,
                 (const KState *)st);
        RC(op_apply_dev(ctx, ctx->x, ctx->r, 1, ctx->b, false, nullptr, 0));
        launch_k(ctx->st, k_dot, (unsigned)ctx->vgrid, kBlock, 0, (const double *)ctx->r, (const double *)ctx->r,
                 ctx->n, ctx->dpart, (const KState *)nullptr);
        ctx->launches += 2;
    }
    RC(rank_scalar(ctx, ctx->dpart, ctx->vgrid, 0, &gath));
    launch_k(ctx->st, k_cg_init_r, 1, 1024, 0, st, ctx->dpart, ctx->vgrid, gath, ctx->nranks);
    ctx->launches++;
    int64_t np = 0;
    RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
    RC(rank_scalar(ctx, ctx->dpart, np, 0, &gath));
    launch_k(ctx->st, k_cg_init_rz, 1, 1024, 0, st, ctx->dpart, np, gath, ctx->nranks);
    launch_k(ctx->st, k_copy, (unsigned)ctx->nblk, kBlock, 0, ctx->p, ctx->z, ctx->n);
    ctx->launches += 2;
    return DFL_OK;
}

// The whole single-rank solve as one CUDA graph: the prologue kernels, the
// while-conditional node with the CG body (refresh IF node inside), and the
// lift -- one launch per solve instead of ~45 host launches around the loop
// graph.  Cached per (deflated, x0, tol, maxiter, refresh): k_cg_start bakes
// them in.
static int build_solve_graph(dfl_ctx *ctx, const dfl_solve_params *p) {
    const bool defl = p->deflated != 0;
    char key[160];
    snprintf(key, sizeof key, "%d/%d/%.17g/%d/%d", (int)defl, (int)use_x0(ctx, p), p->tol, p->maxiter,
             std::max(1, p->refresh_every));
    if (ctx->solve_exec && ctx->solve_key == key) return DFL_OK;
    if (ctx->solve_exec) {
        cudaGraphExecDestroy(ctx->solve_exec);
        ctx->solve_exec = nullptr;
    }
    if (!ctx->st_body) CK(cudaStreamCreateWithFlags(&ctx->st_body, cudaStreamNonBlocking));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    CK(cudaStreamBeginCaptureToGraph(ctx->st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t before = ctx->launches;
    int rc = cg_prologue(ctx, p);
    cudaGraph_t body = nullptr;
    if (rc == DFL_OK) {
        cudaStreamCaptureStatus cs;
        cudaGraph_t capg = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        CK(cudaStreamGetCaptureInfo(ctx->st, &cs, nullptr, &capg, &deps, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wnode;
        CK(cudaGraphAddNode(&wnode, capg, deps, nd, &cp));
        CK(cudaStreamUpdateCaptureDependencies(ctx->st, &wnode, 1, cudaStreamSetCaptureDependencies));
        body = cp.conditional.phGraph_out[0];
        CgGraph G;
        G.use_cond = 1;
        G.h = h;
        const char *ni = getenv("DFL_NO_IF");
        G.use_if = !(ni && ni[0] == '1');
        if (G.use_if) CK(cudaGraphConditionalHandleCreate(&G.hif, body, 0, 0));
        CK(cudaStreamBeginCaptureToGraph(ctx->st_body, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        cudaStream_t main = ctx->st;
        ctx->st = ctx->st_body;
        const int64_t b0 = ctx->launches;
        rc = cg_body(ctx, defl, G);
        ctx->body_kernels = ctx->launches - b0;
        ctx->launches = b0;
        ctx->st = main;
        cudaGraph_t bg = nullptr;
        const cudaError_t be = cudaStreamEndCapture(ctx->st_body, &bg);
        if (rc == DFL_OK && be != cudaSuccess) rc = DFL_E_CUDA;
        if (rc == DFL_OK) rc = lift_dev(ctx, p);
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(ctx->st, &captured);
    ctx->solve_fixed_kernels = ctx->launches - before;
    ctx->launches = before;
    if (rc != DFL_OK) {
        cudaGraphDestroy(g);
        return rc;
    }
    CK(ce);
    CK(cudaGraphInstantiate(&ctx->solve_exec, g, 0));
    cudaGraphDestroy(g);
    ctx->solve_key = key;
    return DFL_OK;
}

int cg_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, bool use_graph) {
    KState *st = ctx->state;
    const bool defl = p->deflated != 0;
    if (use_graph) {
        RC(build_solve_graph(ctx, p));
        CK(cudaGraphLaunch(ctx->solve_exec, ctx->st));
        ctx->launches += ctx->solve_fixed_kernels;
        return DFL_OK;
    }
    RC(cg_prologue(ctx, p));
    // the loop
    if (ctx->comm && g_nccl_graph) {
        // NCCL ranks: the body (collectives included) captured once and replayed
        // per iteration; the host reads `done` one iteration late, so the GPU
        // always has the next iteration queued.  The extra iteration after the
        // last one skips its updates (KState.done) on every rank alike.
        RC(build_body_graph(ctx, defl));
        const int R = std::max(1, p->refresh_every);
        for (int it = 0;; ++it) {
            const int rf = (it + 1) % R == 0 ? 1 : 0;
            CK(cudaGraphLaunch(ctx->body_exec[rf], ctx->st));
            ctx->launches += ctx->body_graph_kernels[rf];
            CK(cudaMemcpyAsync(ctx->h_state2 + (it & 1), st, sizeof(KState), cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaEventRecord(ctx->ev_it[it & 1], ctx->st));
            if (it > 0) {
                RC(comm_wait_event(ctx, ctx->ev_it[(it - 1) & 1]));
                if (ctx->h_state2[(it - 1) & 1].done) break;
            }
        }
    } else {
        // several ranks: host-driven, but the host reads `done` one iteration
        // late, so iteration it+1 (kernels and collectives) is already queued
        // while it waits for iteration it -- no idle GPU between iterations.
        // The speculative iteration after the last skips its updates
        // (KState.done) on every rank alike, and its collectives run on every
        // rank, so all ranks issue the same collective sequence.
        if (!ctx->h_state2) CK(cudaMallocHost(&ctx->h_state2, 2 * sizeof(KState)));
        for (int q = 0; q < 2; ++q)
            if (!ctx->ev_it[q]) CK(cudaEventCreateWithFlags(&ctx->ev_it[q], cudaEventDisableTiming));
        const int R = std::max(1, p->refresh_every);
        for (int it = 0;; ++it) {
            RC(cg_body(ctx, defl, CgGraph{}, (it + 1) % R == 0 ? 1 : 0));
            CK(cudaMemcpyAsync(ctx->h_state2 + (it & 1), st, sizeof(KState), cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaEventRecord(ctx->ev_it[it & 1], ctx->st));
            if (it > 0) {
                RC(comm_wait_event(ctx, ctx->ev_it[(it - 1) & 1]));
                if (ctx->h_state2[(it - 1) & 1].done) break;
            }
        }
    }
    return lift_dev(ctx, p);
}

