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
    if (st->done) return;
    const double rz = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x == 0) st->rz = rz;
}

// iters += 1; pAp (krylov.py:119-126)
__global__ void k_cg_pq(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double pq = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    st->iters += 1;
    st->pq = pq;
    if (pq <= 0.0 || !isfinite(pq)) {
        st->breakdown = DFL_BRK_CURVATURE;
        st->done = 1;
        return;
    }
    st->alpha = st->rz / pq;
    st->refresh_now = (st->iters % st->refresh_every) == 0;
}

// resnorm test (krylov.py:132-136)
__global__ void k_cg_rr(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double rr = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    st->rr = rr;
    st->resnorm = sqrt(fmax(rr, 0.0));
    if (st->resnorm <= st->target) {
        st->converged = 1;
        st->done = 1;
    }
}

// beta (krylov.py:138-143)
__global__ void k_cg_rz(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double rz = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    if (rz == 0.0 || !isfinite(rz)) {
        st->breakdown = DFL_BRK_RZ;
        st->done = 1;
        return;
    }
    st->beta = rz / st->rz;
    st->rz = rz;
}

// multi-rank: r.r and r.z arrive in one allgather (slots 0 and 1); the
// convergence test uses r.r exactly as k_cg_rr, then beta as k_cg_rz
__global__ void k_cg_rrz(KState *st, const double *gath, int nranks) {
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
        st->done = 1;
        return;
    }
    st->beta = rz / st->rz;
    st->rz = rz;
}

__global__ void k_cg_end(KState *st, cudaGraphConditionalHandle h, int use_cond) {
    if (threadIdx.x != 0) return;
    if (!st->done && st->iters >= st->maxiter) st->done = 1;
    if (use_cond) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

// ---------------------------------------------------------------------------
// one CG iteration (krylov.py:119-143) on the projected operator
static int cg_body(dfl_ctx *ctx, bool deflated, cudaGraphConditionalHandle h, int use_cond) {
    KState *st = ctx->state;
    const double *gath;
    // w = A p, Z'w ; t2 ; q = w - AZ t2 ; p.q
    RC(op_apply_dev(ctx, ctx->p, ctx->w, 0, nullptr, deflated, st, 0));
    if (deflated) RC(zt_to_t2(ctx, st, 0, true));
    {
        ProjArgs a = proj_args(ctx, ctx->w, ctx->w, st);
        if (!deflated) a.az_ptr = nullptr, a.K = 0;
        a.dotmode = 1;
        a.dotv = ctx->p;
        a.dot_part = ctx->dpart;
        launch_project<0>(ctx, a);
    }
    RC(rank_scalar(ctx, ctx->dpart, ctx->nblk, 0, &gath));
    k_cg_pq<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, gath, ctx->nranks);
    ctx->launches++;
    // x += alpha p ; r -= alpha q (regular iterations)
    k_cg_update<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->x, ctx->r, ctx->p, ctx->w, ctx->n, ctx->dpart, st);
    ctx->launches++;
    // refresh iterations: r = b' - project(A x)   (krylov.py:128-129)
    RC(op_apply_dev(ctx, ctx->x, ctx->tmp, 0, nullptr, deflated, st, 1));
    if (deflated) RC(zt_to_t2(ctx, st, 1, true));
    {
        ProjArgs a = proj_args(ctx, ctx->tmp, ctx->r, st);
        if (!deflated) a.az_ptr = nullptr, a.K = 0;
        a.base = ctx->bp;
        a.dotmode = 2;
        a.dot_part = ctx->dpart;
        a.need_refresh = 1;
        launch_project<1>(ctx, a);
    }
    int64_t np = 0;
    if (multi(ctx)) {
        // one collective for r.r and r.z: the V-cycle runs before the
        // convergence test (its result is discarded on the last iteration)
        k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->dpart, ctx->nblk, ctx->scal + 0);
        RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
        k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->dpart, np, ctx->scal + 1);
        RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
        k_cg_rrz<<<1, 32, 0, ctx->st>>>(st, ctx->sgather, ctx->nranks);
        ctx->launches += 3;
    } else {
        k_cg_rr<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, nullptr, 1);
        ctx->launches++;
        // z = M r, r.z
        RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
        k_cg_rz<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, np, nullptr, 1);
        ctx->launches++;
    }
    k_cg_p<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->p, ctx->z, ctx->n, st);
    ctx->launches++;
    k_cg_end<<<1, 32, 0, ctx->st>>>(st, h, use_cond);
    ctx->launches++;
    return DFL_OK;
}

static int build_loop_graph(dfl_ctx *ctx, bool deflated) {
    const int key = deflated ? 1 : 0;
    if (ctx->loop_exec && ctx->loop_key == key) return DFL_OK;
    if (ctx->loop_exec) {
        cudaGraphExecDestroy(ctx->loop_exec);
        ctx->loop_exec = nullptr;
    }
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(ctx->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t before = ctx->launches;
    int rc = cg_body(ctx, deflated, h, 1);
    cudaGraph_t captured = nullptr;
    cudaError_t ce = cudaStreamEndCapture(ctx->st, &captured);
    if (rc != DFL_OK) return rc;
    CK(ce);
    ctx->body_kernels = ctx->launches - before;
    ctx->launches = before;
    CK(cudaGraphInstantiate(&ctx->loop_exec, g, 0));
    cudaGraphDestroy(g);
    ctx->loop_key = key;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// the whole solve on the device: b, x in ctx->b / ctx->xin
int cg_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, bool use_graph) {
    KState *st = ctx->state;
    const bool defl = p->deflated != 0;
    const double *gath;
    // x = 0 (y of the deflated system)
    k_fill<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->x, 0.0, ctx->n);
    // ||b||
    k_dot<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->b, ctx->b, ctx->n, ctx->dpart, nullptr);
    ctx->launches += 2;
    RC(rank_scalar(ctx, ctx->dpart, ctx->nblk, 0, &gath));
    k_cg_start<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, gath, ctx->nranks, p->tol, p->maxiter,
                                      std::max(1, p->refresh_every));
    ctx->launches++;
    // b' = project(b) and ||b'||^2
    if (defl) {
        RC(project_dev(ctx, ctx->b, ctx->bp, nullptr, 2));
    } else {
        ProjArgs a = proj_args(ctx, ctx->b, ctx->bp, nullptr);
        a.az_ptr = nullptr;
        a.K = 0;
        a.dotmode = 2;
        a.dot_part = ctx->dpart;
        launch_project<0>(ctx, a);
    }
    RC(rank_scalar(ctx, ctx->dpart, ctx->nblk, 0, &gath));
    k_cg_init_r<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, gath, ctx->nranks);
    k_copy<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->r, ctx->bp, ctx->n);
    ctx->launches += 2;
    int64_t np = 0;
    RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
    RC(rank_scalar(ctx, ctx->dpart, np, 0, &gath));
    k_cg_init_rz<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, np, gath, ctx->nranks);
    k_copy<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->p, ctx->z, ctx->n);
    ctx->launches += 2;
    // the loop
    if (use_graph) {
        RC(build_loop_graph(ctx, defl));
        CK(cudaGraphLaunch(ctx->loop_exec, ctx->st));
    } else {
        for (;;) {
            RC(cg_body(ctx, defl, 0, 0));
            CK(cudaMemcpyAsync(ctx->h_state, st, sizeof(KState), cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            if (ctx->h_state->done) break;
        }
    }
    return lift_dev(ctx, p);
}

