// BiCGStab(2) with the whole iteration on the device (single rank): one CUDA
// graph whose body is one L-group of krylov.py:148-285, inside a
// while-conditional node.  Every scalar of the reference's recurrence lives in
// a device BState and is computed by a single-block kernel with the
// reference's expressions and breakdown tests; the nine data-dependent exits
// (restart-once, mid-group convergence, the MR / omega breakdowns) become
// flags the vector kernels test (ks.done: "the rest of this group is
// skipped", fin: "the loop is over").  The true-residual refresh every 50
// groups is an IF-conditional node.  Several ranks keep the host-driven loop
// of ctx_krylov.cu (its collectives meet at host barriers in the tests).
#include "ctx_impl.cuh"

namespace {

enum { BD_RHO = 0, BD_ALL = 1, BD_ABORTED = 2 };

// ks.done doubles as the group-skip flag read by the shared kernels
// (k_project, k_zt_finish, ...); ks.refresh_now drives the refresh IF node.
struct BState {
    KState ks;
    double rho0, alpha, omega, beta, rho_next, resnorm, target;
    double gp1, tau12, gp2, g1, g2, gpp1, mr0, mr1, mr2;
    int iters, maxiter, fin, brk, restarted, rho_valid, aborted, restart_pending, refresh;
};

// the reference's fail(): restart once (r_shadow = r0, d0 = 0 -- applied by
// k_bg_restart at the start of the next group; rho0, alpha, omega = 1, 0, 1),
// a second breakdown ends the solve with its code (krylov.py:165-175)
__device__ void bg_fail(BState *b, int code) {
    b->rho_valid = 0;
    b->ks.done = 1;
    if (b->restarted) {
        b->brk = code;
        b->fin = 1;
        return;
    }
    b->restarted = 1;
    b->restart_pending = 1;
    b->rho0 = 1.0;
    b->alpha = 0.0;
    b->omega = 1.0;
}

// deterministic sums of nq strided partials (stride kDotStride), valid in all threads
__device__ void bg_reduce(const double *part, int64_t nparts, int nq, double *out) {
    __shared__ double sm[32 * 4];
    __shared__ double res[4];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t j = threadIdx.x; j < nparts; j += blockDim.x)
        for (int q = 0; q < nq; ++q) acc[q] += part[j * kDotStride + q];
    block_sum<4>(acc, sm);
    if (threadIdx.x == 0)
        for (int q = 0; q < 4; ++q) res[q] = acc[q];
    __syncthreads();
    for (int q = 0; q < nq; ++q) out[q] = res[q];
}

__global__ void k_bg_init(BState *b, double target, double bpn, double bpbp, int maxiter, int refresh) {
    DFL_PDL_ENTRY;
    BState s{};
    s.rho0 = 1.0;
    s.alpha = 0.0;
    s.omega = 1.0;
    s.resnorm = bpn;
    s.rho_next = bpbp;  // r[0].shadow of the first step (both are b')
    s.rho_valid = 1;
    s.target = target;
    s.maxiter = maxiter;
    s.refresh = refresh;
    s.fin = !(0 < maxiter && bpn > target);
    s.ks.done = s.fin;
    *b = s;
}

// r_shadow = r0, d0 = 0 after a breakdown-restart (next group's start)
__global__ void __launch_bounds__(kBlock) k_bg_restart(const BState *b, double *shadow, const double *r0, double *d0,
                                                       int64_t n) {
    DFL_PDL_ENTRY;
    if (!b->restart_pending) return;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        shadow[i] = r0[i];
        d0[i] = 0.0;
    }
}

__global__ void k_bg_begin(BState *b) {
    DFL_PDL_ENTRY;
    b->restart_pending = 0;
    if (b->fin) {
        b->ks.done = 1;
        return;
    }
    b->iters += 1;
    b->rho0 = -b->omega * b->rho0;
    b->aborted = 0;
    b->ks.done = 0;
    b->ks.refresh_now = 0;
}

// up to four dot products, per-block partials at stride kDotStride
__global__ void __launch_bounds__(kBlock) k_bg_dots(const BState *b, int mode, const double *__restrict__ a0,
                                                    const double *__restrict__ b0, const double *__restrict__ a1,
                                                    const double *__restrict__ b1, const double *__restrict__ a2,
                                                    const double *__restrict__ b2, const double *__restrict__ a3,
                                                    const double *__restrict__ b3, int nq, int64_t n, double *part) {
    DFL_PDL_ENTRY;
    if (mode == BD_RHO && (b->ks.done || b->rho_valid)) return;
    if (mode == BD_ALL && b->ks.done) return;
    if (mode == BD_ABORTED && !b->aborted) return;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        acc[0] += a0[i] * b0[i];
        if (nq > 1) acc[1] += a1[i] * b1[i];
        if (nq > 2) acc[2] += a2[i] * b2[i];
        if (nq > 3) acc[3] += a3[i] * b3[i];
    }
    __shared__ double sm[32 * 4];
    block_sum<4>(acc, sm);
    if (threadIdx.x == 0)
        for (int q = 0; q < 4; ++q) part[blockIdx.x * kDotStride + q] = acc[q];
}

// rho1 (r[j].shadow) and beta (krylov.py:177-190)
__global__ void k_bg_s1(BState *b, const double *part, int64_t np) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    double v[1] = {0.0};
    const bool need = !b->rho_valid;
    if (need) bg_reduce(part, np, 1, v);
    if (threadIdx.x != 0) return;
    const double rho1 = need ? v[0] : b->rho_next;
    b->rho_valid = 0;
    if (b->rho0 == 0.0 || !isfinite(rho1)) {
        bg_fail(b, DFL_BRK_RHO);
        b->aborted = 1;
        return;
    }
    b->beta = b->alpha * rho1 / b->rho0;
    b->rho0 = rho1;
}

// gamma = op_hat(d_j).shadow, alpha (krylov.py:191-196); part: one partial per block
__global__ void k_bg_s2(BState *b, const double *part, int64_t np) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    const double gd = reduce_parts(part, np);
    if (threadIdx.x != 0) return;
    if (gd == 0.0 || !isfinite(gd)) {
        bg_fail(b, DFL_BRK_SHADOW);
        b->aborted = 1;
        return;
    }
    b->alpha = b->rho0 / gd;
}

// ||r0|| (+ the next rho1 for j = 0, + the minimal-residual dots for j = 1);
// mid-group convergence (krylov.py:203-206, 212-215)
__global__ void k_bg_s3(BState *b, const double *part, int64_t np, int j) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    double v[4];
    bg_reduce(part, np, j == 0 ? 2 : 4, v);
    if (threadIdx.x != 0) return;
    b->resnorm = sqrt(fmax(v[0], 0.0));
    if (j == 0) {
        b->rho_next = v[1];
        b->rho_valid = 1;
    } else {
        b->mr0 = v[1];
        b->mr1 = v[2];
        b->mr2 = v[3];
    }
    if (b->resnorm <= b->target) {
        b->ks.done = 1;
        b->fin = 1;
    }
}

// after an aborted BiCG part: ||r0||, then break or continue with the next group
__global__ void k_bg_after(BState *b, const double *part, int64_t np) {
    DFL_PDL_ENTRY;
    if (!b->aborted) return;
    double v[1];
    bg_reduce(part, np, 1, v);
    if (threadIdx.x != 0) return;
    b->resnorm = sqrt(fmax(v[0], 0.0));
    if (b->brk != DFL_BRK_NONE || b->resnorm <= b->target) b->fin = 1;
}

// minimal-residual step, first half (krylov.py:207-236)
__global__ void k_bg_mr1(BState *b) {
    DFL_PDL_ENTRY;
    if (b->ks.done || threadIdx.x != 0) return;
    const double sigma1 = b->mr1;
    if (sigma1 == 0.0 || !isfinite(sigma1)) {
        bg_fail(b, DFL_BRK_MR);
        return;
    }
    b->gp1 = b->mr0 / sigma1;
    b->tau12 = b->mr2 / sigma1;
}

// r2 -= tau12 r1, partials of (r2.r2, r0.r2)
__global__ void __launch_bounds__(kBlock) k_bg_mr2(const BState *b, double *r2, const double *__restrict__ r1,
                                                   const double *__restrict__ r0, int64_t n, double *part) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    const double tau12 = b->tau12;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double v = sub_rn(r2[i], mul_rn(tau12, r1[i]));
        r2[i] = v;
        acc[0] += v * v;
        acc[1] += r0[i] * v;
    }
    __shared__ double sm[32 * 4];
    block_sum<4>(acc, sm);
    if (threadIdx.x == 0)
        for (int q = 0; q < 4; ++q) part[blockIdx.x * kDotStride + q] = acc[q];
}

// sigma2, gamma'_2 = omega, gamma_1, gamma''_1 (krylov.py:237-250); refresh decision
__global__ void k_bg_mr3(BState *b, const double *part, int64_t np, int use_if, cudaGraphConditionalHandle hif) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    double v[2];
    bg_reduce(part, np, 2, v);
    if (threadIdx.x != 0) return;
    const double sigma2 = v[0];
    if (sigma2 == 0.0 || !isfinite(sigma2)) {
        bg_fail(b, DFL_BRK_MR);
        return;
    }
    const double gp2 = v[1] / sigma2;
    const double g2 = gp2;
    b->omega = g2;
    if (b->omega == 0.0 || !isfinite(b->omega)) {
        bg_fail(b, DFL_BRK_OMEGA);
        return;
    }
    b->gp2 = gp2;
    b->g2 = g2;
    b->g1 = b->gp1 - b->tau12 * g2;
    b->gpp1 = g2 + 0.0;
    b->ks.refresh_now = (b->iters % b->refresh) == 0;
    if (use_if) cudaGraphSetConditional(hif, b->ks.refresh_now ? 1u : 0u);
}

// the group's vector updates (krylov.py:251-255)
__global__ void __launch_bounds__(kBlock) k_bg_final(const BState *b, double *u, double *r0, double *d0,
                                                     const double *__restrict__ r1, const double *__restrict__ r2,
                                                     const double *__restrict__ d1, const double *__restrict__ d2,
                                                     int64_t n) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    const double g1 = b->g1, gp2 = b->gp2, g2 = b->g2, gpp1 = b->gpp1, gp1 = b->gp1;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double r0i = r0[i], r1i = r1[i];
        double ui = add_rn(u[i], mul_rn(g1, r0i));
        double ri = sub_rn(r0i, mul_rn(gp2, r2[i]));
        double di = sub_rn(d0[i], mul_rn(g2, d2[i]));
        di = sub_rn(di, mul_rn(g1, d1[i]));
        ui = add_rn(ui, mul_rn(gpp1, r1i));
        ri = sub_rn(ri, mul_rn(gp1, r1i));
        u[i] = ui;
        r0[i] = ri;
        d0[i] = di;
    }
}

// d_k = r_k - beta d_k, k <= j  (krylov.py:189-190)
__global__ void __launch_bounds__(kBlock) k_bg_d(const BState *b, const double *__restrict__ r0, double *d0,
                                                 const double *__restrict__ r1, double *d1, int cnt, int64_t n) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    const double beta = b->beta;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        d0[i] = sub_rn(r0[i], mul_rn(beta, d0[i]));
        if (cnt > 1) d1[i] = sub_rn(r1[i], mul_rn(beta, d1[i]));
    }
}

// r_k -= alpha d_{k+1}, k <= j; u += alpha d0  (krylov.py:197-200)
__global__ void __launch_bounds__(kBlock) k_bg_r(const BState *b, double *r0, const double *__restrict__ d1,
                                                 double *r1, const double *__restrict__ d2, int cnt, double *u,
                                                 const double *__restrict__ d0, int64_t n) {
    DFL_PDL_ENTRY;
    if (b->ks.done) return;
    const double alpha = b->alpha;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        r0[i] = sub_rn(r0[i], mul_rn(alpha, d1[i]));
        if (cnt > 1) r1[i] = sub_rn(r1[i], mul_rn(alpha, d2[i]));
        u[i] = add_rn(u[i], mul_rn(alpha, d0[i]));
    }
}

// ||r0||, the next group's rho1 = r0.shadow; the loop condition (krylov.py:164)
__global__ void k_bg_end(BState *b, const double *part, int64_t np, cudaGraphConditionalHandle h, int use_if,
                         cudaGraphConditionalHandle hif) {
    DFL_PDL_ENTRY;
    const bool upd = !b->ks.done;
    double v[2] = {0.0, 0.0};
    if (upd) bg_reduce(part, np, 2, v);
    if (threadIdx.x != 0) return;
    if (upd) {
        b->resnorm = sqrt(fmax(v[0], 0.0));
        b->rho_next = v[1];
        b->rho_valid = 1;
    }
    if (!b->fin && !(b->iters < b->maxiter && b->resnorm > b->target)) b->fin = 1;
    cudaGraphSetConditional(h, b->fin ? 0u : 1u);
    if (use_if) cudaGraphSetConditional(hif, 0u);
}

}  // namespace

// ---------------------------------------------------------------------------

static unsigned bg_dot_grid(dfl_ctx *ctx) {
    return (unsigned)std::min<int64_t>(std::max<int64_t>(1, ctx->nblk), 4 * ctx->sm_count);
}

// out = op_hat(v) = project(A (M v)); with dotv: per-block partials of out.dotv in dpart (vgrid)
static int bg_op_hat(dfl_ctx *ctx, bool defl, KState *ks, const double *v, double *out, const double *dotv) {
    RC(vcycle(ctx, v, ctx->zx, ks, nullptr, nullptr));
    RC(op_apply_dev(ctx, ctx->zx, ctx->w, 0, nullptr, defl, ks, 0));
    if (defl) RC(zt_to_t2(ctx, ks, 0, true));
    ProjArgs a = proj_args(ctx, ctx->w, out, ks);
    if (!defl) a.azd = nullptr, a.K = 0;
    if (dotv) {
        a.dotmode = 1;
        a.dotv = dotv;
        a.dot_part = ctx->dpart;
    }
    launch_project<0>(ctx, a);
    return DFL_OK;
}

struct BgGraph {
    cudaGraphConditionalHandle h = 0, hif = 0;
    int use_if = 0;
};

static int bg_body(dfl_ctx *ctx, bool defl, BState *b, const BgGraph &G) {
    const int64_t n = ctx->n;
    const unsigned g = bg_dot_grid(ctx), vg = (unsigned)ctx->vgrid;
    double *r[3] = {ctx->br[0], ctx->br[1], ctx->br[2]};
    double *d[3] = {ctx->bd[0], ctx->bd[1], ctx->bd[2]};
    double *u = ctx->bu, *shadow = ctx->bshadow, *part = ctx->dpart;
    const double *nul = nullptr;
    KState *ks = &b->ks;
    launch_k(ctx->st, k_bg_restart, vg, kBlock, 0, (const BState *)b, shadow, (const double *)r[0], d[0], n);
    launch_k(ctx->st, k_bg_begin, 1, 1, 0, b);
    ctx->launches += 2;
    for (int j = 0; j < 2; ++j) {
        launch_k(ctx->st, k_bg_dots, g, kBlock, 0, (const BState *)b, (int)BD_RHO, (const double *)r[j],
                 (const double *)shadow, nul, nul, nul, nul, nul, nul, 1, n, part);
        launch_k(ctx->st, k_bg_s1, 1, 1024, 0, b, (const double *)part, (int64_t)g);
        launch_k(ctx->st, k_bg_d, vg, kBlock, 0, (const BState *)b, (const double *)r[0], d[0], (const double *)r[1],
                 d[1], j + 1, n);
        ctx->launches += 3;
        RC(bg_op_hat(ctx, defl, ks, d[j], d[j + 1], shadow));
        launch_k(ctx->st, k_bg_s2, 1, 1024, 0, b, (const double *)part, (int64_t)ctx->vgrid);
        launch_k(ctx->st, k_bg_r, vg, kBlock, 0, (const BState *)b, r[0], (const double *)d[1], r[1],
                 (const double *)d[2], j + 1, u, (const double *)d[0], n);
        ctx->launches += 2;
        RC(bg_op_hat(ctx, defl, ks, r[j], r[j + 1], nullptr));
        if (j == 0)
            launch_k(ctx->st, k_bg_dots, g, kBlock, 0, (const BState *)b, (int)BD_ALL, (const double *)r[0],
                     (const double *)r[0], (const double *)r[1], (const double *)shadow, nul, nul, nul, nul, 2, n, part);
        else
            launch_k(ctx->st, k_bg_dots, g, kBlock, 0, (const BState *)b, (int)BD_ALL, (const double *)r[0],
                     (const double *)r[0], (const double *)r[0], (const double *)r[1], (const double *)r[1],
                     (const double *)r[1], (const double *)r[2], (const double *)r[1], 4, n, part);
        launch_k(ctx->st, k_bg_s3, 1, 1024, 0, b, (const double *)part, (int64_t)g, j);
        ctx->launches += 2;
    }
    launch_k(ctx->st, k_bg_dots, g, kBlock, 0, (const BState *)b, (int)BD_ABORTED, (const double *)r[0],
             (const double *)r[0], nul, nul, nul, nul, nul, nul, 1, n, part);
    launch_k(ctx->st, k_bg_after, 1, 1024, 0, b, (const double *)part, (int64_t)g);
    launch_k(ctx->st, k_bg_mr1, 1, 32, 0, b);
    launch_k(ctx->st, k_bg_mr2, g, kBlock, 0, (const BState *)b, r[2], (const double *)r[1], (const double *)r[0], n,
             part);
    launch_k(ctx->st, k_bg_mr3, 1, 1024, 0, b, (const double *)part, (int64_t)g, G.use_if, G.hif);
    launch_k(ctx->st, k_bg_final, vg, kBlock, 0, (const BState *)b, u, r[0], d[0], (const double *)r[1],
             (const double *)r[2], (const double *)d[1], (const double *)d[2], n);
    ctx->launches += 6;
    // refresh: r0 = r0_init - op_hat(u)   (krylov.py:256-257), an IF node
    {
        cudaStreamCaptureStatus cs;
        cudaGraph_t capg = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        CK(cudaStreamGetCaptureInfo(ctx->st, &cs, nullptr, &capg, &deps, &nd));
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = G.hif;
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
        int rc = bg_op_hat(ctx, defl, ks, u, ctx->tmp, nullptr);
        if (rc == DFL_OK) {
            ProjArgs a = proj_args(ctx, ctx->tmp, r[0], ks);
            a.azd = nullptr;
            a.K = 0;
            a.base = ctx->bp;
            launch_project<1>(ctx, a);  // r0 = r0_init - tmp
        }
        ctx->st = main;
        cudaGraph_t g2 = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(ctx->st_if, &g2);
        RC(rc);
        CK(ce);
    }
    launch_k(ctx->st, k_bg_dots, g, kBlock, 0, (const BState *)b, (int)BD_ALL, (const double *)r[0],
             (const double *)r[0], (const double *)r[0], (const double *)shadow, nul, nul, nul, nul, 2, n, part);
    launch_k(ctx->st, k_bg_end, 1, 1024, 0, b, (const double *)part, (int64_t)g, G.h, G.use_if, G.hif);
    ctx->launches += 2;
    return DFL_OK;
}

static int bg_graph(dfl_ctx *ctx, bool defl, BState *b) {
    const int key = 10 + (defl ? 1 : 0);
    if (ctx->bg_exec && ctx->bg_key == key) return DFL_OK;
    if (ctx->bg_exec) {
        cudaGraphExecDestroy(ctx->bg_exec);
        ctx->bg_exec = nullptr;
    }
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    BgGraph G;
    CK(cudaGraphConditionalHandleCreate(&G.h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = G.h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    G.use_if = 1;
    CK(cudaGraphConditionalHandleCreate(&G.hif, body, 0, 0));
    CK(cudaStreamBeginCaptureToGraph(ctx->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t before = ctx->launches;
    int rc = bg_body(ctx, defl, b, G);
    cudaGraph_t captured = nullptr;
    cudaError_t ce = cudaStreamEndCapture(ctx->st, &captured);
    if (rc != DFL_OK) return rc;
    CK(ce);
    ctx->bg_body_kernels = ctx->launches - before;
    ctx->launches = before;
    CK(cudaGraphInstantiate(&ctx->bg_exec, g, 0));
    cudaGraphDestroy(g);
    ctx->bg_key = key;
    return DFL_OK;
}

// BiCGStab(2) with the group loop on the device.  The prologue (||b||, b',
// ||b'||) reads two norms back to the host, as the host-driven version does.
int bicg_solve_graph(dfl_ctx *ctx, const dfl_solve_params *p, KState &out) {
    RC(bicg_prologue(ctx, p, out));
    if (out.converged) return DFL_OK;  // b = 0 or b' = 0: x = 0 already
    if (!ctx->bstate) {
        void *q = nullptr;
        CK(cudaMalloc(&q, sizeof(BState)));
        ctx->allocs.push_back(q);
        ctx->bstate = q;
        CK(cudaMallocHost(&ctx->h_bstate, sizeof(BState)));
    }
    BState *b = static_cast<BState *>(ctx->bstate);
    const bool defl = p->deflated != 0;
    launch_k(ctx->st, k_bg_init, 1, 1, 0, b, out.target, out.resnorm, out.rho1, p->maxiter,
             std::max(1, p->refresh_every));
    ctx->launches++;
    RC(bg_graph(ctx, defl, b));
    CK(cudaGraphLaunch(ctx->bg_exec, ctx->st));
    CK(cudaMemcpyAsync(ctx->h_bstate, b, sizeof(BState), cudaMemcpyDeviceToHost, ctx->st));
    RC(comm_wait(ctx, ctx->st));
    const BState &s = *static_cast<const BState *>(ctx->h_bstate);
    ctx->launches += ctx->bg_body_kernels * std::max(1, s.iters);
    // x = x0 + M(u)  (krylov.py:284-285), into ctx->x (the y of the deflated system)
    RC(vcycle(ctx, ctx->bu, ctx->x, nullptr, nullptr, nullptr));
    if (use_x0(ctx, p)) {
        launch_k(ctx->st, k_addv, (unsigned)ctx->nblk, kBlock, 0, ctx->x, (const double *)ctx->x0, ctx->n);
        ctx->launches++;
    }
    out.iters = s.iters;
    out.resnorm = s.resnorm;
    out.converged = s.resnorm <= out.target;
    out.breakdown = out.converged ? DFL_BRK_NONE : s.brk;
    return DFL_OK;
}
