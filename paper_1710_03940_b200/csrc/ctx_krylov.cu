// BiCGStab(2) and (F)GMRES on the device, host-driven with device reductions.
#include "ctx_impl.cuh"

// ---------------------------------------------------------------------------
// BiCGStab(2) (krylov.py:148-285), right preconditioned: op_hat = op o M with
// op = project o A.  Host-driven: scalars are computed on the host in IEEE
// double with the reference's expressions; every dot is a device reduction
// read back at its branch point.

static int fetch(dfl_ctx *ctx, const double *dev, int n, double *out) {
    CK(cudaMemcpyAsync(ctx->h_dots, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->st));
    RC(comm_wait(ctx, ctx->st));
    for (int q = 0; q < n; ++q) out[q] = ctx->h_dots[q];
    return DFL_OK;
}

// global value of nq interleaved (stride 3) or plain (nq == 0 -> 1 stream) partials
static int global_dots(dfl_ctx *ctx, const double *part, int64_t nparts, int nq, bool strided, double *out) {
    if (strided)
        launch_k(ctx->st, k_reduceq, 1, 1024, 0, part, nparts, nq, ctx->scal);
    else
        launch_k(ctx->st, k_reduce, 1, 1024, 0, part, nparts, ctx->scal);
    ctx->launches++;
    if (multi(ctx)) {
        RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
        launch_k(ctx->st, k_rank_sum, 1, 32, 0, ctx->sgather, ctx->nranks, 8, nq, ctx->scal + 8);
        ctx->launches++;
        return fetch(ctx, ctx->scal + 8, nq, out);
    }
    return fetch(ctx, ctx->scal, nq, out);
}

static unsigned dot_grid(dfl_ctx *ctx) { return (unsigned)std::min<int64_t>(std::max<int64_t>(1, ctx->nblk), 4 * ctx->sm_count); }

static int dots(dfl_ctx *ctx, int nq, const double *a0, const double *b0, const double *a1, const double *b1,
                const double *a2, const double *b2, double *out, const double *a3 = nullptr,
                const double *b3 = nullptr) {
    const unsigned g = dot_grid(ctx);
    launch_k(ctx->st, k_multidot, g, kBlock, 0, a0, b0, a1, b1, a2, b2, a3, b3, nq, ctx->n, ctx->dpart);
    ctx->launches++;
    return global_dots(ctx, ctx->dpart, g, nq, true, out);
}

// out = op_hat(v) = project(A (M v)); with dotv: also returns dot(out, dotv)
static int op_hat(dfl_ctx *ctx, bool defl, const double *v, double *out, const double *dotv, double *dot_out) {
    RC(vcycle(ctx, v, ctx->zx, nullptr, nullptr, nullptr));
    RC(op_apply_dev(ctx, ctx->zx, ctx->w, 0, nullptr, defl, nullptr, 0));
    if (defl) RC(zt_to_t2(ctx, nullptr, 0, true));
    ProjArgs a = proj_args(ctx, ctx->w, out, nullptr);
    if (!defl) a.azd = nullptr, a.K = 0;
    if (dotv) {
        a.dotmode = 1;
        a.dotv = dotv;
        a.dot_part = ctx->dpart;
    }
    launch_project<0>(ctx, a);
    if (dotv) RC(global_dots(ctx, ctx->dpart, ctx->vgrid, 1, false, dot_out));
    return DFL_OK;
}

static int bicg_alloc(dfl_ctx *ctx) {
    if (ctx->bu) return DFL_OK;
    for (int j = 0; j < 3; ++j) {
        RC(dalloc(ctx, &ctx->br[j], ctx->n));
        RC(dalloc(ctx, &ctx->bd[j], ctx->n));
    }
    RC(dalloc(ctx, &ctx->bu, ctx->n));
    RC(dalloc(ctx, &ctx->bshadow, ctx->n));
    RC(dalloc(ctx, &ctx->zx, ctx->n + ctx->n_ghost));
    CK(cudaMemset(ctx->zx, 0, sizeof(double) * (ctx->n + ctx->n_ghost)));
    return DFL_OK;
}

// ||b|| (deflation.py:266), b' = project(b), ||b'||; r0 = shadow = b', d0 = 0,
// u = 0.  out.converged = 1 (and x = 0) when b or b' vanishes
// (krylov.py:270-272); otherwise out.resnorm = ||b'|| and out.rho1 = b'.b'.
int bicg_prologue(dfl_ctx *ctx, const dfl_solve_params *p, KState &out) {
    RC(bicg_alloc(ctx));
    const bool defl = p->deflated != 0;
    const int64_t n = ctx->n;
    const unsigned nb = (unsigned)ctx->nblk;
    out = KState{};
    double val[3];
    RC(dots(ctx, 1, ctx->b, ctx->b, nullptr, nullptr, nullptr, nullptr, val));
    out.bnorm = std::sqrt(std::max(val[0], 0.0));
    const double target = std::max(0.0, p->tol * out.bnorm);  // max(tol*||b'||, atol) with tol = 0
    out.target = target;
    launch_k(ctx->st, k_fill, nb, kBlock, 0, ctx->bu, 0.0, n);
    ctx->launches++;
    if (out.bnorm == 0.0) {
        out.converged = 1;
        launch_k(ctx->st, k_fill, nb, kBlock, 0, ctx->x, 0.0, n);
        ctx->launches++;
        return DFL_OK;
    }
    const bool x0 = use_x0(ctx, p);
    if (defl) {
        RC(project_dev(ctx, ctx->b, ctx->bp, nullptr, 0));
    } else if (x0) {  // r0 = b - A x0 (krylov.py:275)
        launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->x, (const double *)ctx->x0, n);
        ctx->launches++;
        RC(op_apply_dev(ctx, ctx->x, ctx->bp, 1, ctx->b, false, nullptr, 0));
    } else {
        launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->bp, ctx->b, n);
        ctx->launches++;
    }
    RC(dots(ctx, 1, ctx->bp, ctx->bp, nullptr, nullptr, nullptr, nullptr, val));
    out.rho1 = val[0];  // also r[0].shadow of the first step (both are b')
    out.resnorm = std::sqrt(std::max(val[0], 0.0));
    if (out.resnorm == 0.0) {  // the recurrence returns u = 0: x = x0 + M(0)
        out.converged = 1;
        if (x0)
            launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->x, (const double *)ctx->x0, n);
        else
            launch_k(ctx->st, k_fill, nb, kBlock, 0, ctx->x, 0.0, n);
        ctx->launches++;
        return DFL_OK;
    }
    launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->br[0], (const double *)ctx->bp, n);
    launch_k(ctx->st, k_fill, nb, kBlock, 0, ctx->bd[0], 0.0, n);
    launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->bshadow, (const double *)ctx->bp, n);
    ctx->launches += 3;
    return DFL_OK;
}

int bicg_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, KState &out) {
    RC(bicg_prologue(ctx, p, out));
    if (out.converged) return DFL_OK;
    const bool defl = p->deflated != 0;
    const int64_t n = ctx->n;
    const unsigned nb = (unsigned)ctx->nblk;
    const double target = out.target;
    const double bpbp = out.rho1, bpn = out.resnorm;
    double val[3];
    double *r[3] = {ctx->br[0], ctx->br[1], ctx->br[2]};
    double *d[3] = {ctx->bd[0], ctx->bd[1], ctx->bd[2]};
    double *u = ctx->bu, *shadow = ctx->bshadow;
    const double *r0init = ctx->bp;
    double rho0 = 1.0, alpha = 0.0, omega = 1.0;
    bool restarted = false;
    int brk = DFL_BRK_NONE;
    int iters = 0;
    double resnorm = bpn;  // ||r[0]|| with r[0] = b'
    // r[j].shadow is fetched together with the residual norm that precedes it
    // (one reduction, one host round trip); invalid after a restart
    double rho_next = bpbp;
    bool rho_valid = true;
    auto fail = [&](int code) -> int {
        rho_valid = false;
        if (restarted) return code;
        restarted = true;
        // r_shadow = r[0]; d = [0]; rho0, alpha, omega = 1, 0, 1  (krylov.py:165-175)
        launch_k(ctx->st, k_copy, nb, kBlock, 0, shadow, r[0], n);
        launch_k(ctx->st, k_fill, nb, kBlock, 0, d[0], 0.0, n);
        ctx->launches += 2;
        rho0 = 1.0;
        alpha = 0.0;
        omega = 1.0;
        return DFL_BRK_NONE;
    };
    const int refresh = std::max(1, p->refresh_every);
    double mr[3] = {0.0, 0.0, 0.0};  // r0.r1, r1.r1, r2.r1 after the BiCG part
    while (iters < p->maxiter && resnorm > target) {
        ++iters;
        rho0 = -omega * rho0;
        bool aborted = false, mid = false;
        for (int j = 0; j < 2; ++j) {
            double rho1 = rho_next;
            if (!rho_valid) {
                RC(dots(ctx, 1, r[j], shadow, nullptr, nullptr, nullptr, nullptr, val));
                rho1 = val[0];
            }
            rho_valid = false;
            if (rho0 == 0.0 || !std::isfinite(rho1)) {
                brk = fail(DFL_BRK_RHO);
                aborted = true;
                break;
            }
            const double beta = alpha * rho1 / rho0;
            rho0 = rho1;
            launch_k(ctx->st, k_bicg_d, nb, kBlock, 0, r[0], d[0], r[1], d[1], j + 1, beta, n);
            ctx->launches++;
            double gd;
            RC(op_hat(ctx, defl, d[j], d[j + 1], shadow, &gd));
            if (gd == 0.0 || !std::isfinite(gd)) {
                brk = fail(DFL_BRK_SHADOW);
                aborted = true;
                break;
            }
            alpha = rho0 / gd;
            launch_k(ctx->st, k_bicg_r, nb, kBlock, 0, r[0], d[1], r[1], d[2], j + 1, u, d[0], alpha, n, ctx->dpart);
            ctx->launches++;
            RC(op_hat(ctx, defl, r[j], r[j + 1], nullptr, nullptr));
            if (j == 0) {  // ||r0|| and the next step's rho1 = r1.shadow
                double v2[4];
                RC(dots(ctx, 2, r[0], r[0], r[1], shadow, nullptr, nullptr, v2));
                resnorm = std::sqrt(std::max(v2[0], 0.0));
                rho_next = v2[1];
                rho_valid = true;
            } else {  // ||r0|| and the minimal-residual dots
                double v4[4];
                RC(dots(ctx, 4, r[0], r[0], r[0], r[1], r[1], r[1], v4, r[2], r[1]));
                resnorm = std::sqrt(std::max(v4[0], 0.0));
                mr[0] = v4[1];
                mr[1] = v4[2];
                mr[2] = v4[3];
            }
            if (resnorm <= target) {
                mid = true;
                break;
            }
        }
        if (aborted) {
            RC(dots(ctx, 1, r[0], r[0], nullptr, nullptr, nullptr, nullptr, val));
            resnorm = std::sqrt(std::max(val[0], 0.0));
            if (brk != DFL_BRK_NONE || resnorm <= target) break;
            continue;
        }
        if (mid) break;
        // minimal-residual step on r[1..2] (modified Gram-Schmidt, krylov.py:207-255)
        const double sigma1 = mr[1];
        if (sigma1 == 0.0 || !std::isfinite(sigma1)) {
            brk = fail(DFL_BRK_MR);
            if (brk != DFL_BRK_NONE) break;
            continue;
        }
        const double gp1 = mr[0] / sigma1;
        const double tau12 = mr[2] / sigma1;
        {
            const unsigned g = dot_grid(ctx);
            launch_k(ctx->st, k_bicg_mr2, g, kBlock, 0, r[2], r[1], r[0], tau12, n, ctx->dpart);
            ctx->launches++;
            RC(global_dots(ctx, ctx->dpart, g, 2, true, val));
        }
        const double sigma2 = val[0];
        if (sigma2 == 0.0 || !std::isfinite(sigma2)) {
            brk = fail(DFL_BRK_MR);
            if (brk != DFL_BRK_NONE) break;
            continue;
        }
        const double gp2 = val[1] / sigma2;
        const double g2 = gp2;
        omega = g2;
        if (omega == 0.0 || !std::isfinite(omega)) {
            brk = fail(DFL_BRK_OMEGA);
            if (brk != DFL_BRK_NONE) break;
            continue;
        }
        const double g1 = gp1 - tau12 * g2;
        const double gpp1 = g2 + 0.0;
        launch_k(ctx->st, k_bicg_final, nb, kBlock, 0, u, r[0], d[0], r[1], r[2], d[1], d[2], g1, gp2, g2, gpp1, gp1, n,
                                                 ctx->dpart);
        ctx->launches++;
        if (iters % refresh == 0) {
            // r[0] = r0 - op_hat(u)   (krylov.py:256-257)
            RC(op_hat(ctx, defl, u, ctx->tmp, nullptr, nullptr));
            ProjArgs a = proj_args(ctx, ctx->tmp, r[0], nullptr);
            a.azd = nullptr;
            a.K = 0;
            a.base = r0init;
            launch_project<1>(ctx, a);  // r[0] = r0 - tmp
        }
        double v2[4];  // ||r0|| and the next group's rho1 = r0.shadow
        RC(dots(ctx, 2, r[0], r[0], r[0], shadow, nullptr, nullptr, v2));
        resnorm = std::sqrt(std::max(v2[0], 0.0));
        rho_next = v2[1];
        rho_valid = true;
    }
    // x = x0 + M(u)  (krylov.py:284-285), into ctx->x (the y of the deflated system)
    RC(vcycle(ctx, u, ctx->x, nullptr, nullptr, nullptr));
    if (use_x0(ctx, p)) {
        launch_k(ctx->st, k_addv, nb, kBlock, 0, ctx->x, (const double *)ctx->x0, n);
        ctx->launches++;
    }
    out.iters = iters;
    out.resnorm = resnorm;
    out.converged = resnorm <= target;
    out.breakdown = out.converged ? DFL_BRK_NONE : brk;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// Restarted (F)GMRES (krylov.py:288-414), right preconditioned; host-driven:
// the Hessenberg column, the Givens rotations and the back substitution run
// on the host in IEEE double exactly as the reference's Python; one host
// round trip per Arnoldi step.

// Hessenberg column / dot-slot stride: >= restart + 1 (buffers grow with M)
static int gm_alloc(dfl_ctx *ctx, int restart, bool flexible) {
    if (restart < 1) {  // krylov.py:374-375
        ctx->err = "restart length must be positive, got " + std::to_string(restart);
        return DFL_E_CONFIG;
    }
    RC(bicg_alloc(ctx));  // zx
    const int64_t nx = ctx->n + ctx->n_ghost;
    while ((int)ctx->gmV.size() < restart + 1) {
        double *v;
        RC(dalloc(ctx, &v, ctx->n));
        ctx->gmV.push_back(v);
    }
    if (flexible)
        while ((int)ctx->gmZ.size() < restart) {
            double *z;
            RC(dalloc(ctx, &z, nx));  // operator inputs: ghost tail
            CK(cudaMemset(z, 0, sizeof(double) * nx));
            ctx->gmZ.push_back(z);
        }
    if (ctx->gm_ld < restart + 1) {
        int ld = 128;
        while (ld < restart + 1) ld *= 2;
        if (ctx->h_gm) cudaFreeHost(ctx->h_gm);
        RC(dalloc(ctx, (double **)&ctx->gmVp, ld));
        RC(dalloc(ctx, (double **)&ctx->gmZp, ld));
        RC(dalloc(ctx, &ctx->gm_h, ld));
        RC(dalloc(ctx, &ctx->gm_e, ld));
        RC(dalloc(ctx, &ctx->gm_y, ld));
        RC(dalloc(ctx, &ctx->gm_loc, ld));
        RC(dalloc(ctx, &ctx->gm_gath, (int64_t)ld * ctx->nranks));
        RC(dalloc(ctx, &ctx->gm_part, (int64_t)ld * 4 * ctx->sm_count));
        CK(cudaMallocHost(&ctx->h_gm, 4 * (size_t)ld * sizeof(double)));
        ctx->gm_ld = ld;
    }
    CK(cudaMemcpy((void *)ctx->gmVp, ctx->gmV.data(), sizeof(double *) * ctx->gmV.size(), cudaMemcpyHostToDevice));
    if (!ctx->gmZ.empty())
        CK(cudaMemcpy((void *)ctx->gmZp, ctx->gmZ.data(), sizeof(double *) * ctx->gmZ.size(), cudaMemcpyHostToDevice));
    ctx->gm_restart = restart;
    return DFL_OK;
}

// dev_out[0..nvec) = sum over ranks of V[0..nvec) . w
static int gm_vdots(dfl_ctx *ctx, int nvec, const double *w, double *dev_out) {
    const unsigned gx = (unsigned)std::min<int64_t>(std::max<int64_t>(1, ctx->nblk), 4 * ctx->sm_count);
    const dim3 grid(gx, (unsigned)cdiv(nvec, kVecGroup));
    launch_k(ctx->st, k_vdots, grid, kBlock, 0, ctx->gmVp, nvec, w, ctx->n, ctx->gm_part, ctx->gm_ld);
    ctx->launches++;
    if (!multi(ctx)) {
        launch_k(ctx->st, k_vreduce, nvec, 1024, 0, ctx->gm_part, gx, ctx->gm_ld, dev_out);
        ctx->launches++;
        return DFL_OK;
    }
    launch_k(ctx->st, k_vreduce, nvec, 1024, 0, ctx->gm_part, gx, ctx->gm_ld, ctx->gm_loc);
    RC(comm_allgather(ctx, ctx->gm_loc, ctx->gm_gath, ctx->gm_ld));
    launch_k(ctx->st, k_rank_sum, (unsigned)cdiv(nvec, 256), 256, 0, ctx->gm_gath, ctx->nranks, ctx->gm_ld, nvec, dev_out);
    ctx->launches += 2;
    return DFL_OK;
}

// r = b' - project(A x), returns ||r||   (krylov.py:408)
static int gm_residual(dfl_ctx *ctx, bool defl, double *resnorm) {
    RC(op_apply_dev(ctx, ctx->x, ctx->w, 0, nullptr, defl, nullptr, 0));
    if (defl) RC(zt_to_t2(ctx, nullptr, 0, true));
    ProjArgs a = proj_args(ctx, ctx->w, ctx->r, nullptr);
    if (!defl) a.azd = nullptr, a.K = 0;
    a.base = ctx->bp;
    a.dotmode = 2;
    a.dot_part = ctx->dpart;
    launch_project<1>(ctx, a);
    double v[4];
    RC(global_dots(ctx, ctx->dpart, ctx->vgrid, 1, false, v));
    *resnorm = std::sqrt(std::max(v[0], 0.0));
    return DFL_OK;
}

int gmres_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, bool flexible, KState &out) {
    const bool defl = p->deflated != 0;
    const int M = p->restart;
    const int64_t n = ctx->n;
    const unsigned nb = (unsigned)ctx->nblk;
    const unsigned gx = (unsigned)std::min<int64_t>(std::max<int64_t>(1, ctx->nblk), 4 * ctx->sm_count);
    out = KState{};
    double val[4];
    RC(dots(ctx, 1, ctx->b, ctx->b, nullptr, nullptr, nullptr, nullptr, val));
    out.bnorm = std::sqrt(std::max(val[0], 0.0));
    const double target = std::max(0.0, p->tol * out.bnorm);
    out.target = target;
    launch_k(ctx->st, k_fill, nb, kBlock, 0, ctx->x, 0.0, n);
    ctx->launches++;
    if (out.bnorm == 0.0) {
        out.converged = 1;
        return DFL_OK;
    }
    RC(gm_alloc(ctx, M, flexible));  // b != 0: the restart length is checked here, as krylov.py:370-375
    if (defl) {
        RC(project_dev(ctx, ctx->b, ctx->bp, nullptr, 0));
    } else {
        launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->bp, ctx->b, n);
        ctx->launches++;
    }
    double resnorm;
    if (use_x0(ctx, p)) {  // x = x0, r = b - A x0 (krylov.py:383)
        launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->x, (const double *)ctx->x0, n);
        ctx->launches++;
        RC(gm_residual(ctx, defl, &resnorm));
    } else {
        RC(dots(ctx, 1, ctx->bp, ctx->bp, nullptr, nullptr, nullptr, nullptr, val));
        resnorm = std::sqrt(std::max(val[0], 0.0));
        launch_k(ctx->st, k_copy, nb, kBlock, 0, ctx->r, ctx->bp, n);
    }
    if (resnorm == 0.0) {
        out.converged = 1;
        return DFL_OK;
    }
    ctx->launches++;
    std::vector<double> H((size_t)(M + 1) * M), g(M + 1), cs(M), sn(M), y(M);
    auto h = [&](int i, int j) -> double & { return H[(size_t)i * M + j]; };
    int total = 0;
    while (total < p->maxiter && resnorm > target) {
        const int steps = std::min(M, p->maxiter - total);
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = resnorm;
        launch_k(ctx->st, k_vdiv, nb, kBlock, 0, ctx->gmV[0], ctx->r, resnorm, n);  // V0 = r0 / ||r0||
        ctx->launches++;
        int j = 0;
        while (j < steps) {
            double *w = ctx->w;
            if (flexible) {  // z_j = M(V_j), w = project(A z_j)
                RC(vcycle(ctx, ctx->gmV[j], ctx->gmZ[j], nullptr, nullptr, nullptr));
                RC(op_apply_dev(ctx, ctx->gmZ[j], w, 0, nullptr, defl, nullptr, 0));
                if (defl) RC(zt_to_t2(ctx, nullptr, 0, true));
                ProjArgs a = proj_args(ctx, w, w, nullptr);
                if (!defl) a.azd = nullptr, a.K = 0;
                launch_project<0>(ctx, a);
            } else {  // w = project(A (M V_j))
                RC(op_hat(ctx, defl, ctx->gmV[j], ctx->tmp, nullptr, nullptr));
                w = ctx->tmp;
            }
            // two Gram-Schmidt passes against V_0..V_j, then ||w||
            RC(gm_vdots(ctx, j + 1, w, ctx->gm_h));
            launch_k(ctx->st, k_vsub, gx, kBlock, 0, w, ctx->gmVp, ctx->gm_h, j + 1, n, nullptr);
            RC(gm_vdots(ctx, j + 1, w, ctx->gm_e));
            launch_k(ctx->st, k_vsub, gx, kBlock, 0, w, ctx->gmVp, ctx->gm_e, j + 1, n, ctx->dpart);
            ctx->launches += 2;
            RC(global_dots(ctx, ctx->dpart, gx, 1, false, val));
            CK(cudaMemcpyAsync(ctx->h_gm, ctx->gm_h, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaMemcpyAsync(ctx->h_gm + ctx->gm_ld, ctx->gm_e, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost,
                               ctx->st));
            RC(comm_wait(ctx, ctx->st));
            for (int i = 0; i <= j; ++i) {
                h(i, j) = ctx->h_gm[i];
                h(i, j) += ctx->h_gm[ctx->gm_ld + i];
            }
            const double hj1 = std::sqrt(std::max(val[0], 0.0));
            h(j + 1, j) = hj1;
            const bool exact = hj1 == 0.0;
            if (!exact) {
                launch_k(ctx->st, k_vdiv, nb, kBlock, 0, ctx->gmV[j + 1], w, hj1, n);
                ctx->launches++;
            }
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
                h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
                h(i, j) = t;
            }
            const double rad = std::hypot(h(j, j), h(j + 1, j));
            cs[j] = rad == 0.0 ? 1.0 : h(j, j) / rad;
            sn[j] = rad == 0.0 ? 0.0 : h(j + 1, j) / rad;
            h(j, j) = cs[j] * h(j, j) + sn[j] * h(j + 1, j);
            h(j + 1, j) = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            const double res = std::fabs(g[j + 1]);
            ++j;
            if (exact || res <= target) break;
        }
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int q = i + 1; q < j; ++q) s += h(i, q) * y[q];
            y[i] = (g[i] - s) / h(i, i);
        }
        CK(cudaMemcpyAsync(ctx->gm_y, y.data(), sizeof(double) * j, cudaMemcpyHostToDevice, ctx->st));
        if (flexible) {  // x = x + (Z_0 y_0 + y_1 Z_1 + ...)
            launch_k(ctx->st, k_vcombine, gx, kBlock, 0, ctx->x, ctx->x, ctx->gmZp, ctx->gm_y, j, n);
            ctx->launches++;
        } else {  // x = x + M(V_0 y_0 + ...)
            launch_k(ctx->st, k_vcombine, gx, kBlock, 0, ctx->tmp, nullptr, ctx->gmVp, ctx->gm_y, j, n);
            RC(vcycle(ctx, ctx->tmp, ctx->zx, nullptr, nullptr, nullptr));
            launch_k(ctx->st, k_addv, nb, kBlock, 0, ctx->x, ctx->zx, n);
            ctx->launches += 2;
        }
        RC(comm_wait(ctx, ctx->st));  // y (host vector) was read by the async copy above
        total += j;
        RC(gm_residual(ctx, defl, &resnorm));
    }
    out.iters = total;
    out.resnorm = resnorm;
    out.converged = resnorm <= target;
    return DFL_OK;
}

