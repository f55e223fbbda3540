// Pressure-Schur block solver on the device (reference schur.py, paper §4.2):
// outer flexible GMRES on the monolithic saddle-point matrix, right
// preconditioned by the three-step pressure-correction sweep
//   1. K u = b_u                  GMRES, SPAI-0 right preconditioner,
//   2. (S - D diag(K)^-1 G) p = b_p - D u
//                                 FGMRES on the matrix-free Schur operator,
//                                 preconditioner block AMG(project(r)) + lift(r)
//                                 of the deflated solver built on S,
//   3. K u = b_u - G p            as 1.
// Every Krylov method here is the generic restarted (F)GMRES below (Arnoldi
// with two classical Gram-Schmidt passes, host Givens rotations), driven on
// the stream of the pressure context so the deflated-AMG pieces (vcycle,
// project_dev, k_lift) interleave with the block kernels without events.
#include "ctx_impl.cuh"

#include <functional>

static constexpr int kBlkLd = 128;  // max restart + 1

// dst[idx[i]] = src[i]  (BlockSystem.merge, schur.py:77-81)
static __global__ void k_scatter(const double *__restrict__ src, const int *__restrict__ idx, int64_t m,
                                 double *dst) {
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < m) dst[idx[i]] = src[i];
}

static __global__ void k_mul(double *out, const double *__restrict__ a, const double *__restrict__ b, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < n) out[i] = mul_rn(a[i], b[i]);
}

static __global__ void k_sub(double *out, const double *__restrict__ a, const double *__restrict__ b, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < n) out[i] = sub_rn(a[i], b[i]);
}

namespace {

using Apply = std::function<int(const double *in, double *out)>;

// a matrix of the block system: empty (no rows or no entries) -> zero product
struct BMat {
    DMat m;
    int64_t nrows = 0;
    bool zero = true;
};

// workspace of one restarted (F)GMRES level
struct GmSpace {
    int64_t n = 0;
    int cap = 0;
    bool flex = false;
    std::vector<double *> V, Z;
    const double **Vp = nullptr, **Zp = nullptr;
    double *w = nullptr, *t = nullptr, *r = nullptr;
    double *hb = nullptr;    // device: h [0, ld), e [ld, 2 ld), ||w||^2 at 2 ld
    double *y = nullptr;     // device: ld
    double *part = nullptr;  // ld x grid partials
    double *hh = nullptr;    // pinned: copy of hb, then y
};

}  // namespace

struct dfl_block {
    dfl_ctx *ctx = nullptr;   // stream / allocations (the pressure context, or own)
    dfl_ctx *own = nullptr;
    bool pressure = false;    // ctx holds the deflated solver of S
    std::string err;
    int64_t n = 0, nu = 0, np = 0;
    BMat A, K, G, D, S;
    int *uidx = nullptr, *pidx = nullptr;
    double *wK = nullptr, *invKd = nullptr;
    // vectors
    double *b = nullptr, *x = nullptr, *bu = nullptr, *bp = nullptr, *u = nullptr, *p = nullptr, *tu = nullptr,
           *tp = nullptr, *gu = nullptr, *dp = nullptr, *sp = nullptr, *pt = nullptr,
           *pz = nullptr;  // pz, pt: pressure preconditioner scratch
    GmSpace outer, vel, pre;
    std::vector<void *> mine;  // allocations owned by the block (freed with it)
    int64_t bytes = 0;
    int64_t vel_its = 0, pre_its = 0;
};

namespace {

// move the context allocations made since `a0` into the block's ownership
void adopt(dfl_block *B, size_t a0, int64_t b0) {
    auto &al = B->ctx->allocs;
    for (size_t i = a0; i < al.size(); ++i) B->mine.push_back(al[i]);
    B->bytes += B->ctx->bytes - b0;
}

template <class T>
int balloc(dfl_block *B, T **p, int64_t count) {
    const size_t a0 = B->ctx->allocs.size();
    const int64_t b0 = B->ctx->bytes;
    RC(dalloc(B->ctx, p, count));
    adopt(B, a0, b0);
    return DFL_OK;
}

int bmat(dfl_block *B, const dfl_csr *h, int64_t nrows, int64_t ncols, BMat &out) {
    dfl_ctx *ctx = B->ctx;
    out = BMat{};
    out.nrows = nrows;
    if (!h) {
        if (nrows == 0 || ncols == 0) return DFL_OK;
        ctx->err = "missing block matrix";
        return DFL_E_STATE;
    }
    if (h->nrows != nrows || h->ncols != ncols) {
        ctx->err = "block matrix shape does not match the mask";
        return DFL_E_DIMENSION;
    }
    const int64_t nnz = nrows ? h->row_ptr[nrows] - h->row_ptr[0] : 0;
    if (nnz == 0) return DFL_OK;
    const size_t a0 = ctx->allocs.size();
    const int64_t b0 = ctx->bytes;
    HostRows hr{h->nrows, h->ncols, h->row_ptr, h->col_idx, h->values};
    const int rc = upload_matrix(ctx, hr, out.m, {0, nrows});
    adopt(B, a0, b0);
    RC(rc);
    out.zero = false;
    return DFL_OK;
}

inline unsigned nb_of(int64_t n) { return (unsigned)std::max<int64_t>(1, cdiv(n, kBlock)); }

inline unsigned gx_of(const dfl_ctx *ctx, int64_t n) {
    return (unsigned)std::min<int64_t>(std::max<int64_t>(1, cdiv(n, kBlock)), 4 * ctx->sm_count);
}

// y = M x (y has M.nrows entries)
int spmv(dfl_block *B, const BMat &M, const double *x, double *y) {
    dfl_ctx *ctx = B->ctx;
    if (M.nrows == 0) return DFL_OK;
    if (M.zero) {
        k_fill<<<nb_of(M.nrows), kBlock, 0, ctx->st>>>(y, 0.0, M.nrows);
    } else {
        RowArgs a{x, nullptr, nullptr, nullptr, y, nullptr, nullptr};
        launch_rows<MODE_PLAIN, false>(ctx, M.m, a);
    }
    ctx->launches++;
    return DFL_OK;
}

int gm_space(dfl_block *B, GmSpace &S, int64_t n, int cap, bool flex) {
    dfl_ctx *ctx = B->ctx;
    if (cap < 1 || cap + 1 > kBlkLd) {
        ctx->err = "GMRES restart must be in [1, " + std::to_string(kBlkLd - 1) + "]";
        return DFL_E_CONFIG;
    }
    S.n = n;
    S.flex = S.flex || flex;
    if (!S.hb) {
        RC(balloc(B, (double **)&S.Vp, kBlkLd));
        RC(balloc(B, (double **)&S.Zp, kBlkLd));
        RC(balloc(B, &S.hb, 2 * kBlkLd + 2));
        RC(balloc(B, &S.y, kBlkLd));
        RC(balloc(B, &S.part, (int64_t)kBlkLd * 4 * ctx->sm_count));
        RC(balloc(B, &S.w, n));
        RC(balloc(B, &S.t, n));
        RC(balloc(B, &S.r, n));
        CK(cudaMallocHost(&S.hh, (2 * kBlkLd + 2) * sizeof(double)));
    }
    while ((int)S.V.size() < cap + 1) {
        double *v;
        RC(balloc(B, &v, n));
        S.V.push_back(v);
    }
    if (S.flex)
        while ((int)S.Z.size() < cap) {
            double *z;
            RC(balloc(B, &z, n));
            S.Z.push_back(z);
        }
    S.cap = std::max(S.cap, cap);
    CK(cudaMemcpy((void *)S.Vp, S.V.data(), sizeof(double *) * S.V.size(), cudaMemcpyHostToDevice));
    if (!S.Z.empty())
        CK(cudaMemcpy((void *)S.Zp, S.Z.data(), sizeof(double *) * S.Z.size(), cudaMemcpyHostToDevice));
    return DFL_OK;
}

// sqrt(max(v.v, 0)) on the host
int norm(dfl_block *B, GmSpace &S, const double *v, double *out) {
    dfl_ctx *ctx = B->ctx;
    const unsigned g = gx_of(ctx, S.n);
    k_dot<<<g, kBlock, 0, ctx->st>>>(v, v, S.n, S.part, nullptr);
    k_reduce<<<1, 1024, 0, ctx->st>>>(S.part, g, S.hb + 2 * kBlkLd);
    ctx->launches += 2;
    CK(cudaMemcpyAsync(S.hh, S.hb + 2 * kBlkLd, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    *out = std::sqrt(std::max(S.hh[0], 0.0));
    return DFL_OK;
}

// hb[off .. off + nvec) = V[0..nvec) . w
int vdots(dfl_block *B, GmSpace &S, int nvec, const double *w, int off) {
    dfl_ctx *ctx = B->ctx;
    const unsigned gx = gx_of(ctx, S.n);
    const dim3 grid(gx, (unsigned)cdiv(nvec, kVecGroup));
    k_vdots<<<grid, kBlock, 0, ctx->st>>>(S.Vp, nvec, w, S.n, S.part, kBlkLd);
    k_vreduce<<<nvec, 1024, 0, ctx->st>>>(S.part, gx, kBlkLd, S.hb + off);
    ctx->launches += 2;
    return DFL_OK;
}

struct GmOut {
    int iters = 0;
    double resnorm = 0.0;
    bool converged = true;
};

// Restarted (F)GMRES, right preconditioned, x0 = 0 (krylov.py:288-398 with
// the driver of :366-398); target = max(tol ||b||, atol).  M == nullptr: no
// preconditioner.  x receives the solution (n entries).
int gmres_any(dfl_block *B, GmSpace &S, bool flex, const Apply &op, const Apply *M, const double *b, double *x,
              double tol, double atol, int maxiter, int restart, GmOut &res) {
    dfl_ctx *ctx = B->ctx;
    const int64_t n = S.n;
    res = GmOut{};
    if (n == 0) return DFL_OK;
    if (flex && !S.flex) {
        ctx->err = "flexible GMRES on a workspace without Z vectors";
        return DFL_E_STATE;
    }
    const unsigned nb = nb_of(n), gx = gx_of(ctx, n);
    k_fill<<<nb, kBlock, 0, ctx->st>>>(x, 0.0, n);
    ctx->launches++;
    double bnorm;
    RC(norm(B, S, b, &bnorm));
    if (bnorm == 0.0) return DFL_OK;
    const double target = std::max(tol * bnorm, atol);
    const int Mr = std::min(restart, S.cap);
    k_copy<<<nb, kBlock, 0, ctx->st>>>(S.r, b, n);
    ctx->launches++;
    double resnorm = bnorm;
    std::vector<double> H((size_t)(Mr + 1) * Mr), g(Mr + 1), cs(Mr), sn(Mr), y(Mr);
    auto h = [&](int i, int j) -> double & { return H[(size_t)i * Mr + j]; };
    int total = 0;
    while (total < maxiter && resnorm > target) {
        const int steps = std::min(Mr, maxiter - total);
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = resnorm;
        k_vdiv<<<nb, kBlock, 0, ctx->st>>>(S.V[0], S.r, resnorm, n);
        ctx->launches++;
        int j = 0;
        while (j < steps) {
            if (flex) {  // z_j = M(V_j) (a copy without M), w = op(z_j)
                if (M) {
                    RC((*M)(S.V[j], S.Z[j]));
                } else {
                    k_copy<<<nb, kBlock, 0, ctx->st>>>(S.Z[j], S.V[j], n);
                    ctx->launches++;
                }
                RC(op(S.Z[j], S.w));
            } else if (M) {  // w = op(M(V_j))
                RC((*M)(S.V[j], S.t));
                RC(op(S.t, S.w));
            } else {
                RC(op(S.V[j], S.w));
            }
            RC(vdots(B, S, j + 1, S.w, 0));
            k_vsub<<<gx, kBlock, 0, ctx->st>>>(S.w, S.Vp, S.hb, j + 1, n, nullptr);
            RC(vdots(B, S, j + 1, S.w, kBlkLd));
            k_vsub<<<gx, kBlock, 0, ctx->st>>>(S.w, S.Vp, S.hb + kBlkLd, j + 1, n, S.part);
            k_reduce<<<1, 1024, 0, ctx->st>>>(S.part, gx, S.hb + 2 * kBlkLd);
            ctx->launches += 3;
            CK(cudaMemcpyAsync(S.hh, S.hb, sizeof(double) * (2 * kBlkLd + 1), cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            for (int i = 0; i <= j; ++i) {
                h(i, j) = S.hh[i];
                h(i, j) += S.hh[kBlkLd + i];
            }
            const double hj1 = std::sqrt(std::max(S.hh[2 * kBlkLd], 0.0));
            h(j + 1, j) = hj1;
            const bool exact = hj1 == 0.0;
            if (!exact) {
                k_vdiv<<<nb, kBlock, 0, ctx->st>>>(S.V[j + 1], S.w, hj1, n);
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
            const double inner = std::fabs(g[j + 1]);
            ++j;
            if (exact || inner <= target) break;
        }
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int q = i + 1; q < j; ++q) s += h(i, q) * y[q];
            y[i] = (g[i] - s) / h(i, i);
        }
        for (int i = 0; i < j; ++i) S.hh[i] = y[i];
        CK(cudaMemcpyAsync(S.y, S.hh, sizeof(double) * j, cudaMemcpyHostToDevice, ctx->st));
        if (flex) {  // x = x + (Z_0 y_0 + y_1 Z_1 + ...)
            k_vcombine<<<gx, kBlock, 0, ctx->st>>>(x, x, S.Zp, S.y, j, n);
            ctx->launches++;
        } else if (M) {  // x = x + M(V_0 y_0 + ...)
            k_vcombine<<<gx, kBlock, 0, ctx->st>>>(S.w, nullptr, S.Vp, S.y, j, n);
            ctx->launches++;
            RC((*M)(S.w, S.t));
            k_addv<<<nb, kBlock, 0, ctx->st>>>(x, S.t, n);
            ctx->launches++;
        } else {
            k_vcombine<<<gx, kBlock, 0, ctx->st>>>(x, x, S.Vp, S.y, j, n);
            ctx->launches++;
        }
        total += j;
        RC(op(x, S.w));  // r = b - op(x)
        k_sub<<<nb, kBlock, 0, ctx->st>>>(S.r, b, S.w, n);
        ctx->launches++;
        RC(norm(B, S, S.r, &resnorm));  // synchronises: the pinned y copy has been consumed
    }
    res.iters = total;
    res.resnorm = resnorm;
    res.converged = resnorm <= target;
    return DFL_OK;
}

// out = S p - D diag(K)^-1 G p   (schur.py:145-152)
int schur_apply(dfl_block *B, const double *p, double *out) {
    dfl_ctx *ctx = B->ctx;
    if (B->np == 0) return DFL_OK;
    RC(spmv(B, B->S, p, B->sp));
    if (B->nu == 0) {
        k_copy<<<nb_of(B->np), kBlock, 0, ctx->st>>>(out, B->sp, B->np);
        ctx->launches++;
        return DFL_OK;
    }
    RC(spmv(B, B->G, p, B->gu));
    k_mul<<<nb_of(B->nu), kBlock, 0, ctx->st>>>(B->gu, B->invKd, B->gu, B->nu);
    ctx->launches++;
    RC(spmv(B, B->D, B->gu, B->dp));
    k_sub<<<nb_of(B->np), kBlock, 0, ctx->st>>>(out, B->sp, B->dp, B->np);
    ctx->launches++;
    return DFL_OK;
}

struct SweepParams {
    bool uflex, pflex;
    int umaxiter, pmaxiter;
    double utol, ptol;
};

// the three-step sweep (schur.py:235-251): (b_u, b_p) -> (u, p)
int sweep(dfl_block *B, const SweepParams &sp, const double *b_u, const double *b_p, double *u, double *p) {
    dfl_ctx *ctx = B->ctx;
    const Apply opK = [B](const double *v, double *o) { return spmv(B, B->K, v, o); };
    const Apply MK = [B, ctx](const double *v, double *o) {
        k_mul<<<nb_of(B->nu), kBlock, 0, ctx->st>>>(o, B->wK, v, B->nu);
        ctx->launches++;
        return DFL_OK;
    };
    GmOut r;
    if (B->nu) {
        RC(gmres_any(B, B->vel, sp.uflex, opK, &MK, b_u, u, sp.utol, 0.0, sp.umaxiter, 50, r));
        B->vel_its += r.iters;
    }
    if (B->np == 0) return DFL_OK;
    if (B->nu) {  // b_p - D u
        RC(spmv(B, B->D, u, B->dp));
        k_sub<<<nb_of(B->np), kBlock, 0, ctx->st>>>(B->tp, b_p, B->dp, B->np);
    } else {
        k_copy<<<nb_of(B->np), kBlock, 0, ctx->st>>>(B->tp, b_p, B->np);
    }
    ctx->launches++;
    const Apply opS = [B](const double *v, double *o) { return schur_apply(B, v, o); };
    // M(r) = block_amg(project(r)) + coarse_lift(r): project_dev leaves
    // t2 = E^-1 Z' r, which is also the coarse correction of the lift
    const Apply MP = [B, ctx](const double *v, double *o) {
        RC(project_dev(ctx, v, B->pt, nullptr, 0));
        RC(vcycle(ctx, B->pt, B->pz, nullptr, nullptr, nullptr));
        k_lift<<<(unsigned)ctx->ntiles, kBlock, 0, ctx->st>>>(ctx->tiles, ctx->tile_sub, B->pz, ctx->zcols, ctx->n,
                                                              ctx->k, ctx->t2, (int64_t)ctx->first_sub * ctx->k, o,
                                                              1, zcode_of(ctx));
        ctx->launches++;
        return DFL_OK;
    };
    RC(gmres_any(B, B->pre, sp.pflex, opS, B->pressure ? &MP : nullptr, B->tp, p, sp.ptol, 0.0, sp.pmaxiter, 50, r));
    B->pre_its += r.iters;
    if (B->nu) {  // b_u - G p, then the velocity solve again
        RC(spmv(B, B->G, p, B->gu));
        k_sub<<<nb_of(B->nu), kBlock, 0, ctx->st>>>(B->tu, b_u, B->gu, B->nu);
        ctx->launches++;
        RC(gmres_any(B, B->vel, sp.uflex, opK, &MK, B->tu, u, sp.utol, 0.0, sp.umaxiter, 50, r));
        B->vel_its += r.iters;
    }
    return DFL_OK;
}

int sweep_params(dfl_block *B, const dfl_block_params *p, SweepParams &sp) {
    auto flex = [&](int s, bool &f) {
        if (s != DFL_SOLVER_GMRES && s != DFL_SOLVER_FGMRES) {
            B->ctx->err = "the inner solvers of the block preconditioner must be gmres or fgmres";
            return DFL_E_CONFIG;
        }
        f = s == DFL_SOLVER_FGMRES;
        return DFL_OK;
    };
    if (B->np && !B->pressure) {
        B->ctx->err = "a block solve with pressure unknowns needs the pressure context";
        return DFL_E_STATE;
    }
    RC(flex(p->usolver, sp.uflex));
    RC(flex(p->psolver, sp.pflex));
    sp.umaxiter = p->umaxiter;
    sp.pmaxiter = p->pmaxiter;
    sp.utol = p->utol;
    sp.ptol = p->ptol;
    if (B->nu) RC(gm_space(B, B->vel, B->nu, std::max(1, std::min(50, p->umaxiter)), sp.uflex));
    if (B->np) RC(gm_space(B, B->pre, B->np, std::max(1, std::min(50, p->pmaxiter)), sp.pflex));
    return DFL_OK;
}

int stage(dfl_block *B, double *dst, const double *src, int64_t n, int ptr_kind, bool in) {
    if (n == 0) return DFL_OK;
    dfl_ctx *ctx = B->ctx;
    const cudaMemcpyKind k = ptr_kind == DFL_PTR_HOST ? (in ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost)
                                                      : cudaMemcpyDeviceToDevice;
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, k, ctx->st));
    if (!in) CK(cudaStreamSynchronize(ctx->st));
    return DFL_OK;
}

int block_err(dfl_block *B, int rc) {
    if (rc != DFL_OK && B->ctx) B->err = B->ctx->err;
    return rc;
}

int create(dfl_block *B, dfl_ctx *pctx, int device, const dfl_block_desc *d) {
    if (pctx) {
        B->ctx = pctx;
        B->pressure = true;
        if (!pctx->finalized || multi(pctx)) {
            B->err = "the pressure context must be finalized and single-rank";
            return DFL_E_STATE;
        }
        if (!pctx->deflation) {
            B->err = "the pressure context has no deflation basis";
            return DFL_E_STATE;
        }
    } else {
        RC(dfl_ctx_create(device, &B->own));
        B->ctx = B->own;
    }
    dfl_ctx *ctx = B->ctx;
    CK(cudaSetDevice(ctx->device));
    B->n = d->n;
    B->nu = d->n_u;
    B->np = d->n - d->n_u;
    if (d->n < 0 || d->n_u < 0 || B->np < 0 || d->n >= INT32_MAX) {
        ctx->err = "bad block system size";
        return DFL_E_DIMENSION;
    }
    if (pctx && pctx->n != B->np) {
        ctx->err = "pressure context size differs from the pressure block";
        return DFL_E_DIMENSION;
    }
    RC(bmat(B, d->A, B->n, B->n, B->A));
    RC(bmat(B, d->K, B->nu, B->nu, B->K));
    RC(bmat(B, d->G, B->nu, B->np, B->G));
    RC(bmat(B, d->D, B->np, B->nu, B->D));
    RC(bmat(B, d->S, B->np, B->np, B->S));
    auto up_idx = [&](int **dst, const int32_t *src, int64_t m) -> int {
        RC(balloc(B, dst, m));
        if (m) CK(cudaMemcpy(*dst, src, sizeof(int) * m, cudaMemcpyHostToDevice));
        return DFL_OK;
    };
    auto up_vec = [&](double **dst, const double *src, int64_t m) -> int {
        RC(balloc(B, dst, m));
        if (m && src) CK(cudaMemcpy(*dst, src, sizeof(double) * m, cudaMemcpyHostToDevice));
        return DFL_OK;
    };
    RC(up_idx(&B->uidx, d->u_idx, B->nu));
    RC(up_idx(&B->pidx, d->p_idx, B->np));
    RC(up_vec(&B->wK, d->wK, B->nu));
    RC(up_vec(&B->invKd, d->invKdiag, B->nu));
    for (double **v : {&B->bu, &B->u, &B->tu, &B->gu}) RC(up_vec(v, nullptr, B->nu));
    for (double **v : {&B->bp, &B->p, &B->tp, &B->dp, &B->sp, &B->pt, &B->pz}) RC(up_vec(v, nullptr, B->np));
    for (double **v : {&B->b, &B->x}) RC(up_vec(v, nullptr, B->n));
    return DFL_OK;
}

}  // namespace

extern "C" {

int dfl_block_create(dfl_ctx *pctx, int device, const dfl_block_desc *d, dfl_block **out) {
    if (!out || !d) return DFL_E_STATE;
    *out = nullptr;
    auto *B = new dfl_block;
    const int rc = create(B, pctx, device, d);
    if (rc != DFL_OK) {
        dfl::set_setup_error(B->err.empty() && B->ctx ? B->ctx->err : B->err);
        dfl_block_free(B);
        return rc;
    }
    *out = B;
    return DFL_OK;
}

void dfl_block_free(dfl_block *B) {
    if (!B) return;
    for (GmSpace *S : {&B->outer, &B->vel, &B->pre})
        if (S->hh) cudaFreeHost(S->hh);
    if (B->own) {
        dfl_ctx_destroy(B->own);  // frees everything
    } else if (B->ctx) {
        cudaSetDevice(B->ctx->device);
        cudaStreamSynchronize(B->ctx->st);
        auto &al = B->ctx->allocs;
        for (void *q : B->mine) {
            cudaFree(q);
            al.erase(std::remove(al.begin(), al.end(), q), al.end());
        }
        B->ctx->bytes -= B->bytes;
    }
    delete B;
}

const char *dfl_block_last_error(const dfl_block *B) { return B ? B->err.c_str() : dfl::setup_error(); }

int64_t dfl_block_device_bytes(const dfl_block *B) { return B ? B->bytes : 0; }

int dfl_block_apply(dfl_block *B, const double *x, double *y, int ptr_kind) {
    if (!B) return DFL_E_STATE;
    dfl_ctx *ctx = B->ctx;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return DFL_E_CUDA;
    int rc = stage(B, B->b, x, B->n, ptr_kind, true);
    if (rc == DFL_OK) rc = spmv(B, B->A, B->b, B->x);
    if (rc == DFL_OK) rc = stage(B, y, B->x, B->n, ptr_kind, false);
    return block_err(B, rc);
}

int dfl_block_schur_apply(dfl_block *B, const double *p, double *out, int ptr_kind) {
    if (!B) return DFL_E_STATE;
    dfl_ctx *ctx = B->ctx;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return DFL_E_CUDA;
    int rc = stage(B, B->bp, p, B->np, ptr_kind, true);
    if (rc == DFL_OK) rc = schur_apply(B, B->bp, B->tp);
    if (rc == DFL_OK) rc = stage(B, out, B->tp, B->np, ptr_kind, false);
    return block_err(B, rc);
}

int dfl_block_precond(dfl_block *B, const dfl_block_params *prm, const double *b_u, const double *b_p, double *u,
                      double *p, int ptr_kind, int64_t *velocity_iterations, int64_t *pressure_iterations) {
    if (!B || !prm) return DFL_E_STATE;
    dfl_ctx *ctx = B->ctx;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return DFL_E_CUDA;
    SweepParams sp;
    int rc = sweep_params(B, prm, sp);
    B->vel_its = B->pre_its = 0;
    if (rc == DFL_OK) rc = stage(B, B->bu, b_u, B->nu, ptr_kind, true);
    if (rc == DFL_OK) rc = stage(B, B->bp, b_p, B->np, ptr_kind, true);
    // the sweep reads (bu, bp) and writes (u, p); tu / tp are its scratch
    if (rc == DFL_OK) rc = sweep(B, sp, B->bu, B->bp, B->u, B->p);
    if (rc == DFL_OK) rc = stage(B, u, B->u, B->nu, ptr_kind, false);
    if (rc == DFL_OK) rc = stage(B, p, B->p, B->np, ptr_kind, false);
    if (velocity_iterations) *velocity_iterations = B->vel_its;
    if (pressure_iterations) *pressure_iterations = B->pre_its;
    return block_err(B, rc);
}

int dfl_block_solve(dfl_block *B, const dfl_block_params *prm, const double *rhs, double *x, int ptr_kind,
                    dfl_block_report *rep) {
    if (!B || !prm || !rep) return DFL_E_STATE;
    dfl_ctx *ctx = B->ctx;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return DFL_E_CUDA;
    std::memset(rep, 0, sizeof *rep);
    SweepParams sp;
    int rc = sweep_params(B, prm, sp);
    if (rc == DFL_OK && (prm->restart < 1 || prm->restart + 1 > kBlkLd)) {
        ctx->err = "solver.M must be in [1, " + std::to_string(kBlkLd - 1) + "]";
        rc = DFL_E_CONFIG;
    }
    if (rc == DFL_OK) rc = gm_space(B, B->outer, B->n, prm->restart, true);
    if (rc != DFL_OK) return block_err(B, rc);
    B->vel_its = B->pre_its = 0;
    ctx->launches = 0;
    // outer operator: the monolithic matrix; preconditioner: merge(sweep(split(r)))
    const Apply opA = [B](const double *v, double *o) { return spmv(B, B->A, v, o); };
    const Apply Msw = [B, ctx, &sp](const double *r, double *z) {
        if (B->nu) k_gather<<<nb_of(B->nu), kBlock, 0, ctx->st>>>(r, B->uidx, B->nu, B->bu);
        if (B->np) k_gather<<<nb_of(B->np), kBlock, 0, ctx->st>>>(r, B->pidx, B->np, B->bp);
        ctx->launches += 2;
        RC(sweep(B, sp, B->bu, B->bp, B->u, B->p));
        if (B->nu) k_scatter<<<nb_of(B->nu), kBlock, 0, ctx->st>>>(B->u, B->uidx, B->nu, z);
        if (B->np) k_scatter<<<nb_of(B->np), kBlock, 0, ctx->st>>>(B->p, B->pidx, B->np, z);
        ctx->launches += 2;
        return DFL_OK;
    };
    rc = stage(B, B->b, rhs, B->n, ptr_kind, true);
    if (rc != DFL_OK) return block_err(B, rc);
    if (cudaEventRecord(ctx->ev0, ctx->st) != cudaSuccess) return DFL_E_CUDA;
    GmOut r;
    // solver.tol is absolute here: atol = tol ||b||, tol = 0 (schur.py:337-345)
    double bnorm = 0.0;
    rc = norm(B, B->outer, B->b, &bnorm);
    if (rc == DFL_OK)
        rc = gmres_any(B, B->outer, true, opA, &Msw, B->b, B->x, 0.0, prm->tol * bnorm, prm->maxiter, prm->restart, r);
    if (rc != DFL_OK) return block_err(B, rc);
    if (cudaEventRecord(ctx->ev1, ctx->st) != cudaSuccess) return DFL_E_CUDA;
    rc = stage(B, x, B->x, B->n, ptr_kind, false);
    if (rc != DFL_OK) return block_err(B, rc);
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    rep->iterations = r.iters;
    rep->converged = bnorm == 0.0 ? 1 : (r.converged ? 1 : 0);
    rep->solve_seconds = ms * 1e-3;
    rep->velocity_iterations = B->vel_its;
    rep->pressure_iterations = B->pre_its;
    rep->kernel_launches = ctx->launches;
    // true residual ||b - A x|| / ||b|| (schur.py:349-351), outside the timed span
    if (bnorm == 0.0) {
        rep->relative_residual = 0.0;
    } else {
        rc = spmv(B, B->A, B->x, B->outer.w);
        if (rc == DFL_OK) {
            k_sub<<<nb_of(B->n), kBlock, 0, ctx->st>>>(B->outer.r, B->b, B->outer.w, B->n);
            double rn = 0.0;
            rc = norm(B, B->outer, B->outer.r, &rn);
            rep->relative_residual = rn / bnorm;
        }
    }
    if (rc == DFL_OK && cudaGetLastError() != cudaSuccess) rc = DFL_E_CUDA;
    return block_err(B, rc);
}

}  // extern "C"
