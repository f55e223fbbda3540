// Preconditioner, operator and projector applications on the device, plus
// the timing / profiling entry points built on them.
#include "ctx_impl.cuh"

// ---------------------------------------------------------------------------
// V-cycle over all groups: z = M r  (deflation.py:239-250 -> amg.py:201-212).
// With dot_part != nullptr the last kernel of every group also emits the
// per-block partials of r.z; *nparts receives their count.
int vcycle(dfl_ctx *ctx, const double *r, double *z, const KState *st, double *dot_part, int64_t *nparts) {
    int64_t poff = 0;
    for (VGroup &g : ctx->groups) {
        const double *rin = r + g.row0;
        double *zout = z + g.row0;
        const int L = (int)g.lv.size();
        for (int l = 0; l < L; ++l) {
            DLevel &v = g.lv[l];
            const double *in = l == 0 ? rin : v.rv;
            double *next = (l + 1 < L) ? g.lv[l + 1].rv : g.rb;
            if (v.A.fmt == FMT_CODE || v.A.fmt == FMT_CLASS) {
                // w .* r formed at the gather
                RowArgs a{nullptr, v.w, in, nullptr, v.t, nullptr, st};
                launch_rows<MODE_RESID, false>(ctx, v.A, a);
            } else {
                RowArgs a{nullptr, v.w, in, nullptr, v.t, nullptr, st};
                launch_rows<MODE_RESID, false>(ctx, v.Aw, a);
            }
            prof_mark(ctx, "L" + std::to_string(l) + " resid");
            RowArgs b{v.t, nullptr, nullptr, nullptr, next, nullptr, st};
            launch_rows<MODE_PLAIN, false>(ctx, v.R, b);
            prof_mark(ctx, "L" + std::to_string(l) + " restrict");
        }
        {
            const double *rb = L == 0 ? rin : g.rb;
            double *xb = L == 0 ? zout : g.xb;
            launch_k(ctx->st, k_bottom, dim3((unsigned)cdiv(g.max_nb, 32), (unsigned)g.nsub), 256, 0, 
                g.binvT, g.binv_off, g.b_off, rb, xb, st);
            ctx->launches++;
            prof_mark(ctx, "bottom");
        }
        for (int l = L - 1; l >= 0; --l) {
            DLevel &v = g.lv[l];
            const double *in = l == 0 ? rin : v.rv;
            const double *e = (l + 1 < L) ? g.lv[l + 1].xv : g.xb;
            double *out = l == 0 ? zout : v.xv;
            RowArgs a{e, v.w, in, nullptr, v.t, nullptr, st};
            launch_rows<MODE_PROLONG, false>(ctx, v.P, a);
            prof_mark(ctx, "L" + std::to_string(l) + " prolong");
            if (l == 0 && dot_part) {
                RowArgs b{v.t, v.w, in, v.t, out, dot_part + poff, st};
                launch_rows<MODE_POST, true>(ctx, v.A, b);
                poff += parts_for(v.A);
            } else {
                RowArgs b{v.t, v.w, in, v.t, out, nullptr, st};
                launch_rows<MODE_POST, false>(ctx, v.A, b);
            }
            prof_mark(ctx, "L" + std::to_string(l) + " post");
        }
        if (L == 0 && dot_part) {
            // the group's finest level ran without a fused dot: explicit partials
            const int64_t rows = g.row1 - g.row0;
            const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(rows, kBlock), 64));
            launch_k(ctx->st, k_dot, nb, kBlock, 0, rin, zout, rows, dot_part + poff, st);
            ctx->launches++;
            poff += nb;
        }
    }
    if (nparts) *nparts = poff;
    return DFL_OK;
}

// y = A x (opmode 0) or y = b - A x (opmode 1); with zt the Z'y tile partials
int op_apply_dev(dfl_ctx *ctx, double *xin, double *y, int opmode, const double *b, bool zt,
                        const KState *st, int need_refresh) {
    OpArgs a{xin, b, y, ctx->zcols, ctx->n, zt ? ctx->k : 0, ctx->zt_part, st, need_refresh};
    if (ctx->zcode) {
        a.zcode = ctx->zcode;
        a.ztab = ctx->ztab;
        a.zs = ctx->zs;
        for (int c = 0; c < kKmax; ++c) a.ztab_off[c] = ctx->ztab_off[c];
    }
    if (!ctx->split) {
        RC(halo(ctx, xin));
        if (opmode == 0)
            launch_op<0>(ctx, a);
        else
            launch_op<1>(ctx, a);
        return DFL_OK;
    }
    // halo overlapped with the interior rows (runtime.py:283-292 split in two
    // passes): pack -> exchange on the comm stream while the rows without ghost
    // columns run, then the boundary rows
    RC(halo(ctx, xin, ctx->st2));
    a.skip_rows = ctx->bflag;
    if (opmode == 0)
        launch_op<0>(ctx, a);
    else
        launch_op<1>(ctx, a);
    if (!ctx->fab && multi(ctx) && !ctx->nbr.empty()) {  // the exchange ran on st2
        CK(cudaEventRecord(ctx->ev_halo, ctx->st2));
        CK(cudaStreamWaitEvent(ctx->st, ctx->ev_halo, 0));
    }
    a.skip_rows = nullptr;
    if (ctx->nbtiles > 0) {
        if (opmode == 0)
            launch_k(ctx->st, k_op_bnd<0>, (unsigned)ctx->nbtiles, kBlock, 0, ctx->Abnd, ctx->brows, ctx->bstart, ctx->bcnt,
                                                                         ctx->ntiles, a);
        else
            launch_k(ctx->st, k_op_bnd<1>, (unsigned)ctx->nbtiles, kBlock, 0, ctx->Abnd, ctx->brows, ctx->bstart, ctx->bcnt,
                                                                         ctx->ntiles, a);
        ctx->launches++;
    }
    return DFL_OK;
}

// out = project(v) = v - AZ E^-1 Z' v   (deflation.py:230-233)
int project_dev(dfl_ctx *ctx, const double *v, double *out, const KState *st, int dotmode, double *out2) {
    launch_k(ctx->st, k_zt_vec, (unsigned)ctx->ntiles, kBlock, 0, ctx->tiles, v, ctx->zcols, ctx->n, ctx->k, ctx->zt_part,
             zcode_of(ctx));
    ctx->launches++;
    RC(zt_to_t2(ctx, nullptr, 0, false));
    ProjArgs a = proj_args(ctx, v, out, st);
    a.dotmode = dotmode;
    a.dot_part = ctx->dpart;
    a.out2 = out2;
    launch_project<0>(ctx, a);
    return DFL_OK;
}

// x = y + Z E^-1 Z'(b - A y)   (deflation.py:285); y in ctx->x, x -> ctx->xin
int lift_dev(dfl_ctx *ctx, const dfl_solve_params *p) {
    if (p->deflated) {
        RC(op_apply_dev(ctx, ctx->x, ctx->tmp, 1, ctx->b, true, nullptr, 0));
        RC(zt_to_t2(ctx, nullptr, 0, true));
        launch_k(ctx->st, k_lift, (unsigned)ctx->ntiles, kBlock, 0, ctx->tiles, ctx->tile_sub, ctx->x, ctx->zcols, ctx->n,
                                                              ctx->k, ctx->t2, (int64_t)ctx->first_sub * ctx->k,
                                                              ctx->xin, 1, zcode_of(ctx));
    } else {
        launch_k(ctx->st, k_copy, (unsigned)ctx->nblk, kBlock, 0, ctx->xin, ctx->x, ctx->n);
    }
    ctx->launches++;
    return DFL_OK;
}

extern "C" {

int dfl_spmv_csr(const dfl_csr *A, const double *x, double *y, int device) {
    dfl_ctx *ctx = nullptr;
    RC(dfl_ctx_create(device, &ctx));
    std::unique_ptr<dfl_ctx, void (*)(dfl_ctx *)> guard(ctx, dfl_ctx_destroy);
    DMat m;
    HostRows h{A->nrows, A->ncols, A->row_ptr, A->col_idx, A->values};
    int rc = upload_matrix(ctx, h, m, {0, A->nrows});
    if (rc != DFL_OK) {
        dfl::set_setup_error(ctx->err);
        return rc;
    }
    double *dx, *dy;
    RC(upload(ctx, &dx, x, A->ncols));
    RC(dalloc(ctx, &dy, A->nrows));
    RowArgs a{dx, nullptr, nullptr, nullptr, dy, nullptr, nullptr};
    launch_rows<MODE_PLAIN, false>(ctx, m, a);
    cudaError_t e = cudaMemcpyAsync(y, dy, sizeof(double) * A->nrows, cudaMemcpyDeviceToHost, ctx->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    if (e != cudaSuccess) {
        dfl::set_setup_error(cudaGetErrorString(e));
        return DFL_E_CUDA;
    }
    return DFL_OK;
}

// algorithmic bytes: CSR with fp64 values / int32 indices,
// every vector read once and written once per kernel
int dfl_ctx_time(dfl_ctx *ctx, int what_flags, int reps, double *ms, double *bytes) {
    RC(ready(ctx));
    if (reps < 1) reps = 1;
    const bool flush = (what_flags & DFL_TIME_FLUSH_L2) != 0;
    const bool fmt_bytes = (what_flags & DFL_TIME_FORMAT_BYTES) != 0;
    const int what = what_flags & 0xff;
    auto run = [&]() -> int {
        if (what == 0) return op_apply_dev(ctx, ctx->p, ctx->w, 0, nullptr, false, nullptr, 0);
        if (what == 1 || what == 2) return vcycle(ctx, ctx->r, ctx->z, nullptr, nullptr, nullptr);
        if (what == 4) return op_apply_dev(ctx, ctx->p, ctx->w, 0, nullptr, ctx->deflation, nullptr, 0);
        if (what == 5) {  // q = w - AZ t2 with the fused p.q partials (the CG projection)
            ProjArgs a = proj_args(ctx, ctx->w, ctx->tmp, nullptr);
            a.dotmode = 1;
            a.dotv = ctx->p;
            a.dot_part = ctx->dpart;
            launch_project<0>(ctx, a);
            return DFL_OK;
        }
        if (what == 6 && !ctx->groups.empty() && !ctx->groups[0].lv.empty()) {
            VGroup &g = ctx->groups[0];
            double *next = g.lv.size() > 1 ? g.lv[1].rv : g.rb;
            RowArgs b{g.lv[0].t, nullptr, nullptr, nullptr, next, nullptr, nullptr};
            launch_rows<MODE_PLAIN, false>(ctx, g.lv[0].R, b);
            return DFL_OK;
        }
        ctx->err = "unknown timing target";
        return DFL_E_CONFIG;
    };
    // bytes the stored format must move for one pass over M
    auto mat = [](const DMat &M) -> double {
        const double rows = (double)M.nrows;
        if (M.fmt == FMT_CODE) return 8.0 * rows;
        if (M.fmt == FMT_CLASS) return 1.0 * rows;
        if (M.fmt == FMT_PCODE) return (M.pc_wide ? 24.0 : 20.0) * rows;
        if (M.fmt == FMT_CSR) return 12.0 * (double)M.nnz + 4.0 * (rows + 1);
        return 12.0 * (double)M.stored + (M.perm ? 4.0 * rows : 0.0) +
               (M.ell_w ? 0.0 : 8.0 * (rows / 32 + 1));
    };
    if ((what == 0 || what == 4) && fmt_bytes) {
        // the stored layout's bytes: each stored matrix byte once, x read once, y written once
        *bytes = mat(ctx->Aop) + 8.0 * (ctx->n + ctx->n_ghost) + 8.0 * ctx->n;
        if (what == 4 && ctx->deflation) {  // Z columns 1..k-1: dictionary indices + tables, or dense
            *bytes += ctx->zcode ? 2.0 * ctx->zs * ctx->n + 8.0 * ctx->ztab_n : 8.0 * (ctx->k - 1) * ctx->n;
        }
    } else if (what == 0 || what == 4) {
        *bytes = 12.0 * ctx->op_nnz + 4.0 * (ctx->n + 1) + 8.0 * (ctx->n + ctx->n_ghost) + 8.0 * ctx->n;
        if (what == 4 && ctx->deflation) *bytes += 8.0 * (ctx->k - 1) * ctx->n;  // Z columns 1..k-1
    } else if (what == 5 && fmt_bytes) {
        // w, p read, q written + the own-block AZ (dictionary indices + tables, or dense) + extras
        *bytes = 24.0 * ctx->n;
        if (ctx->deflation) {
            const int ks = ctx->k <= 1 ? 1 : ctx->k <= 2 ? 2 : ctx->k <= 4 ? 4 : 8;
            *bytes += ctx->acode ? 2.0 * ks * ctx->n + 8.0 * ctx->atab_n : 8.0 * ctx->k * ctx->n;
            if (ctx->ax_nnz) *bytes += 12.0 * ctx->ax_nnz + 4.0 * (ctx->n + 1);
        }
    } else if (what == 6) {
        if (ctx->groups.empty() || ctx->groups[0].lv.empty()) {
            ctx->err = "no smoothing level to time";
            return DFL_E_CONFIG;
        }
        const VGroup &g = ctx->groups[0];
        const DMat &R = g.lv[0].R;
        const double n = (double)g.rows[0], nc = (double)g.rows[1];
        // t read once, R t written once, plus R itself
        *bytes = (fmt_bytes ? mat(R) : 12.0 * (double)g.nnzP[0] + 4.0 * (nc + 1)) + 8.0 * n + 8.0 * nc;
    } else if (what == 5) {
        // w, p read, q written + AZ (CSR fp64/int32, as uploaded)
        *bytes = 24.0 * ctx->n + (ctx->deflation ? 12.0 * ctx->az_nnz + 4.0 * (ctx->n + 1) : 0.0);
    } else if (what == 2) {
        double b = 0;
        for (auto &g : ctx->groups) {
            for (size_t l = 0; l < g.lv.size(); ++l) {
                const DLevel &v = g.lv[l];
                const double n = (double)g.rows[l], nc = (double)g.rows[l + 1];
                b += (v.A.fmt == FMT_CODE || v.A.fmt == FMT_CLASS) ? 24.0 * n + mat(v.A) + 24.0 * n : mat(v.Aw) + 24.0 * n;  // residual
                b += mat(v.R) + 8.0 * n + 8.0 * nc;                                                // restriction
                b += mat(v.P) + 8.0 * nc + 24.0 * n;                                               // prolongation
                b += mat(v.A) + 40.0 * n;                                                          // post-smoothing
            }
            b += 8.0 * (double)g.nb * (double)g.nb / std::max(1, g.nsub) + 16.0 * (double)g.nb;
        }
        *bytes = b;
    } else {
        double b = 0;
        for (auto &g : ctx->groups) {
            for (size_t l = 0; l < g.lv.size(); ++l) {
                const double n = (double)g.rows[l], nc = (double)g.rows[l + 1];
                b += 24.0 * g.nnzA[l] + 24.0 * g.nnzP[l] + 100.0 * n + 20.0 * nc;
            }
            b += 8.0 * (double)g.nb * (double)g.nb / std::max(1, g.nsub);
        }
        *bytes = b;
    }
    // fill the inputs with something finite
    launch_k(ctx->st, k_fill, (unsigned)cdiv(ctx->n + ctx->n_ghost, kBlock), kBlock, 0, ctx->p, 1.0, ctx->n + ctx->n_ghost);
    launch_k(ctx->st, k_fill, (unsigned)ctx->nblk, kBlock, 0, ctx->r, 1.0, ctx->n);
    launch_k(ctx->st, k_fill, (unsigned)ctx->nblk, kBlock, 0, ctx->w, 1.0, ctx->n);
    if (what == 6) {
        const VGroup &g = ctx->groups[0];
        launch_k(ctx->st, k_fill, (unsigned)cdiv(g.rows[0], kBlock), kBlock, 0, g.lv[0].t, 1.0, g.rows[0]);
    }
    if (what == 3) {  // the V-cycle as the solve runs it: captured once, replayed as a CUDA graph
        double b = 0;
        double tmp = 0;
        RC(dfl_ctx_time(ctx, 1, 1, &tmp, &b));
        *bytes = b;
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
        const int64_t before = ctx->launches;
        int rc = vcycle(ctx, ctx->r, ctx->z, nullptr, nullptr, nullptr);
        CK(cudaStreamEndCapture(ctx->st, &g));
        ctx->launches = before;
        if (rc != DFL_OK) return rc;
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(ge, ctx->st));
        CK(cudaEventRecord(ctx->ev0, ctx->st));
        for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, ctx->st));
        CK(cudaEventRecord(ctx->ev1, ctx->st));
        CK(cudaEventSynchronize(ctx->ev1));
        float t = 0;
        CK(cudaEventElapsedTime(&t, ctx->ev0, ctx->ev1));
        *ms = t / reps;
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        return DFL_OK;
    }
    for (int i = 0; i < 3; ++i) RC(run());
    if (flush) {
        // cold L2 before every launch: write a buffer twice the L2 size, then
        // time the launch alone between its own pair of events
        const size_t fb = (size_t)256 << 20;
        void *buf = nullptr;
        CK(cudaMalloc(&buf, fb));
        double tot = 0.0;
        for (int i = 0; i < reps; ++i) {
            CK(cudaMemsetAsync(buf, i & 0xff, fb, ctx->st));
            CK(cudaEventRecord(ctx->ev0, ctx->st));
            const int rc = run();
            CK(cudaEventRecord(ctx->ev1, ctx->st));
            if (rc != DFL_OK) {
                cudaStreamSynchronize(ctx->st);
                cudaFree(buf);
                return rc;
            }
            CK(cudaEventSynchronize(ctx->ev1));
            float t = 0;
            CK(cudaEventElapsedTime(&t, ctx->ev0, ctx->ev1));
            tot += t;
        }
        CK(cudaFree(buf));
        *ms = tot / reps;
        return DFL_OK;
    }
    CK(cudaEventRecord(ctx->ev0, ctx->st));
    for (int i = 0; i < reps; ++i) RC(run());
    CK(cudaEventRecord(ctx->ev1, ctx->st));
    CK(cudaEventSynchronize(ctx->ev1));
    float t = 0;
    CK(cudaEventElapsedTime(&t, ctx->ev0, ctx->ev1));
    *ms = t / reps;
    return DFL_OK;
}

// per-launch device times of one V-cycle (mean over reps), labels "L<l> <stage>"
int dfl_ctx_profile_vcycle(dfl_ctx *ctx, int reps, int cap, double *ms, char *labels /* cap x 32 */) {
    RC(ready(ctx));
    if (reps < 1) reps = 1;
    launch_k(ctx->st, k_fill, (unsigned)ctx->nblk, kBlock, 0, ctx->r, 1.0, ctx->n);
    RC(vcycle(ctx, ctx->r, ctx->z, nullptr, nullptr, nullptr));
    std::vector<double> acc;
    int count = 0;
    for (int rep = 0; rep < reps; ++rep) {
        ctx->prof_on = true;
        ctx->prof_n = 0;
        prof_mark(ctx, "start");
        RC(vcycle(ctx, ctx->r, ctx->z, nullptr, nullptr, nullptr));
        ctx->prof_on = false;
        CK(cudaStreamSynchronize(ctx->st));
        count = (int)ctx->prof_n - 1;
        acc.resize(count, 0.0);
        for (int i = 0; i < count; ++i) {
            float t = 0;
            CK(cudaEventElapsedTime(&t, ctx->prof_ev[i], ctx->prof_ev[i + 1]));
            acc[i] += t;
        }
    }
    for (int i = 0; i < count && i < cap; ++i) {
        ms[i] = acc[i] / reps;
        std::snprintf(labels + 32 * i, 32, "%s", ctx->prof_lab[i + 1].c_str());
    }
    return std::min(count, cap);
}

}  // extern "C"
