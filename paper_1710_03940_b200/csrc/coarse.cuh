// The coarse end of the V-cycle in ONE persistent cooperative kernel.
//
// Below ~64K rows a level's kernels are latency bound (a few us of work,
// launch + drain dominate).  k_coarse_cycle runs every stage of the levels
// [lc, L) -- pre-smoothing residual, restriction, bottom solve, prolongation,
// post-smoothing -- separated by grid-wide barriers (cooperative launch: all
// CTAs co-resident), with the same per-row arithmetic as the stand-alone
// kernels (kernels.cuh), so results do not depend on where the split is.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace dfl {

// Vectors written earlier in the same (persistent / cluster) kernel are read
// through L2 (ld.global.cg) -- never through the non-coherent L1/texture path.
struct GatherCG {
    const double *x;
    __device__ __forceinline__ double operator()(int c) const { return __ldcg(x + c); }
};
struct GatherWRCG {
    const double *w, *r;
    __device__ __forceinline__ double operator()(int c) const { return mul_rn(__ldg(w + c), __ldcg(r + c)); }
};

template <int MODE>
__device__ __forceinline__ double epilogue_cg(const RowArgs &a, int64_t i, double ax) {
    if (MODE == MODE_PLAIN) return ax;
    if (MODE == MODE_RESID) return sub_rn(__ldcg(a.r + i), ax);
    if (MODE == MODE_PROLONG) return add_rn(mul_rn(__ldg(a.w + i), __ldcg(a.r + i)), ax);
    return add_rn(__ldcg(a.xo + i), mul_rn(__ldg(a.w + i), sub_rn(__ldcg(a.r + i), ax)));
}

constexpr int kMaxCoarse = 16;

struct CLevel {
    DMat A, Aw, P, R;
    const double *w;
    double *rv;  // level rhs (nullptr for the first handled level: uses CoarseArgs::rin)
    double *t;
    double *xv;  // level solution (first handled level: CoarseArgs::xout)
};

struct CoarseArgs {
    int nlev;                      // smoothing levels handled
    CLevel lv[kMaxCoarse];
    // bottom (row-major inverses, one per subdomain of the group)
    const double *binv;
    const int64_t *binv_off;
    const int64_t *b_off;
    int nsub;
    int64_t nb;
    double *rb;                    // bottom rhs (nlev > 0)
    double *xb;                    // bottom solution (nlev > 0)
};

// rows of A distributed over the whole grid: G lanes per row (G == 0: ELL,
// one thread per storage slot)
template <int MODE, int G>
__device__ __forceinline__ void grid_rows(const DMat &A, const RowArgs &a, int64_t gtid, int64_t gthreads) {
    if (G == 0) {
        for (int64_t j = gtid; j < A.nrows; j += gthreads) {
            const int64_t i = A.perm ? (int64_t)__ldg(A.perm + j) : j;
            const double ax = ell_row(A, j, GatherCG{MODE == MODE_RESID ? a.r : a.x});
            a.out[i] = epilogue_cg<MODE>(a, i, ax);
        }
    } else {
        constexpr int GG = G > 0 ? G : 1;
        constexpr int RPW = 32 / GG;
        const int lane = (int)(gtid & 31);
        const int64_t warp = gtid >> 5, nwarps = gthreads >> 5;
        // the loop bound is uniform per warp (shuffles inside csr_row need all lanes)
        for (int64_t wr = warp * RPW; wr < A.nrows; wr += nwarps * RPW) {
            const int64_t row = wr + lane / GG;
            const double ax = csr_row<GG>(A, row, lane % GG, GatherCG{MODE == MODE_RESID ? a.r : a.x});
            if (lane % GG == 0 && row < A.nrows) a.out[row] = epilogue_cg<MODE>(a, row, ax);
        }
    }
}

template <int MODE>
__device__ __forceinline__ void grid_stage(const DMat &A, const RowArgs &a, int64_t gtid, int64_t gthreads) {
    if (A.fmt == FMT_CODE) {  // code table read through L1; RESID gathers w_j * r_j on the fly
        for (int64_t i = gtid; i < A.nrows; i += gthreads) {
            const double ax = MODE == MODE_RESID
                                  ? code_row_g(A, i, GatherWRCG{a.w, a.r}, A.ctab_delta, A.ctab_val)
                                  : code_row_g(A, i, GatherCG{a.x}, A.ctab_delta, A.ctab_val);
            a.out[i] = epilogue_cg<MODE>(a, i, ax);
        }
        return;
    }
    if (A.fmt == FMT_ELL) {
        grid_rows<MODE, 0>(A, a, gtid, gthreads);
        return;
    }
    switch (A.group) {
        case 1: grid_rows<MODE, 1>(A, a, gtid, gthreads); break;
        case 2: grid_rows<MODE, 2>(A, a, gtid, gthreads); break;
        case 4: grid_rows<MODE, 4>(A, a, gtid, gthreads); break;
        case 8: grid_rows<MODE, 8>(A, a, gtid, gthreads); break;
        case 16: grid_rows<MODE, 16>(A, a, gtid, gthreads); break;
        default: grid_rows<MODE, 32>(A, a, gtid, gthreads); break;
    }
}

// bottom: one warp per row, lanes over the row of the row-major inverse
__device__ __forceinline__ void grid_bottom(const CoarseArgs &c, const double *rb, double *xb, int64_t gtid,
                                            int64_t gthreads) {
    const int lane = (int)(gtid & 31);
    const int64_t nw = gthreads >> 5;
    for (int64_t gr = gtid >> 5; gr < c.nb; gr += nw) {
        int s = 0;
        while (s + 1 < c.nsub && c.b_off[s + 1] <= gr) ++s;
        const int64_t o = c.b_off[s];
        const int n = (int)(c.b_off[s + 1] - o);
        const int i = (int)(gr - o);
        const double *M = c.binv + c.binv_off[s] + (int64_t)i * n;
        double acc = 0.0;
        for (int j = lane; j < n; j += 32) acc = fma(__ldg(M + j), __ldcg(rb + o + j), acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) xb[gr] = acc;
    }
}

// rin / xout: rhs and solution of the first handled level (the caller's
// vectors when the whole cycle runs here)
static __global__ void __launch_bounds__(256) k_coarse_cycle(const CoarseArgs *__restrict__ cp, const double *rin,
                                                      double *xout) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const CoarseArgs &c = *cp;
    const double *rb = c.nlev ? c.rb : rin;
    double *xb = c.nlev ? c.xb : xout;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
    for (int l = 0; l < c.nlev; ++l) {
        const CLevel &v = c.lv[l];
        const double *in = l == 0 ? rin : v.rv;
        double *next = (l + 1 < c.nlev) ? c.lv[l + 1].rv : c.rb;
        grid_stage<MODE_RESID>(v.Aw, RowArgs{nullptr, v.w, in, nullptr, v.t, nullptr, nullptr}, gtid, gthreads);
        grid.sync();
        grid_stage<MODE_PLAIN>(v.R, RowArgs{v.t, nullptr, nullptr, nullptr, next, nullptr, nullptr}, gtid, gthreads);
        grid.sync();
    }
    grid_bottom(c, rb, xb, gtid, gthreads);
    for (int l = c.nlev - 1; l >= 0; --l) {
        grid.sync();
        const CLevel &v = c.lv[l];
        const double *in = l == 0 ? rin : v.rv;
        const double *e = (l + 1 < c.nlev) ? c.lv[l + 1].xv : xb;
        double *out = l == 0 ? xout : v.xv;
        grid_stage<MODE_PROLONG>(v.P, RowArgs{e, v.w, in, nullptr, v.t, nullptr, nullptr}, gtid, gthreads);
        grid.sync();
        grid_stage<MODE_POST>(v.A, RowArgs{v.t, v.w, in, v.t, out, nullptr, nullptr}, gtid, gthreads);
    }
}

}  // namespace dfl

namespace dfl {
// ---------------------------------------------------------------------------
// The tiny end of the V-cycle (levels of <= kTinyRows rows and the bottom) in
// ONE thread-block cluster: 8 CTAs x 1024 threads, stages separated by the
// hardware cluster barrier.  Every tiny-level matrix is CSR; one warp per row
// (lanes stride the row, shuffle reduction), the bottom one warp per row of
// the row-major inverse.  Replaces 4 launches per tiny level + the bottom.
constexpr int kTinyRows = 4096;
constexpr int kTinyCtas = 8;
constexpr int kTinyThreads = 1024;

template <int MODE>
__device__ __forceinline__ void tiny_stage(const DMat &A, const RowArgs &a, int gwarp, int nwarps, int lane) {
    const double *xg = MODE == MODE_RESID ? a.r : a.x;
    for (int64_t row = gwarp; row < A.nrows; row += nwarps) {
        double acc = 0.0;
        const int b = __ldg(A.ptr + row), e = __ldg(A.ptr + row + 1);
        for (int k = b + lane; k < e; k += 32) acc += __ldg(A.val + k) * __ldcg(xg + __ldg(A.col + k));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.out[row] = epilogue_cg<MODE>(a, row, acc);
    }
}

static __global__ void __cluster_dims__(kTinyCtas, 1, 1) __launch_bounds__(kTinyThreads)
    k_tiny_cycle(const CoarseArgs *__restrict__ cp, const double *rin, double *xout) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const CoarseArgs &c = *cp;
    const int lane = threadIdx.x & 31;
    const int gwarp = (int)(blockIdx.x * (kTinyThreads / 32) + (threadIdx.x >> 5));
    const int nwarps = (int)(gridDim.x * (kTinyThreads / 32));
    const double *rb = c.nlev ? c.rb : rin;
    double *xb = c.nlev ? c.xb : xout;
    for (int l = 0; l < c.nlev; ++l) {
        const CLevel &v = c.lv[l];
        const double *in = l == 0 ? rin : v.rv;
        double *next = (l + 1 < c.nlev) ? c.lv[l + 1].rv : c.rb;
        tiny_stage<MODE_RESID>(v.Aw, RowArgs{nullptr, v.w, in, nullptr, v.t, nullptr, nullptr}, gwarp, nwarps, lane);
        cluster.sync();
        tiny_stage<MODE_PLAIN>(v.R, RowArgs{v.t, nullptr, nullptr, nullptr, next, nullptr, nullptr}, gwarp, nwarps, lane);
        cluster.sync();
    }
    // bottom: warp per row of the row-major inverse
    for (int64_t gr = gwarp; gr < c.nb; gr += nwarps) {
        int s = 0;
        while (s + 1 < c.nsub && c.b_off[s + 1] <= gr) ++s;
        const int64_t o = c.b_off[s];
        const int n = (int)(c.b_off[s + 1] - o);
        const double *M = c.binv + c.binv_off[s] + (gr - o) * n;
        double acc = 0.0;
        for (int j = lane; j < n; j += 32) acc = fma(__ldg(M + j), __ldcg(rb + o + j), acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) xb[gr] = acc;
    }
    for (int l = c.nlev - 1; l >= 0; --l) {
        cluster.sync();
        const CLevel &v = c.lv[l];
        const double *in = l == 0 ? rin : v.rv;
        const double *e = (l + 1 < c.nlev) ? c.lv[l + 1].xv : xb;
        double *out = l == 0 ? xout : v.xv;
        tiny_stage<MODE_PROLONG>(v.P, RowArgs{e, v.w, in, nullptr, v.t, nullptr, nullptr}, gwarp, nwarps, lane);
        cluster.sync();
        tiny_stage<MODE_POST>(v.A, RowArgs{v.t, v.w, in, v.t, out, nullptr, nullptr}, gwarp, nwarps, lane);
    }
}

}  // namespace dfl
