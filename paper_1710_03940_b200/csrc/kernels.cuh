// sm_100a kernels of the B200 solve phase.
//
// Everything here is HBM-bandwidth bound sparse / vector work in fp64 with
// int32 indices (no stage is a dense contraction, so no tensor cores).
// Matrix storage:
//   * sliced ELL, 32-row slices stored column-major inside the slice: one
//     thread per row, each warp-wide load of a slice column is 256 B of
//     values / 128 B of indices, fully coalesced; rows keep the reference's
//     CSR entry order and are summed sequentially with separate multiply and
//     add (no FMA), so ELL SpMV is bit-identical to _kernels.pyx:11-23.
//   * CSR-vector for long / irregular rows (coarse A, restriction R): a
//     sub-warp of G lanes per row and a shuffle tree (deterministic, but not
//     the reference's sequential order).
// Matrix streams are read with evict-first (ld.global.cs) so the gathered
// vectors stay resident in the 126 MB L2; gathers use the read-only path.
//
// Fused epilogues implement the V(1,1) cycle of amg.py:201-212, the deflation
// projector of deflation.py:230-233 and the CG recurrences of krylov.py:95-145.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dfl {

constexpr int kBlock = 256;       // threads per block for row kernels
constexpr int kKmax = 8;          // max deflation columns per subdomain
constexpr int kEllUnroll = 8;     // slice widths up to this are fully unrolled
#ifndef DFL_ELL_BATCH
#define DFL_ELL_BATCH 8
#endif

enum { FMT_ELL = 0, FMT_CSR = 1, FMT_CODE = 2, FMT_CLASS = 3, FMT_PCODE = 4 };

// FMT_PCODE ("delta/value-coded rows"): matrices with <= 7 entries per row,
// column-sorted rows whose columns lie within 65535 of the row's first one and
// <= 15 distinct values -- the smoothed prolongation of a structured problem
// (150^3: 9 values, deltas <= 12597).  Per row, structure-of-arrays: the first
// column (int32), six 16-bit column deltas (3 x uint32) and one uint32 holding
// the length (3 bits) and seven 4-bit value codes; the value table (16
// doubles) is staged in shared memory.  20 bytes per row instead of 12 per
// ELL slot (72 at width 6); lossless, CSR order, no FMA: bit-identical.
constexpr int kPcMaxLen = 7;

// FMT_CLASS ("row-class coded"): one byte per row.  The most frequent row
// (the interior stencil: ordered (column - row, value) entries, <= 7) is the
// dominant row; a row whose entries are a subset of it (face / edge / corner
// rows of a structured-grid operator) is coded as 0x80 | presence mask, any
// other row as one of <= kMaxClass generic classes.  The table travels as a
// __grid_constant__ kernel parameter.  Lossless: a row is summed in its CSR
// order without FMA, bit-identical to spmv_rows.  The upload falls back to
// CODE / ELL when the rows do not fit.
constexpr int kMaxClass = 64;
struct ClassTab {
    int n;
    int lead;                  // largest column - row (leading gather edge)
    int dom;                   // unused (kept for the table layout)
    int dlen;                  // dominant row: <= 7 entries (offset, value), the rows
    int ddelta[8];             // that are subsets of it carry a presence mask
    double dval[8];
    int len[kMaxClass];
    int delta[kMaxClass][8];
    double val[kMaxClass][8];
};

// FMT_CODE ("stencil-coded ELL"): every row holds <= 8 one-byte codes; code c
// stands for the pair (column - row, value) of a per-matrix table of <= 255
// pairs (255 = padding).  Lossless for matrices with few distinct
// (offset, value) pairs -- structured-grid operators: the 7-point Poisson
// operator has 7 -- and 8 bytes per row instead of 12 per entry.
constexpr unsigned kCodePad = 255u;

struct DMat {
    int fmt = FMT_ELL;
    int ell_w = 0;            // > 0: every slice has this width (no slice_off lookup)
    int group = 1;            // CSR-vector lanes per row
    int64_t nrows = 0, ncols = 0, nnz = 0, stored = 0;
    const int64_t *slice_off = nullptr;  // ELL: nslices + 1 element offsets
    const int *ptr = nullptr;            // CSR row pointer
    const int *col = nullptr;
    const double *val = nullptr;
    const int *perm = nullptr;           // SELL-C-sigma: slot -> row (nullptr: identity)
    // FMT_CODE
    const uint2 *codes = nullptr;        // 8 codes per row, row-major
    int code_lead = 0;                   // largest column - row of the table (leading gather edge)
    // FMT_CLASS
    const uint8_t *cls = nullptr;        // class of every row
    int class_id = -1;                   // index of the ClassTab in the context
    // FMT_PCODE
    const int *pc_c0 = nullptr;          // first column of every row
    const uint32_t *pc_d = nullptr;      // 3 x nrows: 16-bit deltas of entries 1..6 (SoA)
    const uint32_t *pc_v = nullptr;      // length | 4-bit value codes << (3 + 4k)
    const double *pc_tab = nullptr;      // 16 values (wide: up to 256)
    int pc_wide = 0;                     // 8-bit value codes: pc_v = len | c0..c2 << 8.., pc_v + n = c3..c6
    const int *ctab_delta = nullptr;     // column - row of each code
    const double *ctab_val = nullptr;    // value of each code
    int ncodes = 0;
};

// run-time state of one Krylov solve (device resident)
struct KState {
    double bnorm, target;
    double rz, rz_new, alpha, beta, pq, rr, resnorm;
    int iters, done, converged, breakdown, maxiter, refresh_every, refresh_now, pad;
    // bicgstab2 scalars
    double rho0, rho1, omega, gamma_div;
    double brk_val;  // the scalar that broke down (p'Ap or r'z), for the report string
};

// Programmatic dependent launch: every kernel first waits for the grid it
// depends on (griddepcontrol.wait: full completion and memory flush of the
// previous kernel in the stream; a no-op when launched without the PDL
// attribute), so the launch of a kernel overlaps the drain of the one before
// it.  (An early launch_dependents trigger was measured slower for the
// V-cycle: 345 vs 324 us per graph, profiles/r01/README.md.)
#define DFL_PDL_ENTRY asm volatile("griddepcontrol.wait;" ::: "memory")

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

template <class T>
__device__ __forceinline__ T ld_stream(const T *p) { return __ldcs(p); }
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---------------------------------------------------------------------------
// gather functors: the value an entry multiplies
struct GatherX {
    const double *__restrict__ x;
    __device__ __forceinline__ double operator()(int c) const { return __ldg(x + c); }
    // entry at row + d, the row's base address formed once by the caller
    __device__ __forceinline__ double at(const GatherX &b, int d) const { return __ldg(b.x + d); }
    __device__ __forceinline__ GatherX shift(int64_t row) const { return GatherX{x + row}; }
};
// relaxation applied on the fly: (w * r)[c]  (amg.py:193/195 then matvec)
struct GatherWR {
    const double *__restrict__ w;
    const double *__restrict__ r;
    __device__ __forceinline__ double operator()(int c) const { return mul_rn(__ldg(w + c), __ldg(r + c)); }
    __device__ __forceinline__ double at(const GatherWR &b, int d) const {
        return mul_rn(__ldg(b.w + d), __ldg(b.r + d));
    }
    __device__ __forceinline__ GatherWR shift(int64_t row) const { return GatherWR{w + row, r + row}; }
};

// code table into shared memory (called by all threads of the block)
__device__ __forceinline__ void load_codes(const DMat &A, int *sd, double *sv) {
    for (int t = threadIdx.x; t < A.ncodes; t += blockDim.x) {
        sd[t] = A.ctab_delta[t];
        sv[t] = A.ctab_val[t];
    }
    __syncthreads();
}

// sum_k val(c_k) * g(row + delta(c_k)) in storage (= CSR) order, no FMA:
// bit-identical to spmv_rows
template <class G>
__device__ __forceinline__ double code_row_w(uint2 cw, int64_t row, const G &g, const int *sd, const double *sv) {
    unsigned c[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        c[k] = (cw.x >> (8 * k)) & 0xffu;
        c[k + 4] = (cw.y >> (8 * k)) & 0xffu;
    }
    double xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (c[k] != kCodePad) xv[k] = g((int)(row + sd[c[k]]));
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (c[k] != kCodePad) acc = add_rn(acc, mul_rn(sv[c[k]], xv[k]));
    return acc;
}

template <class G>
__device__ __forceinline__ double code_row_g(const DMat &A, int64_t row, const G &g, const int *sd, const double *sv) {
    return code_row_w(__ldcs(A.codes + row), row, g, sd, sv);
}

__device__ __forceinline__ double code_row(const DMat &A, int64_t row, const double *__restrict__ xg,
                                           const int *sd, const double *sv) {
    return code_row_g(A, row, GatherX{xg}, sd, sv);
}

// sequential, CSR-ordered row sum of an ELL row (bit-identical to spmv_rows)
template <class G>
__device__ __forceinline__ double ell_row(const DMat &A, int64_t row, const G &g) {
    const int64_t s = row >> 5;
    const int lane = (int)(row & 31);
    int64_t off;
    int width;
    if (A.ell_w > 0) {  // uniform slices: no dependent index load before the stream
        width = A.ell_w;
        off = s * 32 * (int64_t)width;
    } else {
        off = __ldg(A.slice_off + s);
        width = (int)((__ldg(A.slice_off + s + 1) - off) >> 5);
    }
    const int *cp = A.col + off + lane;
    const double *vp = A.val + off + lane;
    double acc = 0.0;
    if (width <= kEllUnroll) {
        int c[kEllUnroll];
        double v[kEllUnroll], xv[kEllUnroll];
#pragma unroll
        for (int k = 0; k < kEllUnroll; ++k)
            if (k < width) {
                c[k] = ld_stream(cp + 32 * k);
                v[k] = ld_stream(vp + 32 * k);
            }
#pragma unroll
        for (int k = 0; k < kEllUnroll; ++k)
            if (k < width) xv[k] = g(c[k]);
#pragma unroll
        for (int k = 0; k < kEllUnroll; ++k)
            if (k < width) acc = add_rn(acc, mul_rn(v[k], xv[k]));
    } else {
        constexpr int B = DFL_ELL_BATCH;
        for (int k0 = 0; k0 < width; k0 += B) {
            int c[B];
            double v[B], xv[B];
#pragma unroll
            for (int k = 0; k < B; ++k)
                if (k0 + k < width) {
                    c[k] = ld_stream(cp + 32 * (k0 + k));
                    v[k] = ld_stream(vp + 32 * (k0 + k));
                }
#pragma unroll
            for (int k = 0; k < B; ++k)
                if (k0 + k < width) xv[k] = g(c[k]);
#pragma unroll
            for (int k = 0; k < B; ++k)
                if (k0 + k < width) acc = add_rn(acc, mul_rn(v[k], xv[k]));
        }
    }
    return acc;
}

// ELL row with a compile-time uniform width W (the common case: every slice
// padded to the matrix's max row length)
template <int W, class G>
__device__ __forceinline__ double ell_row_w(const DMat &A, int64_t row, const G &g) {
    const int64_t off = (row >> 5) * 32 * W + (row & 31);
    const int *cp = A.col + off;
    const double *vp = A.val + off;
    int c[W];
    double v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        c[k] = ld_stream(cp + 32 * k);
        v[k] = ld_stream(vp + 32 * k);
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) acc = add_rn(acc, mul_rn(v[k], g(c[k])));
    return acc;
}

// sliced ELL, width known per slice: dispatch to a compile-time width so the
// register footprint is that of the widest case actually compiled (<= 8)
template <int W, class G>
__device__ __forceinline__ double ell_slice_w(const DMat &A, int64_t off, const G &g) {
    const int *cp = A.col + off;
    const double *vp = A.val + off;
    int c[W];
    double v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        c[k] = ld_stream(cp + 32 * k);
        v[k] = ld_stream(vp + 32 * k);
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) acc = add_rn(acc, mul_rn(v[k], g(c[k])));
    return acc;
}

#ifndef DFL_SLICE_CHUNK
#define DFL_SLICE_CHUNK 4
#endif
constexpr int kChunk = DFL_SLICE_CHUNK;  // entries of a sliced row whose loads are batched

// chunk of w <= kChunk entries of a sliced row, accumulated into acc in order
template <class G>
__device__ __forceinline__ double ell_chunk(const DMat &A, int64_t o, int w, double acc, const G &g) {
    // exact sequential order, fixed-width predicated batch
    int c[kChunk];
    double v[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k)
        if (k < w) {
            c[k] = ld_stream(A.col + o + 32 * k);
            v[k] = ld_stream(A.val + o + 32 * k);
        }
#pragma unroll
    for (int k = 0; k < kChunk; ++k)
        if (k < w) acc = add_rn(acc, mul_rn(v[k], g(c[k])));
    return acc;
}

template <class G>
__device__ __forceinline__ double ell_row_sliced(const DMat &A, int64_t row, const G &g) {
    const int64_t s = row >> 5;
    const int64_t off = __ldg(A.slice_off + s);
    const int width = (int)((__ldg(A.slice_off + s + 1) - off) >> 5);
    const int64_t o = off + (row & 31);
    double acc = 0.0;
    for (int k0 = 0; k0 < width; k0 += kChunk) {
        acc = ell_chunk(A, o + 32 * k0, min(kChunk, width - k0), acc, g);
    }
    return acc;
}

template <int W, class G>
__device__ __forceinline__ double ell_any(const DMat &A, int64_t row, const G &g) {
    if (W > 0) return ell_row_w<(W > 0 ? W : 1)>(A, row, g);
    return ell_row_sliced(A, row, g);  // slice_off is stored for uniform widths too
}

// CSR row by G lanes with the entry loads of a lane batched kCsrUnroll deep
// (all index/value loads in flight before the gathers); full sum returned on
// all G lanes.  G == 1 keeps the sequential CSR order (bit-identical to
// spmv_rows).
#ifndef DFL_ELL_BATCH
#define DFL_ELL_BATCH 8
#endif
#ifndef DFL_CSR_UNROLL
#define DFL_CSR_UNROLL 8
#endif
#ifndef DFL_CSR_MINB
#define DFL_CSR_MINB 4
#endif
constexpr int kCsrUnroll = DFL_CSR_UNROLL;

template <int G, class Gat>
__device__ __forceinline__ double csr_row(const DMat &A, int64_t row, int sub, const Gat &g) {
    double acc = 0.0;
    if (row < A.nrows) {
        const int b = __ldg(A.ptr + row), e = __ldg(A.ptr + row + 1);
        for (int k0 = b + sub; k0 < e; k0 += kCsrUnroll * G) {
            int c[kCsrUnroll];
            double v[kCsrUnroll], xv[kCsrUnroll];
#pragma unroll
            for (int u = 0; u < kCsrUnroll; ++u)
                if (k0 + u * G < e) {
                    c[u] = ld_stream(A.col + k0 + u * G);
                    v[u] = ld_stream(A.val + k0 + u * G);
                }
#pragma unroll
            for (int u = 0; u < kCsrUnroll; ++u)
                if (k0 + u * G < e) xv[u] = g(c[u]);
#pragma unroll
            for (int u = 0; u < kCsrUnroll; ++u)
                if (k0 + u * G < e) {
                    if (G == 1)
                        acc = add_rn(acc, mul_rn(v[u], xv[u]));
                    else
                        acc += v[u] * xv[u];
                }
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
    return acc;
}

// block-wide sum of NV values (deterministic tree), result valid in thread 0
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *smem /* 32*NV */) {
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(0xffffffffu, v[j], o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) smem[warp * NV + j] = v[j];
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            v[j] = lane < nw ? smem[lane * NV + j] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(0xffffffffu, v[j], o);
        }
    }
}

// Block sum of NV values per thread (NV a power of two <= 32) with a
// transposing warp butterfly: every halving step exchanges half of the
// values (NV/2 + NV/4 + ... shuffles instead of 5 NV), then the remaining
// xor steps reduce one value.  Fixed pattern, hence deterministic.  Returns
// the block total of value j in thread j (j < NV); other threads get 0.
template <int NV>
__device__ __forceinline__ double block_sum_t(double (&v)[NV], double *smem /* 32*NV */) {
    static_assert(NV >= 1 && NV <= 32 && (NV & (NV - 1)) == 0, "NV must be a power of two");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int col = 0;
#pragma unroll
    for (int st = 0; (NV >> st) > 1; ++st) {
        const int h = NV >> (st + 1), o = 16 >> st;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const double send = up ? v[j] : v[j + h];
            const double keep = up ? v[j + h] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
        if (up) col += h;
    }
    constexpr int kRest = 32 / NV;  // lanes that still hold the same column
#pragma unroll
    for (int o = kRest / 2; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    if ((lane & (kRest - 1)) == 0) smem[warp * NV + col] = v[0];
    __syncthreads();
    double tot = 0.0;
    if ((int)threadIdx.x < NV) {
        const int nw = blockDim.x >> 5;
        for (int q = 0; q < nw; ++q) tot += smem[q * NV + threadIdx.x];
    }
    return tot;
}

__device__ __forceinline__ bool skip(const KState *st) { return st != nullptr && st->done; }

// the CG scalar steps of krylov.py:119-143 (also used by the single-block
// kernels of ctx_cg.cu, which call them with the reduced value)
__device__ __forceinline__ void cg_step_pq(KState *st, double pq) {  // iters += 1; alpha
    st->iters += 1;
    st->pq = pq;
    if (pq <= 0.0 || !isfinite(pq)) {
        st->breakdown = DFL_BRK_CURVATURE;
        st->brk_val = pq;
        st->done = 1;
        return;
    }
    st->alpha = st->rz / pq;
    st->refresh_now = (st->iters % st->refresh_every) == 0;
}
__device__ __forceinline__ void cg_step_rr(KState *st, double rr) {  // convergence test
    st->rr = rr;
    st->resnorm = sqrt(fmax(rr, 0.0));
    if (st->resnorm <= st->target) {
        st->converged = 1;
        st->done = 1;
    }
}
__device__ __forceinline__ void cg_step_rz(KState *st, double rz) {  // beta
    if (rz == 0.0 || !isfinite(rz)) {
        st->breakdown = DFL_BRK_RZ;
        st->brk_val = rz;
        st->done = 1;
        return;
    }
    st->beta = rz / st->rz;
    st->rz = rz;
}

// end of a row / vector kernel with one dot partial per block (block_sum<1>
// result in thread 0's v)
__device__ __forceinline__ void dot_out(double *part, double v) {
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// ---------------------------------------------------------------------------
// V-cycle kernels (amg.py:201-212), one per fused stage.
//   RESID  : out = r - A (w .* r)                     (pre-smooth + residual)
//   POST   : out = x + w .* (r - A x)                 (post-smooth), opt. dot r.out
//   PROLONG: out = w .* r + P e                       (coarse correction)
//   PLAIN  : out = A x                                (restriction / operator)
enum { MODE_PLAIN = 0, MODE_RESID = 1, MODE_POST = 2, MODE_PROLONG = 3 };

struct RowArgs {
    const double *x;   // gathered vector (PLAIN / POST: x, PROLONG: e)
    const double *w;   // relaxation weights
    const double *r;   // right-hand side of the level
    const double *xo;  // POST: own x
    double *out;
    double *dot_part;  // POST: per-block r.out partials (nullptr: none)
    const KState *st;
};

template <int MODE>
__device__ __forceinline__ double epilogue(const RowArgs &a, int64_t i, double ax) {
    if (MODE == MODE_PLAIN) return ax;
    if (MODE == MODE_RESID) return sub_rn(__ldg(a.r + i), ax);
    if (MODE == MODE_PROLONG) return add_rn(mul_rn(__ldg(a.w + i), __ldg(a.r + i)), ax);
    // POST: x + w*(r - Ax)
    return add_rn(__ldg(a.xo + i), mul_rn(__ldg(a.w + i), sub_rn(__ldg(a.r + i), ax)));
}

// The row's own operands of the epilogue, loaded before the row's gathers
// (so their DRAM latency overlaps the gather chain instead of following it)
template <int MODE, bool DOT>
struct Own {
    double r = 0.0, w = 0.0, xo = 0.0;
    __device__ __forceinline__ void load(const RowArgs &a, int64_t i) {
        if (MODE != MODE_PLAIN || DOT) r = __ldg(a.r + i);
        if (MODE == MODE_POST || MODE == MODE_PROLONG) w = __ldg(a.w + i);
        if (MODE == MODE_POST) xo = __ldg(a.xo + i);
    }
    // epilogue<MODE> with the preloaded operands (same operation order)
    __device__ __forceinline__ double apply(double ax) const {
        if (MODE == MODE_PLAIN) return ax;
        if (MODE == MODE_RESID) return sub_rn(r, ax);
        if (MODE == MODE_PROLONG) return add_rn(mul_rn(w, r), ax);
        return add_rn(xo, mul_rn(w, sub_rn(r, ax)));
    }
};

// RESID runs on the pre-scaled matrix A diag(w) (values a_ij * w_j, built at
// upload), so it gathers r once per entry instead of w and r.
#ifndef DFL_ELL_MINB
#define DFL_ELL_MINB 1
#endif
#ifndef DFL_ELL_MINB0
#define DFL_ELL_MINB0 6
#endif
template <int MODE, bool DOT, int W>
__global__ void __launch_bounds__(kBlock, W == 0 ? DFL_ELL_MINB0 : DFL_ELL_MINB) k_ell(DMat A, RowArgs a) {
    DFL_PDL_ENTRY;
    double dot = 0.0;
    // one slot per thread; sliced matrices (W == 0) may run grid-stride over
    // one resident wave (launch_rows, DFL_SELL_WAVE)
    for (int64_t j = (int64_t)blockIdx.x * kBlock + threadIdx.x; j < A.nrows; j += (int64_t)gridDim.x * kBlock) {
        const int64_t i = (W == 0 && A.perm) ? (int64_t)__ldg(A.perm + j) : j;  // matrix row
        // short uniform rows: own operands first; long sliced rows (W == 0):
        // after the row, so they do not occupy registers through its chunks
        // (measured: L1 post 39.7 -> 43.6 us when loaded first)
        Own<MODE, DOT> own;
        if (W > 0) own.load(a, i);
        double ax;
        if (MODE == MODE_RESID)
            ax = ell_any<W>(A, j, GatherX{a.r});
        else
            ax = ell_any<W>(A, j, GatherX{a.x});
        if (W == 0) own.load(a, i);
        const double y = own.apply(ax);
        a.out[i] = y;
        if (DOT) dot += own.r * y;
    }
    if (DOT) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        dot_out(a.dot_part, v[0]);
    }
}

// FMT_CODE row kernel, software-pipelined: the codes and the own-row operands
// of the next row are loaded one iteration ahead, and the leading edge of its
// gathers (row + code_lead: data no earlier row has touched, hence a DRAM
// miss in the gather chain) is prefetched into L2, so a row's critical path
// is one L2 gather instead of DRAM (codes) + DRAM (first-touch gather).
template <int MODE, bool DOT>
__global__ void __launch_bounds__(kBlock) k_codep(DMat A, RowArgs a) {
    DFL_PDL_ENTRY;
    __shared__ int sd[256];
    __shared__ double sv[256];
    constexpr bool kR = MODE != MODE_PLAIN || DOT;  // needs r_i
    constexpr bool kPost = MODE == MODE_POST;       // needs w_i, x_i
    const bool wr = MODE == MODE_RESID && a.x == nullptr;
    const double *gx = wr ? a.r : a.x;
    const int64_t n = A.nrows, ncols = A.ncols;
    const int64_t stride = (int64_t)gridDim.x * kBlock;
    int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    uint2 cw = make_uint2(~0u, ~0u);
    double ri = 0.0, wi = 0.0, xi = 0.0;
    if (i < n) {
        cw = __ldcs(A.codes + i);
        if (kR) ri = __ldg(a.r + i);
        if (kPost) {
            wi = __ldg(a.w + i);
            xi = __ldg(a.xo + i);
        }
        const int64_t pe = min(i + (int64_t)A.code_lead, ncols - 1);
        prefetch_l2(gx + pe);
        if (wr) prefetch_l2(a.w + pe);
    }
    load_codes(A, sd, sv);
    double dot = 0.0;
    for (; i < n; i += stride) {
        const int64_t in = i + stride;
        uint2 cn = make_uint2(~0u, ~0u);
        double rn = 0.0, wn = 0.0, xn = 0.0;
        if (in < n) {
            cn = __ldcs(A.codes + in);
            if (kR) rn = __ldg(a.r + in);
            if (kPost) {
                wn = __ldg(a.w + in);
                xn = __ldg(a.xo + in);
            }
            const int64_t pe = min(in + (int64_t)A.code_lead, ncols - 1);
            prefetch_l2(gx + pe);
            if (wr) prefetch_l2(a.w + pe);
        }
        const double ax = wr ? code_row_w(cw, i, GatherWR{a.w, a.r}, sd, sv) : code_row_w(cw, i, GatherX{a.x}, sd, sv);
        double y;
        if (MODE == MODE_PLAIN) y = ax;
        else if (MODE == MODE_RESID) y = sub_rn(ri, ax);
        else if (MODE == MODE_POST) y = add_rn(xi, mul_rn(wi, sub_rn(ri, ax)));
        else y = epilogue<MODE>(a, i, ax);
        a.out[i] = y;
        if (DOT) dot += ri * y;
        cw = cn;
        ri = rn;
        wi = wn;
        xi = xn;
    }
    if (DOT) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        dot_out(a.dot_part, v[0]);
    }
}

// one row of a FMT_CLASS matrix, CSR order, no FMA.  Row byte c:
//   c >= 0x80: the row is a subset of the dominant row (the interior stencil)
//              -- bit k of c says whether its entry k is present; offsets and
//              values are compile-time offsets into the grid-constant table
//              (constant-bank operands), so the warp runs one predicated
//              stream whatever mix of interior / face / edge rows it holds;
//   c <  0x80: generic class id (rows that are not such subsets), summed by a
//              separate out-of-line loop.
template <class G>
__device__ __forceinline__ double class_row_slow(const ClassTab &T, int c, int64_t row, const G &g) {
    double acc = 0.0;
#pragma unroll 1
    for (int k = 0; k < T.len[c]; ++k) acc = add_rn(acc, mul_rn(T.val[c][k], g((int)(row + T.delta[c][k]))));
    return acc;
}

// Dominant-row path: absent entries load nothing and contribute
// dval * 0.0 = +-0, which leaves the running sum unchanged bit for bit (the sum
// starts at +0 and round-to-nearest never produces -0 from it), so the sum
// equals the CSR sum over the present entries without a select per entry;
// the host keeps the path only for finite dominant values.  Unused table
// slots (k >= dlen) hold 0.
template <class G>
__device__ __forceinline__ double class_row(const ClassTab &T, int c, int64_t row, const G &g) {
    if (c & 0x80) {
        const G gr = g.shift(row);
        double xv[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) xv[k] = ((c >> k) & 1) ? g.at(gr, T.ddelta[k]) : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 7; ++k) acc = add_rn(acc, mul_rn(T.dval[k], xv[k]));
        return acc;
    }
    return class_row_slow(T, c, row, g);
}

// rows per thread of the class-coded row kernels (k_class1, k_op_class) and
// their resident blocks per SM (DFL_OPCLASS2_MINB: 16 x 128 threads)
#ifndef DFL_OP_RPT
#define DFL_OP_RPT 2
#endif
constexpr int kOpRpt = DFL_OP_RPT;
#ifndef DFL_OPCLASS2_MINB
#define DFL_OPCLASS2_MINB 16
#endif

// FMT_CLASS row kernel (V-cycle stages): one block per kBlock rows, RPT rows
// per thread (rows i0, i0 + kBlock / RPT, ...; k_op_class's layout), so the
// per-thread fixed cost is paid once per RPT rows and their loads are in
// flight together; the next wave's first DRAM touches (class byte, leading
// gather edge) are prefetched into L2 (pf rows ahead).  Own-row operands are
// loaded before the gathers.  DOT: one partial per block.
template <int MODE, bool DOT, int RPT = kOpRpt>
__global__ void __launch_bounds__(kBlock / RPT, DFL_OPCLASS2_MINB) k_class1(DMat A, RowArgs a,
                                                                           const __grid_constant__ ClassTab T,
                                                                           int64_t pf) {
    DFL_PDL_ENTRY;
    constexpr int TB = kBlock / RPT;
    constexpr bool kR = MODE != MODE_PLAIN || DOT;
    constexpr bool kPost = MODE == MODE_POST;
    const bool wr = MODE == MODE_RESID && a.x == nullptr;
    const int64_t n = A.nrows;
    const int64_t i0 = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (pf > 0) {
        const int64_t ip = i0 + pf;
        if (ip < n) {
            prefetch_l2(A.cls + ip);
            const int64_t pe = min(ip + (int64_t)T.lead, A.ncols - 1);
            prefetch_l2((wr ? a.r : a.x) + pe);
            if (wr) prefetch_l2(a.w + pe);
        }
    }
    int c[RPT];
    double ri[RPT], wi[RPT], xi[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t i = i0 + u * TB;
        const bool valid = i < n;
        c[u] = valid ? (int)__ldcs(A.cls + i) : 0;
        ri[u] = (kR && valid) ? __ldg(a.r + i) : 0.0;
        wi[u] = (kPost && valid) ? __ldg(a.w + i) : 0.0;
        xi[u] = (kPost && valid) ? __ldg(a.xo + i) : 0.0;
    }
    double dot = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t i = i0 + u * TB;
        if (i < n) {
            const double ax = wr ? class_row(T, c[u], i, GatherWR{a.w, a.r}) : class_row(T, c[u], i, GatherX{a.x});
            double y;
            if (MODE == MODE_PLAIN) y = ax;
            else if (MODE == MODE_RESID) y = sub_rn(ri[u], ax);
            else if (MODE == MODE_POST) y = add_rn(xi[u], mul_rn(wi[u], sub_rn(ri[u], ax)));
            else y = epilogue<MODE>(a, i, ax);
            a.out[i] = y;
            if (DOT) dot += ri[u] * y;
        }
    }
    if (DOT) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        dot_out(a.dot_part, v[0]);
    }
}

// FMT_PCODE row kernel: one row per thread.  WIDE: 8-bit value codes (a
// second code word per row, the table of <= 256 values read through L1)
template <int MODE, bool DOT, bool WIDE = false>
__global__ void __launch_bounds__(kBlock) k_pcode(DMat A, RowArgs a) {
    DFL_PDL_ENTRY;
    __shared__ double tab[16];
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const bool valid = i < A.nrows;
    int c0 = 0;
    uint32_t d0 = 0, d1 = 0, d2 = 0, vw = 0, vw2 = 0;
    Own<MODE, DOT> own;
    if (valid) {
        own.load(a, i);
        c0 = __ldcs(A.pc_c0 + i);
        vw = __ldcs(A.pc_v + i);
        if (WIDE) vw2 = __ldcs(A.pc_v + A.nrows + i);
        d0 = __ldcs(A.pc_d + i);
        d1 = __ldcs(A.pc_d + A.nrows + i);
        d2 = __ldcs(A.pc_d + 2 * A.nrows + i);
    }
    if (!WIDE) {
        if (threadIdx.x < 16) tab[threadIdx.x] = A.pc_tab[threadIdx.x];
        __syncthreads();
    }
    double dot = 0.0;
    if (valid) {
        const int len = (int)(vw & 7u);
        const uint32_t dl[3] = {d0, d1, d2};
        const double *x = MODE == MODE_RESID ? a.r : a.x;
        double xv[kPcMaxLen];
#pragma unroll
        for (int k = 0; k < kPcMaxLen; ++k)
            if (k < len) {
                const int col = k == 0 ? c0 : c0 + (int)((dl[(k - 1) >> 1] >> (16 * ((k - 1) & 1))) & 0xffffu);
                xv[k] = __ldg(x + col);
            }
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < kPcMaxLen; ++k)
            if (k < len) {
                const double vk = WIDE ? __ldg(A.pc_tab + ((k < 3 ? vw >> (8 * (k + 1)) : vw2 >> (8 * (k - 3))) & 0xffu))
                                       : tab[(vw >> (3 + 4 * k)) & 0xfu];
                acc = add_rn(acc, mul_rn(vk, xv[k]));
            }
        const double y = own.apply(acc);
        a.out[i] = y;
        if (DOT) dot = own.r * y;
    }
    if (DOT) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        dot_out(a.dot_part, v[0]);
    }
}

template <int G, int MODE, bool DOT>
__global__ void __launch_bounds__(kBlock, DFL_CSR_MINB) k_csr(DMat A, RowArgs a) {
    DFL_PDL_ENTRY;
    constexpr int RPB = kBlock / G;
    const int64_t i = (int64_t)blockIdx.x * RPB + threadIdx.x / G;
    const int sub = threadIdx.x % G;
    Own<MODE, DOT> own;
    if (sub == 0 && i < A.nrows) own.load(a, i);
    double ax;
    if (MODE == MODE_RESID)
        ax = csr_row<G>(A, i, sub, GatherX{a.r});
    else
        ax = csr_row<G>(A, i, sub, GatherX{a.x});
    double dot = 0.0;
    if (sub == 0 && i < A.nrows) {
        const double y = own.apply(ax);
        a.out[i] = y;
        if (DOT) dot = own.r * y;
    }
    if (DOT) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        dot_out(a.dot_part, v[0]);
    }
}

// bottom level: x = inv(A_bottom) r per subdomain.  Grid = (chunks of 32
// rows, subdomains); inside a block the 8 warps split the j range (fixed
// split, deterministic), lane = row, the inverse is stored transposed so the
// lanes read it coalesced; warp partials are added in warp order.
static __global__ void __launch_bounds__(256) k_bottom(const double *__restrict__ invT, const int64_t *__restrict__ inv_off,
                                                const int64_t *__restrict__ off, const double *__restrict__ r,
                                                double *__restrict__ x, const KState *st) {
    DFL_PDL_ENTRY;
    __shared__ double part[8][33];
    const int s = blockIdx.y;
    const int64_t o = off[s];
    const int n = (int)(off[s + 1] - o);
    const int ib = blockIdx.x * 32;
    if (ib >= n) return;
    const double *M = invT + inv_off[s];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jchunk = (n + 7) / 8;
    const int j0 = warp * jchunk, j1 = min(n, j0 + jchunk);
    const int i = ib + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (i < n) {
        int j = j0;
        for (; j + 3 < j1; j += 4) {
            a0 = fma(__ldg(M + (int64_t)j * n + i), __ldg(r + o + j), a0);
            a1 = fma(__ldg(M + (int64_t)(j + 1) * n + i), __ldg(r + o + j + 1), a1);
            a2 = fma(__ldg(M + (int64_t)(j + 2) * n + i), __ldg(r + o + j + 2), a2);
            a3 = fma(__ldg(M + (int64_t)(j + 3) * n + i), __ldg(r + o + j + 3), a3);
        }
        for (; j < j1; ++j) a0 = fma(__ldg(M + (int64_t)j * n + i), __ldg(r + o + j), a0);
    }
    part[warp][lane] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (warp == 0 && i < n) {
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) acc += part[w][lane];
        x[o + i] = acc;
    }
}

// ---------------------------------------------------------------------------
// Operator SpMV (runtime.py:283-292) with the deflation epilogue: per tile
// (tiles never straddle a subdomain) partial sums of Z' y for the k basis
// columns (column 0 is the constant 1; columns 1..k-1 come from zcols).
//   OPMODE 0: y = A x ;  OPMODE 1: y = b - A x
struct Tiles {
    const int64_t *row0;  // ntiles + 1 boundaries are not contiguous across subdomains
    const int64_t *row1;
    int64_t ntiles;
};

// subdomain-aligned tiles without a global table lookup: tile t of
// subdomain s covers rows sub_off[s] + (t - tile_start[s]) * rows_per_tile ...
constexpr int kSubTab = 32;
struct SubTable {
    int n = 0;                 // 0: use the global Tiles arrays
    int rows_per_tile = 0;
    int64_t sub_off[kSubTab + 1];
    int64_t tile_start[kSubTab + 1];
};


// rows [r0, r1) of tile t; returns its subdomain (S.n > 0) or -1.  The table
// is a __grid_constant__ kernel parameter, so the (block-uniform) scan reads
// the constant bank directly; one subdomain -- the common case -- is a
// straight-line path.
__device__ __forceinline__ int tile_rows(const SubTable &S, const Tiles &T, int64_t t, int64_t &r0, int64_t &r1) {
    if (S.n > 0) {
        int s = 0;
        while (s + 1 < S.n && S.tile_start[s + 1] <= t) ++s;
        r0 = S.sub_off[s] + (t - S.tile_start[s]) * S.rows_per_tile;
        r1 = min(r0 + (int64_t)S.rows_per_tile, S.sub_off[s + 1]);
        return s;
    }
    r0 = T.row0[t];
    r1 = T.row1[t];
    return -1;
}

struct OpArgs {
    const double *x;        // gathered input (n_local + n_ghost)
    const double *b;        // OPMODE 1
    double *y;
    const double *zcols;    // (k-1) columns, column-major, length n each
    int64_t n;
    int k;                  // 0: no Z' partials
    double *zt_part;        // ntiles * k
    const KState *st;
    int need_refresh;       // 1: skip unless st->refresh_now
    const uint8_t *skip_rows = nullptr;  // halo overlap: rows with ghost columns are done later
    int64_t pf = 0;  // FMT_CLASS: L2 prefetch distance in rows (0: none)
    // Z columns dictionary-coded (nullptr: dense zcols): zs uint16 per row,
    // column q-1 of the row indexes ztab + ztab_off[q-1]
    const uint16_t *zcode = nullptr;
    const double *ztab = nullptr;
    int zs = 0;
    int ztab_off[kKmax] = {};
};

// the uint16 dictionary indices of row i (S per row: one vector load)
__device__ __forceinline__ void load_codes(const uint16_t *codes, int S, int64_t i, uint32_t (&w)[4]) {
    w[0] = w[1] = w[2] = w[3] = 0u;
    if (S == 4) {
        const uint2 v = __ldcs(reinterpret_cast<const uint2 *>(codes) + i);
        w[0] = v.x, w[1] = v.y;
    } else if (S == 8) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(codes) + i);
        w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    } else if (S == 2) {
        w[0] = __ldcs(reinterpret_cast<const unsigned int *>(codes) + i);
    } else {
        w[0] = __ldcs(reinterpret_cast<const unsigned short *>(codes) + i);
    }
}
__device__ __forceinline__ int code_at(const uint32_t (&w)[4], int c) {
    return (int)((w[c >> 1] >> ((c & 1) * 16)) & 0xffffu);
}

// Z'y partials of one tile: thread c < k writes column c (NV >= k, power of two)
template <int NV>
__device__ __forceinline__ void op_zt(const OpArgs &a, int64_t i, bool valid, double y, int64_t slot) {
    __shared__ double sm[32 * NV];
    double acc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) acc[c] = 0.0;
    if (valid) {
        acc[0] = y;
        if (a.zcode) {
            uint32_t w[4];
            load_codes(a.zcode, a.zs, i, w);
#pragma unroll
            for (int c = 1; c < NV; ++c)
                if (c < a.k) acc[c] = __ldg(a.ztab + a.ztab_off[c - 1] + code_at(w, c - 1)) * y;
        } else {
#pragma unroll
            for (int c = 1; c < NV; ++c)
                if (c < a.k) acc[c] = __ldg(a.zcols + (int64_t)(c - 1) * a.n + i) * y;
        }
    }
    const double tot = block_sum_t<NV>(acc, sm);
    if ((int)threadIdx.x < a.k) a.zt_part[slot * a.k + threadIdx.x] = tot;
}

template <int OPMODE, int W, int NV>
__global__ void __launch_bounds__(kBlock) k_op_ell(DMat A, Tiles T, const __grid_constant__ SubTable S, OpArgs a) {
    DFL_PDL_ENTRY;
    if (a.need_refresh && !a.st->refresh_now) return;
    const int64_t t = blockIdx.x;
    int64_t r0, r1;
    const int sub = tile_rows(S, T, t, r0, r1);
    const int64_t i = r0 + threadIdx.x;
    const bool valid = i < r1 && !(a.skip_rows && a.skip_rows[i]);
    double y = 0.0;
    if (valid) {
        const double ax = ell_any<W>(A, i, GatherX{a.x});
        y = OPMODE == 1 ? sub_rn(__ldg(a.b + i), ax) : ax;
        a.y[i] = y;
    }
    if (a.k > 0) {
        op_zt<NV>(a, i, valid, y, t);
    }
}

template <int OPMODE, int NV>
__global__ void __launch_bounds__(kBlock) k_op_code(DMat A, Tiles T, const __grid_constant__ SubTable S, OpArgs a) {
    DFL_PDL_ENTRY;
    if (a.need_refresh && !a.st->refresh_now) return;
    __shared__ int sd[256];
    __shared__ double sv[256];
    const int64_t t = blockIdx.x;
    int64_t r0, r1;
    const int sub = tile_rows(S, T, t, r0, r1);
    const int64_t i = r0 + threadIdx.x;
    const bool valid = i < r1 && !(a.skip_rows && a.skip_rows[i]);
    const uint2 cw = valid ? __ldcs(A.codes + i) : make_uint2(~0u, ~0u);  // in flight during the table load
    load_codes(A, sd, sv);
    double y = 0.0;
    if (valid) {
        const double ax = code_row_w(cw, i, GatherX{a.x}, sd, sv);
        y = OPMODE == 1 ? sub_rn(__ldg(a.b + i), ax) : ax;
        a.y[i] = y;
    }
    if (a.k > 0) {
        op_zt<NV>(a, i, valid, y, t);
    }
}

// FMT_CLASS operator: one kBlock-row tile per block, RPT rows per thread
// (rows i0 and i0 + kBlock / RPT, ...).  The chain of a row is class byte ->
// table -> gathers; the per-thread fixed cost (tile bounds, prefetch, the Z'y
// tree: about half of the kernel's instructions at one row per thread) is
// paid once per RPT rows, and the RPT rows' loads are in flight together.
// The next wave's first DRAM touches (class byte, leading gather edge) are
// prefetched into L2 (a.pf rows ahead).
template <int OPMODE, int NV, bool ZC, int RPT = kOpRpt>
__global__ void __launch_bounds__(kBlock / RPT, DFL_OPCLASS2_MINB) k_op_class(DMat A, Tiles T,
                                                                              const __grid_constant__ SubTable S,
                                                                              OpArgs a,
                                                                              const __grid_constant__ ClassTab C) {
    DFL_PDL_ENTRY;
    if (a.need_refresh && !a.st->refresh_now) return;
    constexpr int TB = kBlock / RPT;
    const int64_t t = blockIdx.x;
    int64_t r0, r1;
    tile_rows(S, T, t, r0, r1);
    const int64_t i0 = r0 + threadIdx.x;
    if (a.pf > 0) {
        const int64_t ip = i0 + a.pf;
        if (ip < A.nrows) {
            prefetch_l2(A.cls + ip);
            prefetch_l2(a.x + min(ip + (int64_t)C.lead, A.ncols - 1));
        }
    }
    bool valid[RPT];
    int c[RPT];
    double bi[RPT];
    uint32_t zw[RPT][4];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t i = i0 + u * TB;
        valid[u] = i < r1 && !(a.skip_rows && a.skip_rows[i]);
        c[u] = valid[u] ? (int)__ldcs(A.cls + i) : 0;
        bi[u] = (OPMODE == 1 && valid[u]) ? __ldg(a.b + i) : 0.0;
        zw[u][0] = zw[u][1] = zw[u][2] = zw[u][3] = 0u;
        if (ZC && valid[u] && a.k > 1) load_codes(a.zcode, NV, i, zw[u]);
    }
    double y[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t i = i0 + u * TB;
        y[u] = 0.0;
        if (valid[u]) {
            const double ax = class_row(C, c[u], i, GatherX{a.x});
            y[u] = OPMODE == 1 ? sub_rn(bi[u], ax) : ax;
            a.y[i] = y[u];
        }
    }
    if (a.k > 0) {
        __shared__ double sm[32 * NV];
        double acc[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = 0.0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int64_t i = i0 + u * TB;
            acc[0] += valid[u] ? y[u] : 0.0;
#pragma unroll
            for (int q = 1; q < NV; ++q) {
                double z = 0.0;
                if (valid[u] && q < a.k)
                    z = ZC ? __ldg(a.ztab + a.ztab_off[q - 1] + code_at(zw[u], q - 1))
                           : __ldcs(a.zcols + (int64_t)(q - 1) * a.n + i);
                acc[q] += z * y[u];
            }
        }
        const double tot = block_sum_t<NV>(acc, sm);
        if ((int)threadIdx.x < a.k) a.zt_part[t * a.k + threadIdx.x] = tot;
    }
}

template <int G, int OPMODE, int NV = kKmax>
__global__ void __launch_bounds__(kBlock) k_op_csr(DMat A, Tiles T, const __grid_constant__ SubTable S, OpArgs a) {
    DFL_PDL_ENTRY;
    if (a.need_refresh && !a.st->refresh_now) return;
    const int64_t t = blockIdx.x;
    int64_t r0, r1;
    tile_rows(S, T, t, r0, r1);
    const int64_t i = r0 + threadIdx.x / G;
    const int sub = threadIdx.x % G;
    const bool inrange = i < r1 && !(a.skip_rows && a.skip_rows[i]);
    const double ax = csr_row<G>(A, inrange ? i : A.nrows, sub, GatherX{a.x});
    const bool valid = inrange && sub == 0;
    double y = 0.0;
    if (valid) {
        y = OPMODE == 1 ? sub_rn(__ldg(a.b + i), ax) : ax;
        a.y[i] = y;
    }
    if (a.k > 0) op_zt<NV>(a, i, valid, y, t);
}

// Halo overlap, second pass: the rows with ghost columns (listed in brows,
// grouped in subdomain-aligned tiles of <= 256) once the ghosts arrived.
// Same per-row arithmetic as the first pass; Z'y partials of tile bt go to
// zt_part[(toff + bt) * k ...].
template <int OPMODE>
__global__ void __launch_bounds__(kBlock) k_op_bnd(DMat A, const int *__restrict__ brows,
                                                   const int *__restrict__ bstart, const int *__restrict__ bcnt,
                                                   int64_t toff, OpArgs a) {
    DFL_PDL_ENTRY;
    if (a.need_refresh && !a.st->refresh_now) return;
    const int64_t bt = blockIdx.x;
    const bool valid = (int)threadIdx.x < bcnt[bt];
    const int64_t slot = valid ? bstart[bt] + threadIdx.x : 0;  // row of the boundary matrix A
    const int64_t i = valid ? brows[slot] : 0;                   // row of the operator
    double y = 0.0;
    if (valid) {
        double ax = 0.0;
        if (A.fmt == FMT_CSR) {
            for (int e = A.ptr[slot]; e < A.ptr[slot + 1]; ++e) ax = add_rn(ax, mul_rn(A.val[e], __ldg(a.x + A.col[e])));
        } else {
            ax = ell_row_sliced(A, slot, GatherX{a.x});
        }
        y = OPMODE == 1 ? sub_rn(__ldg(a.b + i), ax) : ax;
        a.y[i] = y;
    }
    if (a.k > 0) op_zt<kKmax>(a, i, valid, y, toff + bt);
}

// Z' v partials without a product (project(b), coarse_lift(r))
// the dictionary-coded Z columns (OpArgs::zcode) for the kernels outside the
// operator; code == nullptr: read the dense columns
struct ZCode {
    const uint16_t *code = nullptr;
    const double *tab = nullptr;
    int stride = 0;
    int off[kKmax] = {};
};
// Z column c (1..k-1) of row i
__device__ __forceinline__ double zcol(const ZCode &zc, const double *zcols, int64_t n, int c, int64_t i,
                                       const uint32_t (&w)[4]) {
    return zc.code ? __ldg(zc.tab + zc.off[c - 1] + code_at(w, c - 1)) : __ldg(zcols + (int64_t)(c - 1) * n + i);
}

static __global__ void __launch_bounds__(kBlock) k_zt_vec(Tiles T, const double *__restrict__ v,
                                                   const double *__restrict__ zcols, int64_t n,
                                                   int k, double *zt_part, const ZCode zc) {
    DFL_PDL_ENTRY;
    const int64_t t = blockIdx.x;
    __shared__ double sm[32 * kKmax];
    double acc[kKmax];
#pragma unroll
    for (int c = 0; c < kKmax; ++c) acc[c] = 0.0;
    for (int64_t i = T.row0[t] + threadIdx.x; i < T.row1[t]; i += blockDim.x) {  // tiles may be wider than the block
        const double y = v[i];
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (zc.code && k > 1) load_codes(zc.code, zc.stride, i, w);
        acc[0] += y;
#pragma unroll
        for (int c = 1; c < kKmax; ++c)
            if (c < k) acc[c] += zcol(zc, zcols, n, c, i, w) * y;
    }
    block_sum<kKmax>(acc, sm);
    if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < kKmax; ++c)
            if (c < k) zt_part[t * k + c] = acc[c];
}

// deterministic sum of nparts partials (one block; read through L2: the
// partials may come from other blocks of the calling kernel)
__device__ __forceinline__ double reduce_parts(const double *part, int64_t nparts) {
    __shared__ double sm[32];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int64_t step = blockDim.x;
    int64_t j = threadIdx.x;
    for (; j + 3 * step < nparts; j += 4 * step) {
        a0 += __ldcg(part + j);
        a1 += __ldcg(part + j + step);
        a2 += __ldcg(part + j + 2 * step);
        a3 += __ldcg(part + j + 3 * step);
    }
    for (; j < nparts; j += step) a0 += __ldcg(part + j);
    double v[1] = {(a0 + a1) + (a2 + a3)};
    block_sum<1>(v, sm);
    __shared__ double total;
    if (threadIdx.x == 0) total = v[0];
    __syncthreads();
    return total;
}

// Sum tile partials per local subdomain -> t (global coarse numbering at
// first_col), then (Einv != nullptr) t2 = E^{-1} t with the replicated
// inverse.  Grid (G, nsub): block (g, s) reads chunk g of subdomain s's tile
// partials -- one contiguous, coalesced range of the row-major zt_part (tile
// t, value c at t * k + c); thread i of the first (blockDim / k) * k always
// sees value i % k -- reduces them per value with a fixed-shape tree and
// writes scratch[(s * G + g) * k + c].  The last block (atomic ticket) adds
// the chunks in chunk order (deterministic) and applies E^{-1}.
constexpr int kZtMaxChunks = 64;
static __global__ void __launch_bounds__(256) k_zt_finish(const double *__restrict__ zt_part,
                                                   const int64_t *__restrict__ sub_tiles, int nsub, int k,
                                                   double *t_out, int64_t first_col, const double *Einv,
                                                   int64_t K, double *t2, const KState *st, int need_refresh,
                                                   unsigned int *ticket, double *scratch,
                                                   const int64_t *sub_tiles2 = nullptr, int64_t toff2 = 0,
                                                   const double *extra_part = nullptr, int64_t extra_n = 0,
                                                   double *extra_out = nullptr) {
    DFL_PDL_ENTRY;
    if (skip(st)) return;
    if (need_refresh && !st->refresh_now) return;
    const int g = blockIdx.x, G = gridDim.x, s = blockIdx.y;
    const int nt = (int)(blockDim.x / k) * k;
    const int i = threadIdx.x;
    __shared__ double sm[256];
    double acc = 0.0;
    if (i < nt) {
        const int64_t t0 = sub_tiles[s], t1 = sub_tiles[s + 1];
        const int64_t e0 = (t0 + (t1 - t0) * g / G) * k, e1 = (t0 + (t1 - t0) * (g + 1) / G) * k;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int64_t e = e0 + i;
        for (; e + 3 * nt < e1; e += 4 * nt) {
            a0 += zt_part[e];
            a1 += zt_part[e + nt];
            a2 += zt_part[e + 2 * nt];
            a3 += zt_part[e + 3 * nt];
        }
        for (; e < e1; e += nt) a0 += zt_part[e];
        acc = (a0 + a1) + (a2 + a3);
        if (sub_tiles2 && g == G - 1)  // boundary-row tiles of the halo-overlapped operator
            for (int64_t e2 = (toff2 + sub_tiles2[s]) * k + i; e2 < (toff2 + sub_tiles2[s + 1]) * k; e2 += nt)
                acc += zt_part[e2];
    }
    sm[i] = acc;
    __syncthreads();
    for (int ng = nt / k; ng > 1;) {  // groups of k lanes, halved each step
        const int half = (ng + 1) / 2;
        if (i < (ng - half) * k) sm[i] += sm[i + half * k];
        __syncthreads();
        ng = half;
    }
    __shared__ bool last;
    if (i < k) scratch[((int64_t)s * G + g) * k + i] = sm[i];
    __syncthreads();
    if (i == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const volatile double *sc = scratch;
    for (int v = i; v < nsub * k; v += blockDim.x) {
        const int vs = v / k, vc = v % k;
        double tot = 0.0;
        for (int j = 0; j < G; ++j) tot += sc[((int64_t)vs * G + j) * k + vc];
        t_out[first_col + v] = tot;
    }
    if (Einv != nullptr) {
        __syncthreads();
        const volatile double *tv = t_out;
        for (int64_t r = i; r < K; r += blockDim.x) {
            double a = 0.0;
            for (int64_t j = 0; j < K; ++j) a = fma(Einv[r * K + j], tv[j], a);
            t2[r] = a;
        }
    }
    if (extra_part != nullptr) {  // the caller's per-block partials (CG: rank-local p.w)
        const double e = reduce_parts(extra_part, extra_n);
        if (i == 0) *extra_out = e;
    }
    if (i == 0) *ticket = 0u;
}

// several ranks: unpack the allgathered rank slots (tg + q * slot, cnt[q]
// values each) into t, t2 = E^{-1} t (Einv != nullptr), and for deflated CG
// (fold_st != nullptr) pAp = sum_q (p.w)_q - t . t2 in rank / index order (the
// rank-local p.w rides in the last entry of every slot; A symmetric:
// p'AZ t2 = (Z'Ap)' t2) followed by the alpha step.  One block.
static __global__ void __launch_bounds__(256) k_unpack(const double *tg, int nranks, int64_t slot,
                                                const int64_t *__restrict__ cnt, double *t, const double *Einv,
                                                int64_t K, double *t2, const KState *st, int need_refresh,
                                                KState *fold_st) {
    DFL_PDL_ENTRY;
    if (skip(st)) return;
    if (need_refresh && !st->refresh_now) return;
    int64_t pos = 0;
    for (int q = 0; q < nranks; ++q) {
        const int64_t c = cnt[q];
        for (int64_t j = threadIdx.x; j < c; j += blockDim.x) t[pos + j] = tg[(int64_t)q * slot + j];
        pos += c;
    }
    if (Einv == nullptr) return;
    __syncthreads();
    for (int64_t r = threadIdx.x; r < K; r += blockDim.x) {
        double a = 0.0;
        for (int64_t j = 0; j < K; ++j) a = fma(Einv[r * K + j], t[j], a);
        t2[r] = a;
    }
    if (fold_st == nullptr) return;
    __syncthreads();
    if (threadIdx.x != 0) return;
    double pw = 0.0;
    for (int q = 0; q < nranks; ++q) pw += tg[(int64_t)q * slot + slot - 1];
    double tt = 0.0;
    for (int64_t j = 0; j < K; ++j) tt += t[j] * t2[j];
    cg_step_pq(fold_st, pw - tt);
}

// AZ storage (deflation.py:140-149): row i of AZ has its entries in the k
// columns of its own subdomain (always present: a_ii z_i) plus, on rows next
// to another subdomain, a few in that subdomain's columns.  The own block is
// stored dense (k x n, column-major, absent entries as 0.0) and the rest as a
// CSR of "extra" entries (nullptr if there are none).  AZ t2 is summed in
// column order like matvec(AZ, .): extras left of the own block, the block,
// extras right of it.  An explicit 0.0 adds +-0 to the running sum, which
// leaves it unchanged, so the result equals the CSR sum bit for bit.
struct ProjArgs {
    const double *azd;     // k x n own-block values (nullptr: no deflation term)
    const uint16_t *acode; // the same values dictionary-coded (code_stride(k) per row), nullptr: read azd
    const double *atab;
    int atab_off[kKmax];
    const int *ax_ptr;     // extras (n + 1 row pointer), nullptr: none
    const uint8_t *ax_flag;  // 1 on the rows that have extras (read instead of ax_ptr on every row)
    const int *ax_col;
    const double *ax_val;
    const int64_t *sub_off;  // nsub + 1 local row offsets (device)
    int nsub;
    int k;
    int64_t own_base;      // global coarse column of the rank's first subdomain
    const double *t2;   // K
    int64_t K;
    int64_t n;
    const double *in;   // w
    double *out;        // w - AZ t2   (may alias in)
    double *out2;       // optional second copy of out (the CG prologue's r = b')
    const double *dotv; // dotmode 1: partial dot(dotv, out)
    const double *base; // MODE 1: out = base - (in - AZ t2)
    double *dot_part;
    int dotmode;        // 0: none, 1: dot(dotv, out), 2: dot(out, out)
    const KState *st;
    int need_refresh;   // 1: only when refresh_now, 0: always, -1: only when !refresh_now
};

// t2 is read through the read-only path (every thread of a subdomain reads the
// same k values: L1 broadcast), so no shared-memory staging and no barrier
// stands in front of the streaming loads
template <int KZ>
__device__ __forceinline__ double az_row(const ProjArgs &a, int64_t i, int s) {
    double v[KZ];
    if (a.acode) {
        uint32_t w[4];
        load_codes(a.acode, KZ, i, w);
#pragma unroll
        for (int c = 0; c < KZ; ++c)
            if (c < a.k) v[c] = __ldg(a.atab + a.atab_off[c] + code_at(w, c));
    } else {
#pragma unroll
        for (int c = 0; c < KZ; ++c)
            if (c < a.k) v[c] = __ldcs(a.azd + (int64_t)c * a.n + i);
    }
    const double *t2o = a.t2 + a.own_base + (int64_t)s * a.k;
    const int64_t own0 = a.own_base + (int64_t)s * a.k;
    double acc = 0.0;
    int e = 0, e1 = 0;
    if (a.ax_ptr && __ldg(a.ax_flag + i)) {
        e = __ldg(a.ax_ptr + i);
        e1 = __ldg(a.ax_ptr + i + 1);
        for (; e < e1 && __ldg(a.ax_col + e) < own0; ++e)
            acc = add_rn(acc, mul_rn(__ldg(a.ax_val + e), __ldg(a.t2 + __ldg(a.ax_col + e))));
    }
#pragma unroll
    for (int c = 0; c < KZ; ++c)
        if (c < a.k) acc = add_rn(acc, mul_rn(v[c], __ldg(t2o + c)));
    for (; e < e1; ++e) acc = add_rn(acc, mul_rn(__ldg(a.ax_val + e), __ldg(a.t2 + __ldg(a.ax_col + e))));
    return acc;
}

// q = w - AZ t2 (+ dot partial p.q);  refresh variant: r = b' - (w - AZ t2) (+ r.r)
// 6 resident blocks (40 registers): 20.4 vs 22.1 us at the compiler's 48
// registers / 5 blocks (150^3, k = 4); 8 blocks spill, and so does KZ = 8 at 6
#ifndef DFL_PROJ_MINB
#define DFL_PROJ_MINB 6
#endif
template <int MODE, int KZ>
__global__ void __launch_bounds__(kBlock, KZ > 4 ? 4 : DFL_PROJ_MINB) k_project(ProjArgs a) {
    DFL_PDL_ENTRY;
    if (skip(a.st)) return;
    if (a.need_refresh == 1 && !a.st->refresh_now) return;
    double dot = 0.0;  // grid-stride (grid = ctx->vgrid): one partial per block
    // subdomain of the thread's rows (increasing): a cursor over sub_off
    int s = 0;
    int64_t snext = a.nsub > 1 ? __ldg(a.sub_off + 1) : INT64_MAX;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * kBlock) {
        while (i >= snext) snext = (++s + 1 < a.nsub) ? __ldg(a.sub_off + s + 1) : INT64_MAX;
        double q = a.in[i];
        if (a.azd) q = sub_rn(q, az_row<KZ>(a, i, s));
        if (MODE == 1) q = sub_rn(__ldg(a.base + i), q);
        a.out[i] = q;
        if (a.out2) a.out2[i] = q;
        if (a.dotmode == 1) dot += __ldg(a.dotv + i) * q;
        if (a.dotmode == 2) dot += q * q;
    }
    if (a.dotmode != 0) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        dot_out(a.dot_part, v[0]);
    }
}

// x = y + Z t2 (coarse_lift, deflation.py:235-237 & :285): Z row i has the
// entries [1, zcols(i, 1..k-1)] at columns s*k .. s*k+k-1, summed in order.
static __global__ void __launch_bounds__(kBlock) k_lift(Tiles T, const int *tile_sub, const double *__restrict__ y,
                                                 const double *__restrict__ zcols, int64_t n, int k,
                                                 const double *__restrict__ t2, int64_t first_col,
                                                 double *out, int add_y, const ZCode zc) {
    DFL_PDL_ENTRY;
    const int64_t t = blockIdx.x;
    const int64_t base = (first_col + (int64_t)tile_sub[t] * k);
    for (int64_t i = T.row0[t] + threadIdx.x; i < T.row1[t]; i += blockDim.x) {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (zc.code && k > 1) load_codes(zc.code, zc.stride, i, w);
        double acc = add_rn(0.0, mul_rn(1.0, t2[base]));
        for (int c = 1; c < k; ++c) acc = add_rn(acc, mul_rn(zcol(zc, zcols, n, c, i, w), t2[base + c]));
        out[i] = add_y ? add_rn(y[i], acc) : acc;
    }
}

// ---------------------------------------------------------------------------
// vector kernels and reductions

static __global__ void __launch_bounds__(kBlock) k_dot(const double *__restrict__ a, const double *__restrict__ b,
                                                int64_t n, double *part, const KState *st) {
    DFL_PDL_ENTRY;
    if (skip(st)) return;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        acc += a[i] * b[i];
    __shared__ double sm[32];
    double v[1] = {acc};
    block_sum<1>(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// deterministic sum of part[0], part[ld], part[2 ld], ... (one block)
__device__ __forceinline__ double reduce_parts_strided(const double *part, int64_t nparts, int ld) {
    __shared__ double sm[32];
    double acc = 0.0;
    for (int64_t j = threadIdx.x; j < nparts; j += blockDim.x) acc += part[j * ld];
    double v[1] = {acc};
    block_sum<1>(v, sm);
    __shared__ double total;
    if (threadIdx.x == 0) total = v[0];
    __syncthreads();
    return total;
}

static __global__ void k_reduce(const double *part, int64_t nparts, double *out) {
    DFL_PDL_ENTRY;
    const double s = reduce_parts(part, nparts);
    if (threadIdx.x == 0) *out = s;
}

// CG update (krylov.py:127-131): x += alpha p;  r -= alpha q  (+ r.r partial)
// On refresh iterations only x is updated here (r comes from the refresh path).
static __global__ void __launch_bounds__(kBlock) k_cg_update(double *x, double *r, const double *__restrict__ p,
                                                      const double *__restrict__ q, int64_t n, double *part,
                                                      const KState *st, double *rr_out = nullptr,
                                                      unsigned int *ticket = nullptr) {
    DFL_PDL_ENTRY;
    if (skip(st)) return;
    const double alpha = st->alpha;
    const bool refresh = st->refresh_now;
    double dot = 0.0;  // grid-stride (grid = ctx->vgrid)
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double pi = p[i];
        x[i] = add_rn(x[i], mul_rn(alpha, pi));
        if (!refresh) {
            const double ri = sub_rn(r[i], mul_rn(alpha, q[i]));
            r[i] = ri;
            dot += ri * ri;
        }
    }
    if (!refresh) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        dot_out(part, v[0]);
        if (rr_out != nullptr) {  // several ranks: the last block sums the partials for the allgather
            __shared__ bool last;
            if (threadIdx.x == 0) {
                __threadfence();
                last = atomicAdd(ticket, 1u) == gridDim.x - 1;
            }
            __syncthreads();
            if (!last) return;
            __threadfence();
            const double rr = reduce_parts(part, gridDim.x);
            if (threadIdx.x == 0) {
                *rr_out = rr;
                *ticket = 0u;
            }
        }
    }
}

// p = z + beta p (krylov.py:142).  With a graph handle, block 0 also ends the
// iteration (maxiter test, while condition) and clears the refresh IF
// condition for the next iteration.
static __global__ void __launch_bounds__(kBlock) k_cg_p(double *p, const double *__restrict__ z, int64_t n,
                                                 KState *st, int use_cond, cudaGraphConditionalHandle h,
                                                 int use_if, cudaGraphConditionalHandle hif) {
    DFL_PDL_ENTRY;
    if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) {
        const bool done = st->done || st->iters >= st->maxiter;
        if (done && !st->done) st->done = 1;  // maxiter: the loop ends, p is not needed
        cudaGraphSetConditional(h, done ? 0u : 1u);
        if (use_if) cudaGraphSetConditional(hif, 0u);
    }
    if (skip(st)) return;
    const double beta = st->beta;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        p[i] = add_rn(z[i], mul_rn(beta, p[i]));
}

// dst = src unless the solve already ended (b = 0 keeps the zero solution)
static __global__ void k_copy_live(double *dst, const double *src, int64_t n, const KState *st) {
    DFL_PDL_ENTRY;
    if (skip(st)) return;
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < n) dst[i] = src[i];
}

static __global__ void k_copy(double *dst, const double *src, int64_t n) {
    DFL_PDL_ENTRY;
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < n) dst[i] = src[i];
}

static __global__ void k_fill(double *dst, double v, int64_t n) {
    DFL_PDL_ENTRY;
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < n) dst[i] = v;
}

// halo: pack own values to send, in neighbour order
static __global__ void k_gather(const double *__restrict__ src, const int *__restrict__ idx, int64_t m, double *dst) {
    DFL_PDL_ENTRY;
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < m) dst[i] = src[idx[i]];
}

// sum rank-gathered scalars in rank order: out[v] = sum_q g[q*stride + v]
static __global__ void k_rank_sum(const double *g, int nranks, int stride, int nv, double *out) {
    DFL_PDL_ENTRY;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    double acc = 0.0;
    for (int q = 0; q < nranks; ++q) acc += g[(int64_t)q * stride + v];
    out[v] = acc;
}

}  // namespace dfl

namespace dfl {
// ---------------------------------------------------------------------------
// BiCGStab(2) vector kernels (krylov.py:148-262).  Coefficients are computed on
// the host in IEEE double exactly as the reference's Python scalars and passed
// by value; every update keeps the reference's operation order (no FMA).

// up to four dot products sharing one pass: part[blk*4 + q] = sum a_q . b_q
constexpr int kDotStride = 4;
static __global__ void __launch_bounds__(kBlock) k_multidot(const double *__restrict__ a0, const double *__restrict__ b0,
                                                     const double *__restrict__ a1, const double *__restrict__ b1,
                                                     const double *__restrict__ a2, const double *__restrict__ b2,
                                                     const double *__restrict__ a3, const double *__restrict__ b3,
                                                     int nq, int64_t n, double *part) {
    DFL_PDL_ENTRY;
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

// reduce nq interleaved partial streams (stride kDotStride) -> out[0..nq)
static __global__ void k_reduceq(const double *part, int64_t nparts, int nq, double *out) {
    DFL_PDL_ENTRY;
    __shared__ double sm[32 * 4];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t j = threadIdx.x; j < nparts; j += blockDim.x)
        for (int q = 0; q < 4; ++q) acc[q] += part[j * kDotStride + q];
    block_sum<4>(acc, sm);
    if (threadIdx.x == 0)
        for (int q = 0; q < nq; ++q) out[q] = acc[q];
}

// d_i = r_i - beta d_i for i < cnt  (krylov.py:189-190)
static __global__ void __launch_bounds__(kBlock) k_bicg_d(const double *__restrict__ r0, double *d0,
                                                   const double *__restrict__ r1, double *d1, int cnt, double beta,
                                                   int64_t n) {
    DFL_PDL_ENTRY;
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    d0[i] = sub_rn(r0[i], mul_rn(beta, d0[i]));
    if (cnt > 1) d1[i] = sub_rn(r1[i], mul_rn(beta, d1[i]));
}

// r_i -= alpha d_{i+1} for i < cnt; u += alpha d_0; partial r_0.r_0
// (krylov.py:199-203)
static __global__ void __launch_bounds__(kBlock) k_bicg_r(double *r0, const double *__restrict__ d1, double *r1,
                                                   const double *__restrict__ d2, int cnt, double *u,
                                                   const double *__restrict__ d0, double alpha, int64_t n,
                                                   double *part) {
    DFL_PDL_ENTRY;
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double dot = 0.0;
    if (i < n) {
        const double a = sub_rn(r0[i], mul_rn(alpha, d1[i]));
        r0[i] = a;
        dot = a * a;
        if (cnt > 1) r1[i] = sub_rn(r1[i], mul_rn(alpha, d2[i]));
        u[i] = add_rn(u[i], mul_rn(alpha, d0[i]));
    }
    __shared__ double sm[32];
    double v[1] = {dot};
    block_sum<1>(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// r2 -= tau12 r1; partials (r2.r2, r0.r2)   (krylov.py:218-225)
static __global__ void __launch_bounds__(kBlock) k_bicg_mr2(double *r2, const double *__restrict__ r1,
                                                     const double *__restrict__ r0, double tau12, int64_t n,
                                                     double *part) {
    DFL_PDL_ENTRY;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double v = sub_rn(r2[i], mul_rn(tau12, r1[i]));
        r2[i] = v;
        acc[0] += v * v;
        acc[1] += r0[i] * v;
    }
    __shared__ double sm[32 * 3];
    block_sum<3>(acc, sm);
    if (threadIdx.x == 0)
        for (int q = 0; q < 3; ++q) part[blockIdx.x * kDotStride + q] = acc[q];
}

// the closing updates of one BiCGStab(2) group (krylov.py:247-253):
//   u += g1 r0; r0 -= gp2 r2; d0 -= g2 d2; d0 -= g1 d1; u += gpp1 r1; r0 -= gp1 r1
// + partial r0.r0 (unless the recurrence is refreshed afterwards)
static __global__ void __launch_bounds__(kBlock) k_bicg_final(double *u, double *r0, double *d0,
                                                       const double *__restrict__ r1, const double *__restrict__ r2,
                                                       const double *__restrict__ d1, const double *__restrict__ d2,
                                                       double g1, double gp2, double g2, double gpp1, double gp1,
                                                       int64_t n, double *part) {
    DFL_PDL_ENTRY;
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    double dot = 0.0;
    if (i < n) {
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
        dot = ri * ri;
    }
    __shared__ double sm[32];
    double v[1] = {dot};
    block_sum<1>(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

}  // namespace dfl

namespace dfl {
// ---------------------------------------------------------------------------
// (F)GMRES kernels (krylov.py:288-414): Arnoldi with two Gram-Schmidt passes
// over the basis, done as classical Gram-Schmidt per pass (one multi-vector
// reduction + one multi-vector update) instead of the reference's modified
// Gram-Schmidt loop -- equal in exact arithmetic, both re-orthogonalised.

constexpr int kVecGroup = 8;  // basis vectors per block of k_vdots

// part[bx * ld + i] = sum over the block's rows of V_i . w, i in [8*by, 8*by+8)
static __global__ void __launch_bounds__(kBlock) k_vdots(const double *const *__restrict__ V, int nvec,
                                                  const double *__restrict__ w, int64_t n, double *part, int ld) {
    DFL_PDL_ENTRY;
    const int i0 = blockIdx.y * kVecGroup;
    double acc[kVecGroup];
#pragma unroll
    for (int q = 0; q < kVecGroup; ++q) acc[q] = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x; e < n; e += (int64_t)gridDim.x * kBlock) {
        const double we = w[e];
#pragma unroll
        for (int q = 0; q < kVecGroup; ++q)
            if (i0 + q < nvec) acc[q] += V[i0 + q][e] * we;
    }
    __shared__ double sm[32 * kVecGroup];
    block_sum<kVecGroup>(acc, sm);
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < kVecGroup; ++q)
            if (i0 + q < nvec) part[(int64_t)blockIdx.x * ld + i0 + q] = acc[q];
}

// out[i] = sum_bx part[bx * ld + i]   (one block per i)
static __global__ void k_vreduce(const double *part, int64_t nbx, int ld, double *out) {
    DFL_PDL_ENTRY;
    const double s = reduce_parts_strided(part + blockIdx.x, nbx, ld);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// w -= h_0 V_0; w -= h_1 V_1; ... (one rounding per step, as the MGS updates);
// optional partial of w.w after the update
static __global__ void __launch_bounds__(kBlock) k_vsub(double *w, const double *const *__restrict__ V, const double *h,
                                                 int nvec, int64_t n, double *part) {
    DFL_PDL_ENTRY;
    double dot = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x; e < n; e += (int64_t)gridDim.x * kBlock) {
        double we = w[e];
        for (int i = 0; i < nvec; ++i) we = sub_rn(we, mul_rn(h[i], V[i][e]));
        w[e] = we;
        dot += we * we;
    }
    if (part) {
        __shared__ double sm[32];
        double v[1] = {dot};
        block_sum<1>(v, sm);
        if (threadIdx.x == 0) part[blockIdx.x] = v[0];
    }
}

// out = (x +) (v_0 y_0 + y_1 v_1 + ...)  in the reference's order
// (krylov.py:355-363, then x = x + update :407)
static __global__ void __launch_bounds__(kBlock) k_vcombine(double *out, const double *x, const double *const *__restrict__ V,
                                                     const double *y, int nvec, int64_t n) {
    DFL_PDL_ENTRY;
    for (int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x; e < n; e += (int64_t)gridDim.x * kBlock) {
        double u = mul_rn(V[0][e], y[0]);
        for (int i = 1; i < nvec; ++i) u = add_rn(u, mul_rn(y[i], V[i][e]));
        out[e] = x ? add_rn(x[e], u) : u;
    }
}

// x = x + u
static __global__ void __launch_bounds__(kBlock) k_addv(double *x, const double *__restrict__ u, int64_t n) {
    DFL_PDL_ENTRY;
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (e < n) x[e] = add_rn(x[e], u[e]);
}

// out = in / s   (V_{j+1} = w / h_{j+1,j}, V_0 = r / ||r||)
static __global__ void __launch_bounds__(kBlock) k_vdiv(double *out, const double *in, double s, int64_t n) {
    DFL_PDL_ENTRY;
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (e < n) out[e] = __ddiv_rn(in[e], s);
}

}  // namespace dfl

namespace dfl {
// ---------------------------------------------------------------------------
// Inexact coarse solve (deflation.py:166-178): y ~= E^{-1} t by restarted GMRES
// on the small dense E (restart K, maxiter 4K+20, relative tolerance
// coarse_tol), one block, no preconditioner, x0 = 0 -- krylov.py:288-407 with
// op = E @ v.  Scratch: (K+1) x K basis + K x K Hessenberg + vectors.

__device__ __forceinline__ double blk_dot(const double *a, const double *b, int K, double *sm) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < K; i += blockDim.x) acc += a[i] * b[i];
    double v[1] = {acc};
    block_sum<1>(v, sm);
    __shared__ double res;
    if (threadIdx.x == 0) res = v[0];
    __syncthreads();
    const double r = res;
    __syncthreads();
    return r;
}

static __global__ void __launch_bounds__(256) k_egmres(const double *__restrict__ E, int K, const double *t, double *y,
                                                double tol, double *scr, const KState *st, int need_refresh) {
    DFL_PDL_ENTRY;
    if (skip(st)) return;
    if (need_refresh && !st->refresh_now) return;
    __shared__ double sm[32];
    const int restart = K, maxiter = 4 * K + 20;
    double *V = scr;                          // (K+1) x K
    double *H = V + (size_t)(K + 1) * K;      // (K+1) x K, row-major [i * K + j]
    double *x = H + (size_t)(K + 1) * K;      // K
    double *r = x + K;                        // K
    double *w = r + K;                        // K
    double *g = w + K;                        // K+1
    double *cs = g + K + 1, *sn = cs + K, *yy = sn + K;
    const double bnorm = sqrt(fmax(blk_dot(t, t, K, sm), 0.0));
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        x[i] = 0.0;
        r[i] = t[i];
    }
    __syncthreads();
    if (bnorm == 0.0) {
        for (int i = threadIdx.x; i < K; i += blockDim.x) y[i] = 0.0;
        return;
    }
    const double target = tol * bnorm;
    double res = sqrt(fmax(blk_dot(r, r, K, sm), 0.0));
    int total = 0;
    while (total < maxiter && res > target) {
        const int steps = min(restart, maxiter - total);
        for (int i = threadIdx.x; i < K; i += blockDim.x) V[i] = r[i] / res;
        if (threadIdx.x == 0) {
            for (int q = 0; q <= K; ++q) g[q] = 0.0;
            g[0] = res;
        }
        __syncthreads();
        int j = 0;
        while (j < steps) {
            const double *vj = V + (size_t)j * K;
            for (int i = threadIdx.x; i < K; i += blockDim.x) {  // w = E v_j
                double a = 0.0;
                for (int q = 0; q < K; ++q) a += E[(size_t)i * K + q] * vj[q];
                w[i] = a;
            }
            __syncthreads();
            for (int pass = 0; pass < 2; ++pass)
                for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt, re-orthogonalised
                    const double h = blk_dot(w, V + (size_t)i * K, K, sm);
                    if (threadIdx.x == 0) H[(size_t)i * K + j] = pass == 0 ? h : H[(size_t)i * K + j] + h;
                    for (int q = threadIdx.x; q < K; q += blockDim.x) w[q] = w[q] - h * V[(size_t)i * K + q];
                    __syncthreads();
                }
            const double hn = sqrt(fmax(blk_dot(w, w, K, sm), 0.0));
            const bool exact = hn == 0.0;
            if (!exact)
                for (int q = threadIdx.x; q < K; q += blockDim.x) V[(size_t)(j + 1) * K + q] = w[q] / hn;
            if (threadIdx.x == 0) {
                H[(size_t)(j + 1) * K + j] = hn;
                for (int i = 0; i < j; ++i) {
                    const double a = H[(size_t)i * K + j], b = H[(size_t)(i + 1) * K + j];
                    H[(size_t)(i + 1) * K + j] = -sn[i] * a + cs[i] * b;
                    H[(size_t)i * K + j] = cs[i] * a + sn[i] * b;
                }
                const double a = H[(size_t)j * K + j], b = H[(size_t)(j + 1) * K + j];
                const double rad = hypot(a, b);
                cs[j] = rad == 0.0 ? 1.0 : a / rad;
                sn[j] = rad == 0.0 ? 0.0 : b / rad;
                H[(size_t)j * K + j] = cs[j] * a + sn[j] * b;
                H[(size_t)(j + 1) * K + j] = 0.0;
                g[j + 1] = -sn[j] * g[j];
                g[j] = cs[j] * g[j];
            }
            __syncthreads();
            const double inner = fabs(g[j + 1]);
            ++j;
            if (exact || inner <= target) break;
        }
        if (threadIdx.x == 0)
            for (int i = j - 1; i >= 0; --i) {
                double s = 0.0;
                for (int q = i + 1; q < j; ++q) s += H[(size_t)i * K + q] * yy[q];
                yy[i] = (g[i] - s) / H[(size_t)i * K + i];
            }
        __syncthreads();
        for (int q = threadIdx.x; q < K; q += blockDim.x) {
            double u = V[q] * yy[0];
            for (int i = 1; i < j; ++i) u = u + yy[i] * V[(size_t)i * K + q];
            x[q] = x[q] + u;
        }
        __syncthreads();
        total += j;
        for (int i = threadIdx.x; i < K; i += blockDim.x) {  // r = t - E x
            double a = 0.0;
            for (int q = 0; q < K; ++q) a += E[(size_t)i * K + q] * x[q];
            r[i] = t[i] - a;
        }
        __syncthreads();
        res = sqrt(fmax(blk_dot(r, r, K, sm), 0.0));
    }
    for (int i = threadIdx.x; i < K; i += blockDim.x) y[i] = x[i];
}

}  // namespace dfl
