// Persistent, TMA-bulk-pipelined sparse row kernels (sm_100a).
//
// The matrix stream (values + column indices) of a row tile is contiguous in
// memory for both storage formats, so one elected thread moves it into shared
// memory with two cp.async.bulk copies that complete on an mbarrier
// (transaction-count based), several tiles ahead of the consumers.  Bytes in
// flight per SM are therefore set by the stage ring (~64-100 KB), not by
// registers or occupancy, which is what an HBM-bound SpMV needs on B200.
// Threads read their entries from shared memory, gather the vector through
// L1/L2 (__ldg) and apply the fused epilogue of the V-cycle / operator stage.
// The per-row summation order is the one of kernels.cuh (ELL and CSR G=1:
// sequential CSR order, bit-identical to the reference's spmv_rows).
#pragma once

#include "kernels.cuh"

namespace dfl {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 1-D bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// all operands of the fused row kernels
enum { PMODE_PLAIN = 0, PMODE_RESID = 1, PMODE_POST = 2, PMODE_PROLONG = 3, PMODE_OP = 4, PMODE_OPRES = 5 };

struct SpArgs {
    const double *x = nullptr;   // gathered vector
    const double *w = nullptr;   // relaxation weights
    const double *r = nullptr;   // level right-hand side
    const double *xo = nullptr;  // POST: own x
    const double *b = nullptr;   // OPRES: y = b - A x
    double *out = nullptr;
    double *part = nullptr;      // per-tile partials: r.out (POST) or Z'out (OP*, k values)
    const double *zcols = nullptr;
    int64_t zn = 0;
    int k = 0;
    const KState *st = nullptr;
    int need_refresh = 0;
};

template <int MODE>
__device__ __forceinline__ double pipe_epilogue(const SpArgs &a, int64_t i, double ax) {
    if (MODE == PMODE_PLAIN || MODE == PMODE_OP) return ax;
    if (MODE == PMODE_OPRES) return sub_rn(__ldg(a.b + i), ax);
    if (MODE == PMODE_RESID) return sub_rn(__ldg(a.r + i), ax);
    if (MODE == PMODE_PROLONG) return add_rn(mul_rn(__ldg(a.w + i), __ldg(a.r + i)), ax);
    return add_rn(__ldg(a.xo + i), mul_rn(__ldg(a.w + i), sub_rn(__ldg(a.r + i), ax)));
}

// ELL row from a staged tile: entries of slice s start at slice_off[s] - e0
template <class Gat>
__device__ __forceinline__ double ell_row_smem(const DMat &A, int64_t row, int64_t e0, const double *vs,
                                               const int *cs, const Gat &g) {
    const int64_t s = row >> 5;
    const int lane = (int)(row & 31);
    const int64_t off = __ldg(A.slice_off + s);
    const int width = (int)((__ldg(A.slice_off + s + 1) - off) >> 5);
    const int base = (int)(off - e0) + lane;
    double acc = 0.0;
    if (width <= kEllUnroll) {
        double xv[kEllUnroll];
#pragma unroll
        for (int k = 0; k < kEllUnroll; ++k)
            if (k < width) xv[k] = g(cs[base + 32 * k]);
#pragma unroll
        for (int k = 0; k < kEllUnroll; ++k)
            if (k < width) acc = add_rn(acc, mul_rn(vs[base + 32 * k], xv[k]));
    } else {
        for (int k = 0; k < width; ++k) acc = add_rn(acc, mul_rn(vs[base + 32 * k], g(cs[base + 32 * k])));
    }
    return acc;
}

template <int G, class Gat>
__device__ __forceinline__ double csr_row_smem(const DMat &A, int64_t row, bool valid, int sub, int64_t e0,
                                               const double *vs, const int *cs, const Gat &g) {
    double acc = 0.0;
    if (valid) {
        const int b = (int)(__ldg(A.ptr + row) - e0), e = (int)(__ldg(A.ptr + row + 1) - e0);
        if (G == 1) {
            for (int k = b; k < e; ++k) acc = add_rn(acc, mul_rn(vs[k], g(cs[k])));
        } else {
            for (int k = b + sub; k < e; k += G) acc += vs[k] * g(cs[k]);
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
    return acc;
}

constexpr int kPipeThreads = 256;

// G == 0: sliced ELL (one row per thread per tile); G >= 1: CSR with G lanes
// per row, rows of the tile in passes of 256/G.
template <int G, int MODE, bool PART>
__global__ void __launch_bounds__(kPipeThreads) k_pipe(DMat A, SpArgs a) {
    const Pipe &T = A.pipe;
    if (skip(a.st)) return;
    if (a.need_refresh && !a.st->refresh_now) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = T.stages;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    double *vbuf = reinterpret_cast<double *>(smem + 128);
    int *cbuf = reinterpret_cast<int *>(vbuf + (size_t)S * T.cap);
    const int tid = threadIdx.x;
    const int64_t P = gridDim.x;
    uint64_t pol = 0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
        pol = policy_evict_first();
    }
    __syncthreads();
    auto issue = [&](int64_t i) {
        const int64_t c = blockIdx.x + i * P;
        if (c >= T.ntiles) return;
        const int s = (int)(i % S);
        const int64_t e0 = T.e0[c];
        const uint32_t n = (uint32_t)T.ecnt[c];
        mbar_expect_tx(&bar[s], n * 12u);
        bulk_g2s(vbuf + (size_t)s * T.cap, A.val + e0, n * 8u, &bar[s], pol);
        bulk_g2s(cbuf + (size_t)s * T.cap, A.col + e0, n * 4u, &bar[s], pol);
    };
    if (tid == 0)
        for (int i = 0; i < S; ++i) issue(i);
    constexpr int NP = (MODE == PMODE_OP || MODE == PMODE_OPRES) ? kKmax : 1;
    for (int64_t i = 0;; ++i) {
        const int64_t c = blockIdx.x + i * P;
        if (c >= T.ntiles) break;
        const int s = (int)(i % S);
        mbar_wait(&bar[s], (uint32_t)((i / S) & 1));
        const double *vs = vbuf + (size_t)s * T.cap;
        const int *cs = cbuf + (size_t)s * T.cap;
        const int64_t e0 = T.e0[c], r0 = T.row0[c], r1 = T.row1[c];
        double acc[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[j] = 0.0;
        auto finish_row = [&](int64_t row, double ax) {
            const double y = pipe_epilogue<MODE>(a, row, ax);
            a.out[row] = y;
            if (PART) {
                if (MODE == PMODE_POST) {
                    acc[0] += __ldg(a.r + row) * y;
                } else {
                    acc[0] += y;
#pragma unroll
                    for (int j = 1; j < NP; ++j)
                        if (j < a.k) acc[j] += __ldg(a.zcols + (int64_t)(j - 1) * a.zn + row) * y;
                }
            }
        };
        if (G == 0) {
            const int64_t row = r0 + tid;
            if (row < r1) {
                double ax;
                if (MODE == PMODE_RESID)
                    ax = ell_row_smem(A, row, e0, vs, cs, GatherX{a.r});
                else
                    ax = ell_row_smem(A, row, e0, vs, cs, GatherX{a.x});
                finish_row(row, ax);
            }
        } else {
            constexpr int GG = G > 0 ? G : 1;
            constexpr int RPP = kPipeThreads / GG;
            const int sub = tid % GG;
            for (int64_t rb = r0; rb < r1; rb += RPP) {
                const int64_t row = rb + tid / GG;
                const bool valid = row < r1;
                double ax;
                if (MODE == PMODE_RESID)
                    ax = csr_row_smem<GG>(A, row, valid, sub, e0, vs, cs, GatherX{a.r});
                else
                    ax = csr_row_smem<GG>(A, row, valid, sub, e0, vs, cs, GatherX{a.x});
                if (valid && sub == 0) finish_row(row, ax);
            }
        }
        if (PART) {
            __shared__ double sm[32 * NP];
            block_sum<NP>(acc, sm);
            if (tid == 0) {
                if (MODE == PMODE_POST)
                    a.part[c] = acc[0];
                else
                    for (int j = 0; j < a.k; ++j) a.part[c * a.k + j] = acc[j];
            }
        }
        __syncthreads();  // every thread is done with stage s
        if (tid == 0) {
            fence_proxy_async_smem();
            issue(i + S);
        }
    }
}

}  // namespace dfl
