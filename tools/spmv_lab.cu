// SpMV design lab (not part of the product): times kernel variants for the
// fine-level 7-point operator (150^3, fp64 values, int32 indices, sliced ELL
// with 32-row slices) on one B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o spmv_lab tools/spmv_lab.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1710_03940_b200/csrc/kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int W = 7;

__global__ void k_build(int N, int n, int *col, double *val) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int x = i % N, y = (i / N) % N, z = i / (N * N);
    int c[7];
    double v[7];
    int k = 0;
    int64_t NN = (int64_t)N * N;
    if (z > 0) { c[k] = i - NN; v[k++] = -1; }
    if (y > 0) { c[k] = i - N; v[k++] = -1; }
    if (x > 0) { c[k] = i - 1; v[k++] = -1; }
    c[k] = i; v[k++] = 6;
    if (x < N - 1) { c[k] = i + 1; v[k++] = -1; }
    if (y < N - 1) { c[k] = i + N; v[k++] = -1; }
    if (z < N - 1) { c[k] = i + NN; v[k++] = -1; }
    int last = c[k - 1];
    for (; k < 7; ++k) { c[k] = last; v[k] = 0; }
    int64_t s = i >> 5, lane = i & 31;
    for (int j = 0; j < 7; ++j) {
        col[s * 32 * W + j * 32 + lane] = c[j];
        val[s * 32 * W + j * 32 + lane] = v[j];
    }
}

// V1: one row per thread, register staged
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_v1(int n, const int *__restrict__ col, const double *__restrict__ val,
                                                  const double *__restrict__ x, double *__restrict__ y) {
    int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    const int *cp = col + (i >> 5) * 32 * W + (i & 31);
    const double *vp = val + (i >> 5) * 32 * W + (i & 31);
    int c[W];
    double v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) { c[k] = __ldcs(cp + 32 * k); v[k] = __ldcs(vp + 32 * k); }
    double acc = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) acc = __dadd_rn(acc, __dmul_rn(v[k], __ldg(x + c[k])));
    y[i] = acc;
}

// V2: R rows per thread (rows t, t+stride...) all loads issued up front
template <int R>
__global__ void __launch_bounds__(256) k_v2(int n, const int *__restrict__ col, const double *__restrict__ val,
                                            const double *__restrict__ x, double *__restrict__ y) {
    int64_t base = ((int64_t)blockIdx.x * R) * 256 + threadIdx.x;
    int c[R][W];
    double v[R][W], xv[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int64_t i = base + r * 256;
        if (i < n) {
            const int *cp = col + (i >> 5) * 32 * W + (i & 31);
            const double *vp = val + (i >> 5) * 32 * W + (i & 31);
#pragma unroll
            for (int k = 0; k < W; ++k) { c[r][k] = __ldcs(cp + 32 * k); v[r][k] = __ldcs(vp + 32 * k); }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (base + r * 256 < n)
#pragma unroll
            for (int k = 0; k < W; ++k) xv[r][k] = __ldg(x + c[r][k]);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int64_t i = base + r * 256;
        if (i < n) {
            double acc = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) acc = __dadd_rn(acc, __dmul_rn(v[r][k], xv[r][k]));
            y[i] = acc;
        }
    }
}

// V3: persistent warps, software pipelined: prefetch next slice's col/val
__global__ void __launch_bounds__(256) k_v3(int n, const int *__restrict__ col, const double *__restrict__ val,
                                            const double *__restrict__ x, double *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    int64_t ns = (n + 31) / 32;
    int c[W], c2[W];
    double v[W], v2[W];
    int64_t s = warp;
    if (s < ns)
#pragma unroll
        for (int k = 0; k < W; ++k) { c[k] = __ldcs(col + s * 32 * W + k * 32 + lane); v[k] = __ldcs(val + s * 32 * W + k * 32 + lane); }
    for (; s < ns; s += nw) {
        int64_t sn = s + nw;
        if (sn < ns)
#pragma unroll
            for (int k = 0; k < W; ++k) { c2[k] = __ldcs(col + sn * 32 * W + k * 32 + lane); v2[k] = __ldcs(val + sn * 32 * W + k * 32 + lane); }
        double acc = 0;
        double xv[W];
#pragma unroll
        for (int k = 0; k < W; ++k) xv[k] = __ldg(x + c[k]);
#pragma unroll
        for (int k = 0; k < W; ++k) acc = __dadd_rn(acc, __dmul_rn(v[k], xv[k]));
        int64_t i = s * 32 + lane;
        if (i < n) y[i] = acc;
#pragma unroll
        for (int k = 0; k < W; ++k) { c[k] = c2[k]; v[k] = v2[k]; }
    }
}

// stream-read roofline: read the matrix arrays + x, write y
__global__ void k_stream(int64_t m, const double4 *__restrict__ a, double *out) {
    double acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double2 t = __ldcs((const double2 *)(a + i)); double2 u = __ldcs((const double2 *)(a + i) + 1);
        acc += t.x + t.y + u.x + u.y;
    }
    if (acc == 12345.678) out[0] = acc;
}

// V4: no gather -- reads col/val, uses x[row] (what a perfectly cached gather costs)
__global__ void __launch_bounds__(256) k_v4(int n, const int *__restrict__ col, const double *__restrict__ val,
                                            const double *__restrict__ x, double *__restrict__ y) {
    int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    const int *cp = col + (i >> 5) * 32 * W + (i & 31);
    const double *vp = val + (i >> 5) * 32 * W + (i & 31);
    double acc = 0;
    int cs = 0;
#pragma unroll
    for (int k = 0; k < W; ++k) { cs += __ldcs(cp + 32 * k); acc += __ldcs(vp + 32 * k); }
    y[i] = acc * x[i] + cs;
}

int main() {
    const int N = 150;
    const int n = N * N * N;
    const int64_t ns = (n + 31) / 32;
    int *col;
    double *val, *x, *y;
    CK(cudaMalloc(&col, ns * 32 * W * 4));
    CK(cudaMalloc(&val, ns * 32 * W * 8));
    CK(cudaMalloc(&x, (size_t)n * 8));
    CK(cudaMalloc(&y, (size_t)n * 8));
    CK(cudaMemset(col, 0, ns * 32 * W * 4));
    CK(cudaMemset(val, 0, ns * 32 * W * 8));
    k_build<<<(n + 255) / 256, 256>>>(N, n, col, val);
    std::vector<double> hx(n, 1.0);
    CK(cudaMemcpy(x, hx.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const double bytes = 12.0 * n * 7 /*ELL incl padding approx*/ + 8.0 * n + 8.0 * n;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char *name, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        const int reps = 30;
        for (int i = 0; i < reps; ++i) fn();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        printf("%-28s %8.1f us  %7.0f GB/s (ELL bytes %.0f MB)\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9, bytes / 1e6);
    };
    const int g256 = (n + 255) / 256;
    timeit("v1 minb1", [&] { k_v1<1><<<g256, 256>>>(n, col, val, x, y); });
    timeit("v1 minb6", [&] { k_v1<6><<<g256, 256>>>(n, col, val, x, y); });
    timeit("v1 minb8", [&] { k_v1<8><<<g256, 256>>>(n, col, val, x, y); });
    timeit("v2 R2", [&] { k_v2<2><<<(g256 + 1) / 2, 256>>>(n, col, val, x, y); });
    timeit("v2 R4", [&] { k_v2<4><<<(g256 + 3) / 4, 256>>>(n, col, val, x, y); });
    for (int bps : {4, 8, 16}) {
        char nm[64];
        snprintf(nm, sizeof nm, "v3 persistent %d/SM", bps);
        timeit(nm, [&] { k_v3<<<nsm * bps, 256>>>(n, col, val, x, y); });
    }
    {
        dfl::DMat A;
        A.fmt = dfl::FMT_ELL; A.ell_w = 7; A.nrows = n; A.ncols = n; A.nnz = (int64_t)n * 7; A.col = col; A.val = val;
        double *w;
        CK(cudaMalloc(&w, (size_t)n * 8));
        CK(cudaMemcpy(w, hx.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
        dfl::RowArgs ra{x, w, x, x, y, nullptr, nullptr};
        timeit("prod k_ell PLAIN", [&] { dfl::k_ell<dfl::MODE_PLAIN, false><<<g256, 256>>>(A, ra); });
        timeit("prod k_ell RESID", [&] { dfl::k_ell<dfl::MODE_RESID, false><<<g256, 256>>>(A, ra); });
        timeit("prod k_ell POST+dot", [&] { dfl::k_ell<dfl::MODE_POST, true><<<g256, 256>>>(A, dfl::RowArgs{x, w, x, x, y, w, nullptr}); });
        dfl::SubTable S{};
        S.n = 1; S.rows_per_tile = 256; S.sub_off[0] = 0; S.sub_off[1] = n; S.tile_start[0] = 0; S.tile_start[1] = g256;
        dfl::Tiles T{nullptr, nullptr, g256};
        dfl::OpArgs oa{x, nullptr, y, nullptr, n, 0, nullptr, nullptr, 0};
        timeit("prod k_op_ell k=0", [&] { dfl::k_op_ell<0><<<g256, 256>>>(A, T, S, oa); });
        double *part;
        CK(cudaMalloc(&part, (size_t)g256 * 8 * 8));
        dfl::OpArgs ob{x, nullptr, y, w, n, 4, part, nullptr, 0};
        timeit("prod k_op_ell k=4", [&] { dfl::k_op_ell<0><<<g256, 256>>>(A, T, S, ob); });
    }
    timeit("v4 no-gather", [&] { k_v4<<<g256, 256>>>(n, col, val, x, y); });
    const int64_t m4 = (int64_t)(bytes / 32);
    double *big;
    CK(cudaMalloc(&big, m4 * 32));
    CK(cudaMemset(big, 0, m4 * 32));
    timeit("stream read (same bytes)", [&] { k_stream<<<nsm * 8, 256>>>(m4, (const double4 *)big, y); });
    return 0;
}
