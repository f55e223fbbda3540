// Smoothed-aggregation setup products on the GPU.
//
// The sequential pieces stay on the host (greedy aggregation amg.py:87-125 is
// ordered by construction, the bottom LU); the O(nnz) and product-shaped
// pieces run here, one thread per output row, each row computed with exactly
// the host's (and the reference's) arithmetic so the hierarchy is bit-for-bit
// the one host_setup.cpp builds:
//   * strength filter            amg.py:70-84
//   * smoothed prolongation      amg.py:136-157 ((I - w D^-1 S) T, from_coo sum)
//   * stable transpose R = P'    _kernels.pyx:26-52 (radix sort by column: stable in row order)
//   * Galerkin products A P, R (A P)  _kernels.pyx:55-115
// The Gustavson product sums every output entry over the A-row entries in
// CSR order; here a row is a k-way merge of the sorted B rows its A entries
// select, and each output column is accumulated by scanning the merge heads
// in A-row order -- the same order, so the same rounding.  Products are
// explicit __dmul_rn / __dadd_rn (no FMA contraction).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "host_setup.hpp"

namespace dfl {

namespace {

constexpr int kT = 256;

struct DCsr {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int64_t *ptr = nullptr, *col = nullptr;
    double *val = nullptr;
};

struct Dev {
    cudaStream_t st = nullptr;
    cudaMemPool_t pool = nullptr;  // trimmed when the build ends (the pages stay mapped during it)
    uint64_t old_threshold = 0;
    std::vector<void *> live;
    std::string err;
    bool ok = true;
    void *alloc(size_t bytes) {
        void *p = nullptr;
        if (bytes == 0) bytes = 8;
        if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) {
            ok = false;
            err = "device allocation of " + std::to_string(bytes) + " bytes failed in setup";
            cudaGetLastError();
            return nullptr;
        }
        live.push_back(p);
        return p;
    }
    void release(void *p) {
        if (!p) return;
        for (auto &q : live)
            if (q == p) {
                cudaFreeAsync(p, st);
                q = nullptr;
                return;
            }
    }
    void free_csr(DCsr &m) {
        release(m.ptr);
        release(m.col);
        release(m.val);
        m = DCsr{};
    }
    ~Dev() {
        for (void *p : live)
            if (p) cudaFreeAsync(p, st);
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
        if (pool) {
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &old_threshold);
            cudaMemPoolTrimTo(pool, 0);
        }
    }
};

#define DCK(x)                                                                       \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            set_setup_error(std::string("CUDA error in device setup: ") + #x + ": " + \
                            cudaGetErrorString(e_));                                 \
            return DFL_E_CUDA;                                                     \
        }                                                                            \
    } while (0)

inline unsigned blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

// ---- kernels ---------------------------------------------------------------

// |a_ij| > eps sqrt(|a_ii| |a_jj|) or i == j (amg.py:70-84); pass 0 counts,
// pass 1 copies the kept entries in CSR order
template <bool FILL>
__global__ void k_strength(int64_t n, const int64_t *__restrict__ ap, const int64_t *__restrict__ ac,
                           const double *__restrict__ av, const double *__restrict__ d, double eps,
                           int64_t *__restrict__ cnt_or_ptr, int64_t *__restrict__ sc, double *__restrict__ sv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double di = fabs(d[i]);
    int64_t o = FILL ? cnt_or_ptr[i] : 0;
    for (int64_t k = ap[i]; k < ap[i + 1]; ++k) {
        const int64_t j = ac[k];
        const double th = __dmul_rn(eps, sqrt(__dmul_rn(di, fabs(d[j]))));
        if (j == i || fabs(av[k]) > th) {
            if (FILL) {
                sc[o] = j;
                sv[o] = av[k];
            }
            ++o;
        }
    }
    if (!FILL) cnt_or_ptr[i] = o;
}

// P row i: the distinct labels of S row i in ascending order, each with the
// S values of that label summed in CSR order (S T, T piecewise constant),
// scaled by -(omega / d_i); the entry at label_i gets 1.0 + scaled, or 1.0
// alone if S row i has no entry of its own aggregate (amg.py:136-157).
template <bool FILL>
__global__ void k_prolong(int64_t n, const int64_t *__restrict__ sp, const int64_t *__restrict__ sc,
                          const double *__restrict__ sv, const int64_t *__restrict__ label,
                          const double *__restrict__ d, double omega, int64_t *__restrict__ cnt_or_ptr,
                          int64_t *__restrict__ pc, double *__restrict__ pv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t k0 = sp[i], k1 = sp[i + 1];
    const int64_t li = label[i];
    const double neg = -(omega / d[i]);
    int64_t o = FILL ? cnt_or_ptr[i] : 0;
    bool placed = false;
    int64_t prev = -1;
    for (;;) {
        int64_t j = INT64_MAX;
        for (int64_t k = k0; k < k1; ++k) {
            const int64_t l = label[sc[k]];
            if (l > prev && l < j) j = l;
        }
        if (j == INT64_MAX) break;
        if (FILL) {
            double acc = 0.0;
            for (int64_t k = k0; k < k1; ++k)
                if (label[sc[k]] == j) acc = __dadd_rn(acc, __dmul_rn(sv[k], 1.0));
            const double scaled = __dmul_rn(neg, acc);
            if (!placed && j > li) {
                pc[o] = li;
                pv[o] = 1.0;
                ++o;
                placed = true;
            }
            pc[o] = j;
            if (j == li) {
                pv[o] = __dadd_rn(1.0, scaled);
                placed = true;
            } else {
                pv[o] = scaled;
            }
            ++o;
        } else {
            if (!placed && j > li) {
                ++o;
                placed = true;
            }
            if (j == li) placed = true;
            ++o;
        }
        prev = j;
    }
    if (!placed) {
        if (FILL) {
            pc[o] = li;
            pv[o] = 1.0;
        }
        ++o;
    }
    if (!FILL) cnt_or_ptr[i] = o;
}

// C row i = sum_k a_ik B_k: merge of the sorted B rows selected by A row i;
// every output column sums its products in A-row order (Gustavson order).
template <int LMAX, bool FILL>
__global__ void __launch_bounds__(kT) k_spgemm(int64_t n, const int64_t *__restrict__ ap, const int64_t *__restrict__ ac,
                                               const double *__restrict__ av, const int64_t *__restrict__ bp,
                                               const int64_t *__restrict__ bc, const double *__restrict__ bv,
                                               int64_t *__restrict__ cnt_or_ptr, int64_t *__restrict__ cc,
                                               double *__restrict__ cv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t pos[LMAX], end[LMAX], head[LMAX];
    const int64_t k0 = ap[i];
    const int L = (int)(ap[i + 1] - k0);
    for (int t = 0; t < L; ++t) {
        const int64_t r = ac[k0 + t];
        pos[t] = bp[r];
        end[t] = bp[r + 1];
        head[t] = pos[t] < end[t] ? bc[pos[t]] : INT64_MAX;
    }
    int64_t o = FILL ? cnt_or_ptr[i] : 0;
    for (;;) {
        int64_t j = INT64_MAX;
        for (int t = 0; t < L; ++t) j = head[t] < j ? head[t] : j;
        if (j == INT64_MAX) break;
        double acc = 0.0;
        for (int t = 0; t < L; ++t)
            if (head[t] == j) {
                if (FILL) acc = __dadd_rn(acc, __dmul_rn(av[k0 + t], bv[pos[t]]));
                ++pos[t];
                head[t] = pos[t] < end[t] ? bc[pos[t]] : INT64_MAX;
            }
        if (FILL) {
            cc[o] = j;
            cv[o] = acc;
        }
        ++o;
    }
    if (!FILL) cnt_or_ptr[i] = o;
}

__global__ void k_row_of(int64_t n, const int64_t *__restrict__ ptr, int64_t *__restrict__ row) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) row[k] = i;
}

__global__ void k_col_keys(int64_t nnz, const int64_t *__restrict__ col, uint32_t *__restrict__ key,
                           int64_t *__restrict__ idx, unsigned long long *__restrict__ count) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    key[k] = (uint32_t)col[k];
    idx[k] = k;
    atomicAdd(count + col[k], 1ull);
}

__global__ void k_gather_t(int64_t nnz, const int64_t *__restrict__ idx, const int64_t *__restrict__ row,
                           const double *__restrict__ val, int64_t *__restrict__ tc, double *__restrict__ tv) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const int64_t s = idx[k];
    tc[k] = row[s];
    tv[k] = val[s];
}

// ---- host helpers ----------------------------------------------------------

// counts[n] (+1 slot) -> exclusive prefix in place; returns the total
int scan_counts(Dev &dv, int64_t *cnt, int64_t n, int64_t &total) {
    size_t tmp = 0;
    DCK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, cnt, n + 1, dv.st));
    void *t = dv.alloc(tmp);
    if (!dv.ok) return DFL_E_CUDA;
    DCK(cub::DeviceScan::ExclusiveSum(t, tmp, cnt, cnt, n + 1, dv.st));
    dv.release(t);
    DCK(cudaMemcpyAsync(&total, cnt + n, sizeof(int64_t), cudaMemcpyDeviceToHost, dv.st));
    DCK(cudaStreamSynchronize(dv.st));
    return DFL_OK;
}

int upload(Dev &dv, const Csr &h, DCsr &d) {
    d.nrows = h.nrows;
    d.ncols = h.ncols;
    d.nnz = h.nnz();
    d.ptr = (int64_t *)dv.alloc(sizeof(int64_t) * (h.nrows + 1));
    d.col = (int64_t *)dv.alloc(sizeof(int64_t) * d.nnz);
    d.val = (double *)dv.alloc(sizeof(double) * d.nnz);
    if (!dv.ok) return DFL_E_CUDA;
    DCK(cudaMemcpyAsync(d.ptr, h.ptr.data(), sizeof(int64_t) * (h.nrows + 1), cudaMemcpyHostToDevice, dv.st));
    DCK(cudaMemcpyAsync(d.col, h.col.data(), sizeof(int64_t) * d.nnz, cudaMemcpyHostToDevice, dv.st));
    DCK(cudaMemcpyAsync(d.val, h.val.data(), sizeof(double) * d.nnz, cudaMemcpyHostToDevice, dv.st));
    return DFL_OK;
}

int download(Dev &dv, const DCsr &d, Csr &h, bool values = true) {
    h.nrows = d.nrows;
    h.ncols = d.ncols;
    h.ptr.resize(d.nrows + 1);
    h.col.resize(d.nnz);
    h.val.resize(values ? d.nnz : 0);
    DCK(cudaMemcpyAsync(h.ptr.data(), d.ptr, sizeof(int64_t) * (d.nrows + 1), cudaMemcpyDeviceToHost, dv.st));
    DCK(cudaMemcpyAsync(h.col.data(), d.col, sizeof(int64_t) * d.nnz, cudaMemcpyDeviceToHost, dv.st));
    if (values) DCK(cudaMemcpyAsync(h.val.data(), d.val, sizeof(double) * d.nnz, cudaMemcpyDeviceToHost, dv.st));
    DCK(cudaStreamSynchronize(dv.st));
    return DFL_OK;
}

// allocate an output with counts already scanned into c.ptr
int alloc_fill(Dev &dv, DCsr &c, int64_t total) {
    c.nnz = total;
    c.col = (int64_t *)dv.alloc(sizeof(int64_t) * total);
    c.val = (double *)dv.alloc(sizeof(double) * total);
    return dv.ok ? DFL_OK : DFL_E_CUDA;
}

template <int LMAX>
void launch_spgemm(Dev &dv, const DCsr &a, const DCsr &b, DCsr &c, bool fill) {
    if (fill)
        k_spgemm<LMAX, true><<<blocks(a.nrows), kT, 0, dv.st>>>(a.nrows, a.ptr, a.col, a.val, b.ptr, b.col, b.val,
                                                               c.ptr, c.col, c.val);
    else
        k_spgemm<LMAX, false><<<blocks(a.nrows), kT, 0, dv.st>>>(a.nrows, a.ptr, a.col, a.val, b.ptr, b.col, b.val,
                                                                c.ptr, nullptr, nullptr);
}

constexpr int64_t kMaxMergeRow = 256;
constexpr int64_t kMinDeviceRows = 20000;

// DFL_SETUP_MIN_ROWS overrides the smallest level whose products run on the device
int64_t min_device_rows() {
    const char *e = std::getenv("DFL_SETUP_MIN_ROWS");
    return e ? std::atoll(e) : kMinDeviceRows;
}

// C = A B on the device; a_max_row = longest A row (<= kMaxMergeRow)
int spgemm_dev(Dev &dv, const DCsr &a, const DCsr &b, int64_t a_max_row, DCsr &c) {
    c.nrows = a.nrows;
    c.ncols = b.ncols;
    c.ptr = (int64_t *)dv.alloc(sizeof(int64_t) * (a.nrows + 1));
    if (!dv.ok) return DFL_E_CUDA;
    DCK(cudaMemsetAsync(c.ptr + a.nrows, 0, sizeof(int64_t), dv.st));
    auto go = [&](bool fill) {
        if (a_max_row <= 8) launch_spgemm<8>(dv, a, b, c, fill);
        else if (a_max_row <= 32) launch_spgemm<32>(dv, a, b, c, fill);
        else if (a_max_row <= 64) launch_spgemm<64>(dv, a, b, c, fill);
        else launch_spgemm<kMaxMergeRow>(dv, a, b, c, fill);
    };
    go(false);
    DCK(cudaGetLastError());
    int64_t total = 0;
    int rc = scan_counts(dv, c.ptr, a.nrows, total);
    if (rc != DFL_OK) return rc;
    if ((rc = alloc_fill(dv, c, total)) != DFL_OK) return rc;
    go(true);
    DCK(cudaGetLastError());
    return DFL_OK;
}

// stable transpose (column-major order of the row-major entries)
int transpose_dev(Dev &dv, const DCsr &a, DCsr &t) {
    t.nrows = a.ncols;
    t.ncols = a.nrows;
    t.nnz = a.nnz;
    t.ptr = (int64_t *)dv.alloc(sizeof(int64_t) * (a.ncols + 1));
    int64_t *row = (int64_t *)dv.alloc(sizeof(int64_t) * a.nnz);
    uint32_t *key = (uint32_t *)dv.alloc(sizeof(uint32_t) * a.nnz);
    uint32_t *key2 = (uint32_t *)dv.alloc(sizeof(uint32_t) * a.nnz);
    int64_t *idx = (int64_t *)dv.alloc(sizeof(int64_t) * a.nnz);
    int64_t *idx2 = (int64_t *)dv.alloc(sizeof(int64_t) * a.nnz);
    if (!dv.ok) return DFL_E_CUDA;
    DCK(cudaMemsetAsync(t.ptr, 0, sizeof(int64_t) * (a.ncols + 1), dv.st));
    k_row_of<<<blocks(a.nrows), kT, 0, dv.st>>>(a.nrows, a.ptr, row);
    k_col_keys<<<blocks(a.nnz), kT, 0, dv.st>>>(a.nnz, a.col, key, idx, (unsigned long long *)t.ptr);
    DCK(cudaGetLastError());
    int bits = 1;
    while (bits < 32 && (int64_t(1) << bits) < a.ncols) ++bits;
    cub::DoubleBuffer<uint32_t> kb(key, key2);
    cub::DoubleBuffer<int64_t> vb(idx, idx2);
    size_t tmp = 0;
    DCK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, a.nnz, 0, bits, dv.st));
    void *tb = dv.alloc(tmp);
    if (!dv.ok) return DFL_E_CUDA;
    DCK(cub::DeviceRadixSort::SortPairs(tb, tmp, kb, vb, a.nnz, 0, bits, dv.st));
    int64_t total = 0;
    int rc = scan_counts(dv, t.ptr, a.ncols, total);
    if (rc != DFL_OK) return rc;
    t.col = (int64_t *)dv.alloc(sizeof(int64_t) * a.nnz);
    t.val = (double *)dv.alloc(sizeof(double) * a.nnz);
    if (!dv.ok) return DFL_E_CUDA;
    k_gather_t<<<blocks(a.nnz), kT, 0, dv.st>>>(a.nnz, vb.Current(), row, a.val, t.col, t.val);
    DCK(cudaGetLastError());
    for (void *p : {(void *)row, (void *)key, (void *)key2, (void *)idx, (void *)idx2, tb}) dv.release(p);
    return DFL_OK;
}

int64_t max_row(const Csr &a) {
    int64_t m = 0;
    for (int64_t i = 0; i < a.nrows; ++i) m = std::max(m, a.ptr[i + 1] - a.ptr[i]);
    return m;
}

}  // namespace

static thread_local int g_setup_device = -1;  // per calling thread (ranks may build concurrently)

void set_setup_device(int device) { g_setup_device = device; }
int setup_device() { return g_setup_device; }

// amg.py:217-250 with the per-level products on the device (see the header)
int build_hierarchy_dev(const Csr &a0, const dfl_amg_options &o, Hierarchy &h) {
    DCK(cudaSetDevice(g_setup_device));
    Dev dv;
    DCK(cudaStreamCreateWithFlags(&dv.st, cudaStreamNonBlocking));
    {
        // keep the stream-ordered pool's pages mapped across the per-level syncs
        DCK(cudaDeviceGetDefaultMemPool(&dv.pool, g_setup_device));
        DCK(cudaMemPoolGetAttribute(dv.pool, cudaMemPoolAttrReleaseThreshold, &dv.old_threshold));
        uint64_t keep = UINT64_MAX;
        DCK(cudaMemPoolSetAttribute(dv.pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    h.levels.clear();
    h.relax = o.relax;
    const bool verbose = std::getenv("DFL_SETUP_VERBOSE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    Csr cur = a0;
    DCsr dA;
    int rc = upload(dv, cur, dA);
    if (rc != DFL_OK) return rc;
    int li = 0;
    for (;;) {
        if (cur.nrows <= o.coarse_enough || li + 1 >= o.max_levels) return close_bottom(h, std::move(cur));
        auto t0 = now();
        std::vector<double> d;
        if (!diagonal(cur, d, "strength graph")) return DFL_E_STRUCTURE;
        const double eps = o.eps_strong * std::ldexp(1.0, -li);
        const int64_t n = cur.nrows;
        double *dd = (double *)dv.alloc(sizeof(double) * n);
        int64_t *dlabel = (int64_t *)dv.alloc(sizeof(int64_t) * n);
        DCsr dS;
        dS.nrows = dS.ncols = n;
        dS.ptr = (int64_t *)dv.alloc(sizeof(int64_t) * (n + 1));
        if (!dv.ok) {
            set_setup_error(dv.err);
            return DFL_E_CUDA;
        }
        DCK(cudaMemcpyAsync(dd, d.data(), sizeof(double) * n, cudaMemcpyHostToDevice, dv.st));
        DCK(cudaMemsetAsync(dS.ptr + n, 0, sizeof(int64_t), dv.st));
        k_strength<false><<<blocks(n), kT, 0, dv.st>>>(n, dA.ptr, dA.col, dA.val, dd, eps, dS.ptr, nullptr, nullptr);
        DCK(cudaGetLastError());
        int64_t snnz = 0;
        if ((rc = scan_counts(dv, dS.ptr, n, snnz)) != DFL_OK) return rc;
        if ((rc = alloc_fill(dv, dS, snnz)) != DFL_OK) return rc;
        k_strength<true><<<blocks(n), kT, 0, dv.st>>>(n, dA.ptr, dA.col, dA.val, dd, eps, dS.ptr, dS.col, dS.val);
        DCK(cudaGetLastError());
        Csr s;
        if ((rc = download(dv, dS, s, false)) != DFL_OK) return rc;
        auto t1 = now();
        std::vector<int64_t> label;
        const int64_t naggr = aggregate(s, label);
        auto t2 = now();
        if (verbose) fprintf(stderr, "L%d [dev] strength %.0f ms aggregate %.0f ms\n", li, ms(t0, t1), ms(t1, t2));
        if (naggr == cur.nrows) return close_bottom(h, std::move(cur));
        for (int64_t i = 0; i < n; ++i)
            if (label[i] < 0) {
                set_setup_error("aggregation left an unassigned node");
                return DFL_E_STRUCTURE;
            }
        // P (amg.py:136-157)
        DCK(cudaMemcpyAsync(dlabel, label.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, dv.st));
        DCsr dP;
        dP.nrows = n;
        dP.ncols = naggr;
        dP.ptr = (int64_t *)dv.alloc(sizeof(int64_t) * (n + 1));
        if (!dv.ok) return DFL_E_CUDA;
        DCK(cudaMemsetAsync(dP.ptr + n, 0, sizeof(int64_t), dv.st));
        k_prolong<false><<<blocks(n), kT, 0, dv.st>>>(n, dS.ptr, dS.col, dS.val, dlabel, dd, o.omega, dP.ptr,
                                                       nullptr, nullptr);
        DCK(cudaGetLastError());
        int64_t pnnz = 0;
        if ((rc = scan_counts(dv, dP.ptr, n, pnnz)) != DFL_OK) return rc;
        if ((rc = alloc_fill(dv, dP, pnnz)) != DFL_OK) return rc;
        k_prolong<true><<<blocks(n), kT, 0, dv.st>>>(n, dS.ptr, dS.col, dS.val, dlabel, dd, o.omega, dP.ptr, dP.col,
                                                      dP.val);
        DCK(cudaGetLastError());
        dv.free_csr(dS);
        dv.release(dd);
        dv.release(dlabel);
        DCsr dR;
        if ((rc = transpose_dev(dv, dP, dR)) != DFL_OK) return rc;
        Level lv;
        if ((rc = download(dv, dP, lv.P)) != DFL_OK) return rc;
        if ((rc = download(dv, dR, lv.R)) != DFL_OK) return rc;
        lv.w.resize(n);
        if (o.relax == DFL_RELAX_DAMPED_JACOBI) {
            for (int64_t i = 0; i < n; ++i) lv.w[i] = o.damping * (1.0 / d[i]);
        } else {
            for (int64_t i = 0; i < n; ++i) {
                double sq = 0.0;
                for (int64_t k = cur.ptr[i]; k < cur.ptr[i + 1]; ++k) sq = sq + cur.val[k] * cur.val[k];
                lv.w[i] = d[i] / sq;
            }
        }
        auto t3 = now();
        // Galerkin R (A P) (amg.py:247); rows too long for the merge kernel go to the host product
        Csr next;
        const int64_t am = max_row(cur), rm = max_row(lv.R);
        // (and small levels, where a thread per row leaves the GPU idle: L3 at 150^3 6 ms host, 24 ms device)
        if (am <= kMaxMergeRow && rm <= kMaxMergeRow && n >= min_device_rows()) {
            DCsr dAP, dN;
            if ((rc = spgemm_dev(dv, dA, dP, am, dAP)) != DFL_OK) return rc;
            if ((rc = spgemm_dev(dv, dR, dAP, rm, dN)) != DFL_OK) return rc;
            dv.free_csr(dAP);
            if ((rc = download(dv, dN, next)) != DFL_OK) return rc;
            dv.free_csr(dA);
            dA = dN;
        } else {
            Csr ap = spgemm(cur, lv.P);
            next = spgemm(lv.R, ap);
            dv.free_csr(dA);
            if ((rc = upload(dv, next, dA)) != DFL_OK) return rc;
        }
        dv.free_csr(dP);
        dv.free_csr(dR);
        if (verbose) fprintf(stderr, "L%d [dev] P+R+w %.0f ms RAP %.0f ms\n", li, ms(t2, t3), ms(t3, now()));
        lv.A = std::move(cur);
        h.levels.push_back(std::move(lv));
        cur = std::move(next);
        ++li;
    }
}

}  // namespace dfl

extern "C" int dfl_setup_device(int device) {
    if (device >= 0) {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || device >= count) {
            cudaGetLastError();
            dfl::set_setup_error("no such CUDA device for the setup");
            return DFL_E_CUDA;
        }
    }
    dfl::set_setup_device(device);
    return DFL_OK;
}
