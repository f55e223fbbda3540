// Structured test problems generated on the GPU.
//
// The same rows as problems.py local_rows (the reference's 7-point Poisson
// generator pkg/src/deflamg/problems.py:143-171 in the box-contiguous ordering
// of problems.py:65-104, plus the jump-coefficient and convection-diffusion
// operators of BASELINE.md §4), bit for bit: one thread per row computes its
// node, its neighbours' unknown indices through the box ordering, the
// stencil values with the host's operation order (explicit _rn intrinsics, no
// FMA), and writes the entries sorted by column (stable insertion sort of the
// seven slots, invalid neighbours dropped).  Also the node coordinates and the
// natural-order -> unknown map.  Host side: problems.make_problem(device=...).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <string>
#include <vector>

#include "host_setup.hpp"

namespace {

constexpr int kT = 256;

struct Geo {
    int64_t nx, ny, nz, mx, my, mz, nboxes;
    const int64_t *ex, *ey, *ez;    // box edges per axis (m+1)
    const int64_t *start;           // box start unknowns (nboxes+1)
    double hx, hy, hz;
};

struct Stencil {
    int kind;
    int cells;
    double contrast;
    double off[6];  // poisson / convdiff neighbour values per (axis, step)
    double diag;
};

__device__ __forceinline__ int64_t upper(const int64_t *a, int64_t n, int64_t v) {
    // searchsorted(a[0..n), v, side="right") - 1
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

__device__ __forceinline__ void node_of(const Geo &g, int64_t idx, int64_t &ix, int64_t &iy, int64_t &iz) {
    const int64_t box = upper(g.start, g.nboxes + 1, idx);
    const int64_t bx = box % g.mx, by = (box / g.mx) % g.my, bz = box / (g.mx * g.my);
    const int64_t ox = g.ex[bx], oy = g.ey[by], oz = g.ez[bz];
    const int64_t ex = g.ex[bx + 1] - ox, ey = g.ey[by + 1] - oy;
    const int64_t loc = idx - g.start[box];
    ix = ox + loc % ex;
    iy = oy + (loc / ex) % ey;
    iz = oz + loc / (ex * ey);
}

__device__ __forceinline__ int64_t index_of(const Geo &g, int64_t ix, int64_t iy, int64_t iz) {
    const int64_t bx = upper(g.ex, g.mx + 1, ix), by = upper(g.ey, g.my + 1, iy), bz = upper(g.ez, g.mz + 1, iz);
    const int64_t box = bx + g.mx * (by + g.my * bz);
    const int64_t ox = g.ex[bx], oy = g.ey[by], oz = g.ez[bz];
    const int64_t ex = g.ex[bx + 1] - ox, ey = g.ey[by + 1] - oy;
    return g.start[box] + (ix - ox) + ex * ((iy - oy) + ey * (iz - oz));
}

// _kappa (problems.py:127-131): floor(cells (i+1) h) summed over the axes, odd -> contrast
__device__ __forceinline__ double kappa(const Geo &g, const Stencil &s, int64_t ix, int64_t iy, int64_t iz) {
    const double a = floor(__dmul_rn((double)(s.cells * (ix + 1)), g.hx));
    const double b = floor(__dmul_rn((double)(s.cells * (iy + 1)), g.hy));
    const double c = floor(__dmul_rn((double)(s.cells * (iz + 1)), g.hz));
    const int64_t t = (int64_t)__dadd_rn(__dadd_rn(a, b), c);
    return (t % 2 == 1) ? s.contrast : 1.0;
}

template <bool FILL>
__global__ void k_gen_rows(Geo g, Stencil s, int64_t r0, int64_t nr, int64_t *__restrict__ ptr,
                           int64_t *__restrict__ col, double *__restrict__ val, double *__restrict__ coords) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nr) return;
    const int64_t row = r0 + i;
    int64_t ix, iy, iz;
    node_of(g, row, ix, iy, iz);
    int64_t c[7];
    double v[7];
    c[0] = row;
    const int64_t ext[3] = {g.nx, g.ny, g.nz};
    const int64_t xyz[3] = {ix, iy, iz};
    const double kap = s.kind == DFL_GEN_JUMP ? kappa(g, s, ix, iy, iz) : 0.0;
    double diag = 0.0;
    int slot = 1;
    for (int axis = 0; axis < 3; ++axis)
        for (int step = -1; step <= 1; step += 2) {
            int64_t nb[3] = {ix, iy, iz};
            nb[axis] = xyz[axis] + step;
            const bool ok = nb[axis] >= 0 && nb[axis] < ext[axis];
            c[slot] = ok ? index_of(g, nb[0], nb[1], nb[2]) : -1;
            if (s.kind == DFL_GEN_JUMP) {
                const double kj = ok ? kappa(g, s, nb[0], nb[1], nb[2]) : 1.0;
                const double face = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, kap), kj), __dadd_rn(kap, kj));
                v[slot] = -face;
                diag = __dadd_rn(diag, ok ? face : kap);
            } else {
                v[slot] = s.off[slot - 1];
            }
            ++slot;
        }
    v[0] = s.kind == DFL_GEN_JUMP ? diag : s.diag;
    if constexpr (!FILL) {
        int cnt = 0;
        for (int k = 0; k < 7; ++k) cnt += c[k] >= 0;
        ptr[i] = cnt;
        if (coords) {
            coords[3 * i + 0] = __dmul_rn((double)(ix + 1), g.hx);
            coords[3 * i + 1] = __dmul_rn((double)(iy + 1), g.hy);
            coords[3 * i + 2] = __dmul_rn((double)(iz + 1), g.hz);
        }
        return;
    } else {
        // stable insertion sort by column, invalid (-1) last
        for (int k = 1; k < 7; ++k) {
            const int64_t kc = c[k] >= 0 ? c[k] : INT64_MAX;
            const int64_t cc = c[k];
            const double vv = v[k];
            int q = k - 1;
            while (q >= 0 && (c[q] >= 0 ? c[q] : INT64_MAX) > kc) {
                c[q + 1] = c[q];
                v[q + 1] = v[q];
                --q;
            }
            c[q + 1] = cc;
            v[q + 1] = vv;
        }
        int64_t o = ptr[i];
        for (int k = 0; k < 7; ++k)
            if (c[k] >= 0) {
                col[o] = c[k];
                val[o] = v[k];
                ++o;
            }
    }
}

__global__ void k_gen_uon(Geo g, int64_t n, int64_t *__restrict__ uon) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    uon[k] = index_of(g, k % g.nx, (k / g.nx) % g.ny, k / (g.nx * g.ny));
}

struct Buf {
    std::vector<void *> p;
    template <class T>
    T *get(size_t n) {
        void *q = nullptr;
        if (cudaMalloc(&q, sizeof(T) * (n ? n : 1)) != cudaSuccess) return nullptr;
        p.push_back(q);
        return (T *)q;
    }
    ~Buf() {
        for (void *q : p) cudaFree(q);
    }
};

#define GCK(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            dfl::set_setup_error(std::string("CUDA error in generator: ") + cudaGetErrorString(e_)); \
            return DFL_E_CUDA;                                                                   \
        }                                                                                        \
    } while (0)

// problems.py _edges / BoxOrdering on the host (tiny), uploaded for the kernels
int make_geo(const dfl_gen_params *p, Buf &buf, Geo &g, int64_t &n) {
    std::vector<int64_t> e[3];
    for (int a = 0; a < 3; ++a) {
        const int64_t len = p->shape[a], parts = p->boxes[a];
        if (len < 1 || parts < 1 || parts > len) {
            dfl::set_setup_error("cannot cut an axis of " + std::to_string(len) + " nodes into " +
                                 std::to_string(parts) + " boxes");
            return DFL_E_PARTITION;
        }
        const int64_t q = len / parts, rem = len % parts;
        e[a].push_back(0);
        for (int64_t b = 0; b < parts; ++b) e[a].push_back(e[a].back() + q + (b < rem ? 1 : 0));
    }
    const int64_t mx = p->boxes[0], my = p->boxes[1], mz = p->boxes[2];
    std::vector<int64_t> start{0};
    for (int64_t bz = 0; bz < mz; ++bz)
        for (int64_t by = 0; by < my; ++by)
            for (int64_t bx = 0; bx < mx; ++bx)
                start.push_back(start.back() + (e[0][bx + 1] - e[0][bx]) * (e[1][by + 1] - e[1][by]) *
                                                   (e[2][bz + 1] - e[2][bz]));
    n = start.back();
    int64_t *d[4];
    const std::vector<int64_t> *src[4] = {&e[0], &e[1], &e[2], &start};
    for (int k = 0; k < 4; ++k) {
        d[k] = buf.get<int64_t>(src[k]->size());
        if (!d[k]) {
            dfl::set_setup_error("device allocation failed in the generator");
            return DFL_E_CUDA;
        }
        GCK(cudaMemcpy(d[k], src[k]->data(), sizeof(int64_t) * src[k]->size(), cudaMemcpyHostToDevice));
    }
    g = Geo{p->shape[0], p->shape[1], p->shape[2], mx, my, mz, mx * my * mz, d[0], d[1], d[2], d[3],
            1.0 / (double)(p->shape[0] + 1), 1.0 / (double)(p->shape[1] + 1), 1.0 / (double)(p->shape[2] + 1)};
    return DFL_OK;
}

inline unsigned blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

}  // namespace

extern "C" {

int dfl_gen_rows(int device, const dfl_gen_params *p, int64_t r0, int64_t r1, int64_t *row_ptr, int64_t *col_idx,
                 double *values, int64_t *nnz, double *coords) {
    if (!p || !row_ptr || !col_idx || !values || !nnz) return DFL_E_STATE;
    if (p->kind < DFL_GEN_POISSON || p->kind > DFL_GEN_CONVDIFF) {
        dfl::set_setup_error("unknown problem kind");
        return DFL_E_CONFIG;
    }
    GCK(cudaSetDevice(device));
    Buf buf;
    Geo g;
    int64_t n = 0;
    int rc = make_geo(p, buf, g, n);
    if (rc != DFL_OK) return rc;
    if (r0 < 0 || r1 < r0 || r1 > n) {
        dfl::set_setup_error("row range outside the grid");
        return DFL_E_DIMENSION;
    }
    const int64_t nr = r1 - r0;
    Stencil s{};
    s.kind = p->kind;
    s.cells = p->cells;
    s.contrast = p->contrast;
    s.diag = 6.0;
    for (int a = 0; a < 3; ++a) {
        const double ca = p->kind == DFL_GEN_CONVDIFF ? p->conv[a] : 0.0;
        s.off[2 * a] = p->kind == DFL_GEN_CONVDIFF ? -1.0 - ca : -1.0;
        s.off[2 * a + 1] = p->kind == DFL_GEN_CONVDIFF ? -1.0 + ca : -1.0;
    }
    int64_t *dptr = buf.get<int64_t>(nr + 1);
    int64_t *dcol = buf.get<int64_t>(7 * nr);
    double *dval = buf.get<double>(7 * nr);
    double *dxyz = coords ? buf.get<double>(3 * nr) : nullptr;
    if (!dptr || !dcol || !dval || (coords && !dxyz)) {
        dfl::set_setup_error("device allocation failed in the generator");
        return DFL_E_CUDA;
    }
    GCK(cudaMemset(dptr + nr, 0, sizeof(int64_t)));
    k_gen_rows<false><<<blocks(nr), kT>>>(g, s, r0, nr, dptr, nullptr, nullptr, dxyz);
    GCK(cudaGetLastError());
    size_t tmp = 0;
    GCK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, dptr, dptr, nr + 1));
    void *t = buf.get<char>(tmp);
    if (!t) return DFL_E_CUDA;
    GCK(cub::DeviceScan::ExclusiveSum(t, tmp, dptr, dptr, nr + 1));
    k_gen_rows<true><<<blocks(nr), kT>>>(g, s, r0, nr, dptr, dcol, dval, nullptr);
    GCK(cudaGetLastError());
    GCK(cudaMemcpy(row_ptr, dptr, sizeof(int64_t) * (nr + 1), cudaMemcpyDeviceToHost));
    *nnz = row_ptr[nr];
    GCK(cudaMemcpy(col_idx, dcol, sizeof(int64_t) * *nnz, cudaMemcpyDeviceToHost));
    GCK(cudaMemcpy(values, dval, sizeof(double) * *nnz, cudaMemcpyDeviceToHost));
    if (coords) GCK(cudaMemcpy(coords, dxyz, sizeof(double) * 3 * nr, cudaMemcpyDeviceToHost));
    return DFL_OK;
}

int dfl_gen_unknown_of_node(int device, const dfl_gen_params *p, int64_t *uon) {
    if (!p || !uon) return DFL_E_STATE;
    GCK(cudaSetDevice(device));
    Buf buf;
    Geo g;
    int64_t n = 0;
    int rc = make_geo(p, buf, g, n);
    if (rc != DFL_OK) return rc;
    int64_t *d = buf.get<int64_t>(n);
    if (!d) return DFL_E_CUDA;
    k_gen_uon<<<blocks(n), kT>>>(g, n, d);
    GCK(cudaGetLastError());
    GCK(cudaMemcpy(uon, d, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    return DFL_OK;
}

}  // extern "C"
