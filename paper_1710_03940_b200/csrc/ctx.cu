// Device context of one rank: uploads the host setup products into
// device-resident layouts and runs the solve phase (deflation.py:254-312)
// entirely on the GPU.  The Krylov loop is a CUDA graph with a device-side
// while-conditional, so a whole CG solve is a handful of launches and no
// host round trip per iteration (single rank); with several ranks the loop is
// host-driven with NCCL collectives between kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/dflb200.h"
#include "host_setup.hpp"
#include "kernels.cuh"
#include "spmv_pipe.cuh"
#include "coarse.cuh"

using namespace dfl;

// ---------------------------------------------------------------------------
// minimal NCCL surface, loaded lazily (no link-time dependency)
namespace {
typedef struct {
    char internal[128];
} NcclId;
typedef void *NcclComm;
enum { ncclDouble_ = 8 };
struct Nccl {
    void *h = nullptr;
    int (*GetUniqueId)(NcclId *) = nullptr;
    int (*CommInitRank)(NcclComm *, int, NcclId, int) = nullptr;
    int (*CommDestroy)(NcclComm) = nullptr;
    int (*AllGather)(const void *, void *, size_t, int, NcclComm, cudaStream_t) = nullptr;
    int (*Send)(const void *, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    int (*Recv)(void *, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
    bool load(std::string &err) {
        if (h) return true;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            err = "cannot load libnccl.so.2";
            return false;
        }
#define LD(f, s)                                            \
    f = reinterpret_cast<decltype(f)>(dlsym(h, s));         \
    if (!f) {                                               \
        err = std::string("libnccl lacks ") + s;            \
        return false;                                       \
    }
        LD(GetUniqueId, "ncclGetUniqueId");
        LD(CommInitRank, "ncclCommInitRank");
        LD(CommDestroy, "ncclCommDestroy");
        LD(AllGather, "ncclAllGather");
        LD(Send, "ncclSend");
        LD(Recv, "ncclRecv");
        LD(GroupStart, "ncclGroupStart");
        LD(GroupEnd, "ncclGroupEnd");
        LD(GetErrorString, "ncclGetErrorString");
#undef LD
        return true;
    }
};
Nccl g_nccl;
}  // namespace

static bool g_use_pipe = false;  // TMA-staged variant (DFL_PIPE=1); see profiles/r01
static bool g_use_vcode = false;  // value-coded ELL for V-cycle P/R with <= 255 values (DFL_VCODE=1; measured neutral)
static double g_small_per_lane = 12.0;  // DFL_CSR_PER_LANE_SMALL: entries per lane for levels < 50K rows
static bool g_use_code = true;    // stencil-coded ELL for few-(offset, value) matrices (DFL_NO_CODE=1 disables)
static bool g_use_tiny = false;   // cluster kernel for the tiny levels (DFL_TINY=1; measured slower, profiles/r01)
static bool g_use_coarse = false;  // cooperative coarse-cycle kernel (DFL_COARSE=1; measured slower, profiles/r01)
static constexpr int64_t kCoarseRows = 65536;  // levels at or below this size run in k_coarse_cycle
// layout experiments (profiling knobs, read once per context creation)
// (measured on 150^3, see profiles/r01/README.md: CSR-vector with ~12 entries
// per lane beats SELL-32-1024 for the coarse operators and R / P)
static bool g_allow_sell = false;    // DFL_SELL=1: SELL-C-sigma for every irregular matrix
static int g_csr_g = 0;              // DFL_CSR_G=n forces the CSR lanes per row
static double g_csr_per_lane = 12.0; // DFL_CSR_PER_LANE: target entries per lane

// ---------------------------------------------------------------------------

struct DLevel {
    DMat A, P, R;
    DMat Aw;  // A diag(w): the pre-smoothing residual r - A (w .* r) in one gather
    double *wr = nullptr;  // coded A: w .* r gathered by the residual kernel
    double *w = nullptr;
    int64_t n = 0, nc = 0;
    double *rv = nullptr;  // level right-hand side (l >= 1)
    double *t = nullptr;   // residual / prolongation scratch
    double *xv = nullptr;  // level solution (l >= 1)
};

struct VGroup {
    int sub0 = 0, nsub = 0;
    int64_t row0 = 0, row1 = 0;
    std::vector<DLevel> lv;          // smoothing levels
    int64_t nb = 0;                  // bottom rows (all subdomains of the group)
    double *rb = nullptr, *xb = nullptr;
    double *binvT = nullptr;
    int64_t *binv_off = nullptr;     // per subdomain offset into binvT
    int64_t *b_off = nullptr;        // nsub + 1 row offsets in rb
    int max_nb = 0;
    // levels [lc, L) and the bottom run in one cooperative kernel (coarse.cuh)
    int lc = -1;                     // -1: no coarse kernel
    CoarseArgs *cargs = nullptr;     // device copy
    int lt = -1;                     // levels [lt, L) + bottom run in k_tiny_cycle (-1: none)
    CoarseArgs *targs = nullptr;
    unsigned coarse_grid = 0;
    double *binv = nullptr;          // row-major inverses for the cooperative kernel
    // host-side statistics
    std::vector<int64_t> nnzA, nnzP, rows;
};

// In-process communicator for testing the multi-rank path without NCCL: the
// ranks are contexts driven by different host threads (one device or
// several); every collective synchronises its stream, meets the other ranks
// at a host barrier and copies from the peers' published device buffers.
struct dfl_fabric {
    int nranks = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    std::vector<dfl_ctx *> ctxs;
    std::vector<const double *> pub;  // per-rank published buffer of the current collective
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long gen = generation;
        if (++arrived == nranks) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

struct dfl_ctx {
    int device = 0;
    dfl_fabric *fab = nullptr;
    int sm_count = 148;
    std::vector<int64_t> op_sub_tiles_h;
    int64_t *op_sub_tiles = nullptr;   // first op-pipe tile of every subdomain
    cudaStream_t st = nullptr;
    std::string err;
    std::vector<void *> allocs;
    int64_t bytes = 0;
    // comm
    int nranks = 1, rank = 0;
    NcclComm comm = nullptr;
    // operator
    bool have_op = false, finalized = false;
    int64_t n = 0, n_ghost = 0;
    int nsub = 0;
    std::vector<int64_t> sub_off;
    DMat Aop;
    std::vector<int64_t> op_nnz_rows;  // host stats
    int64_t op_nnz = 0;
    // tiles (per subdomain, rows per tile = op rows per block)
    Tiles tiles{};
    SubTable subtab{};
    int64_t ntiles = 0;
    int *tile_sub = nullptr;
    int64_t *sub_tiles = nullptr;       // device nsub + 1
    std::vector<int64_t> h_sub_tiles;
    // halo
    std::vector<int> nbr;
    std::vector<int64_t> recv_cnt, send_cnt;
    int *send_idx = nullptr;
    int64_t nsend = 0;
    double *sendbuf = nullptr;
    // halo overlap: rows with ghost columns run after the exchange
    bool split = false;
    uint8_t *bflag = nullptr;
    int *brows = nullptr, *bstart = nullptr, *bcnt = nullptr;
    int64_t nbtiles = 0;
    int64_t *sub_btiles = nullptr;
    cudaStream_t st2 = nullptr;
    cudaEvent_t ev_packed = nullptr, ev_halo = nullptr;
    // hierarchies
    std::vector<dfl::Hierarchy> pending;
    std::vector<int> pending_set;
    std::vector<VGroup> groups;
    int relax = DFL_RELAX_DAMPED_JACOBI;
    // deflation
    bool deflation = false;
    int k = 0;
    int64_t K = 0;
    int first_sub = 0;
    double *zcols = nullptr;
    int *az_ptr = nullptr, *az_col = nullptr;
    double *az_val = nullptr;
    int64_t az_nnz = 0;
    double *Einv = nullptr;
    // inexact coarse solve (deflation.py:166-178): inner GMRES on E
    bool inexact = false;
    double *Edense = nullptr, *egm_scr = nullptr;
    double coarse_tol = 1e-2;
    double *tvec = nullptr, *t2 = nullptr;
    double *zt_part = nullptr;
    double *tgather = nullptr;  // nranks * maxsub * k
    unsigned int *ticket = nullptr;
    int max_nsub = 0;
    std::vector<int> rank_nsub;  // subdomains per rank (runtime.rank_subdomains)
    // work vectors (n, or n + n_ghost for operator inputs)
    double *b = nullptr, *bp = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr,
           *w = nullptr, *tmp = nullptr, *xin = nullptr, *yout = nullptr;
    double *dpart = nullptr;
    int64_t nblk = 0;
    // BiCGStab(2) work vectors (allocated on first use)
    double *br[3] = {nullptr, nullptr, nullptr}, *bd[3] = {nullptr, nullptr, nullptr};
    double *bu = nullptr, *bshadow = nullptr, *zx = nullptr;
    double *h_dots = nullptr;  // pinned
    // (F)GMRES (allocated on first use)
    int gm_restart = 0;
    std::vector<double *> gmV, gmZ;
    const double **gmVp = nullptr, **gmZp = nullptr;  // device pointer arrays
    double *gm_h = nullptr, *gm_e = nullptr, *gm_y = nullptr, *gm_part = nullptr, *gm_loc = nullptr,
           *gm_gath = nullptr, *h_gm = nullptr;
    double *scal = nullptr;     // [0..7] local reduced scalars
    double *sgather = nullptr;  // nranks * 8
    KState *state = nullptr;
    KState *h_state = nullptr;  // pinned
    // graph
    cudaGraphExec_t loop_exec = nullptr;
    int loop_key = -1;
    int64_t body_kernels = 0;
    int64_t launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // per-launch profiling of the V-cycle (dfl_ctx_profile_vcycle)
    bool prof_on = false;
    std::vector<cudaEvent_t> prof_ev;
    std::vector<std::string> prof_lab;
    size_t prof_n = 0;
};

static void prof_mark(dfl_ctx *ctx, const std::string &label) {
    if (!ctx->prof_on) return;
    if (ctx->prof_n >= ctx->prof_ev.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->prof_ev.push_back(e);
        ctx->prof_lab.emplace_back();
    }
    cudaEventRecord(ctx->prof_ev[ctx->prof_n], ctx->st);
    ctx->prof_lab[ctx->prof_n] = label;
    ctx->prof_n++;
}

#define CK(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) {                                                             \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
            return DFL_E_CUDA;                                                               \
        }                                                                                    \
    } while (0)
#define RC(call)                       \
    do {                               \
        int r_ = (call);               \
        if (r_ != DFL_OK) return r_;   \
    } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

template <class T>
static int dalloc(dfl_ctx *ctx, T **p, int64_t count) {
    *p = nullptr;
    if (count <= 0) count = 1;
    void *q = nullptr;
    CK(cudaMalloc(&q, sizeof(T) * (size_t)count));
    ctx->allocs.push_back(q);
    ctx->bytes += sizeof(T) * count;
    *p = static_cast<T *>(q);
    return DFL_OK;
}

template <class T>
static int upload(dfl_ctx *ctx, T **p, const T *h, int64_t count) {
    RC(dalloc(ctx, p, count));
    if (count > 0) CK(cudaMemcpy(*p, h, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice));
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// matrix upload with format selection

struct HostRows {
    int64_t nrows, ncols;
    const int64_t *ptr;
    const int64_t *col;
    const double *val;
};

static int build_pipe(dfl_ctx *ctx, const HostRows &h, DMat &m, const std::vector<int64_t> &soff,
                      const std::vector<int64_t> &bounds, std::vector<int64_t> *bound_tiles);

// colscale != nullptr: also upload the column-scaled values a_ij * colscale_j
// in the same layout (shares the index arrays) into *scaled.
// FMT_CODE encoder: every row <= 8 entries and <= 255 distinct (column - row,
// value-bits) pairs; returns false when the matrix does not qualify
static int try_upload_code(dfl_ctx *ctx, const HostRows &h, DMat &m, bool &ok) {
    ok = false;
    struct Key {
        int64_t d;
        uint64_t v;
        bool operator==(const Key &o) const { return d == o.d && v == o.v; }
    };
    struct KH {
        size_t operator()(const Key &k) const { return std::hash<int64_t>()(k.d) * 1000003u ^ std::hash<uint64_t>()(k.v); }
    };
    std::unordered_map<Key, int, KH> dict;
    std::vector<int> delta;
    std::vector<double> val;
    std::vector<uint8_t> codes((size_t)h.nrows * 8, (uint8_t)kCodePad);
    for (int64_t i = 0; i < h.nrows; ++i) {
        const int64_t b = h.ptr[i], e = h.ptr[i + 1];
        if (e - b > 8) return DFL_OK;
        for (int64_t k = b; k < e; ++k) {
            uint64_t bits;
            std::memcpy(&bits, &h.val[k], 8);
            const int64_t d = h.col[k] - i;
            if (d < INT32_MIN || d > INT32_MAX) return DFL_OK;
            auto it = dict.find(Key{d, bits});
            int code;
            if (it == dict.end()) {
                if (dict.size() >= kCodePad) return DFL_OK;
                code = (int)dict.size();
                dict.emplace(Key{d, bits}, code);
                delta.push_back((int)d);
                val.push_back(h.val[k]);
            } else {
                code = it->second;
            }
            codes[(size_t)i * 8 + (k - b)] = (uint8_t)code;
        }
    }
    m.fmt = FMT_CODE;
    m.stored = m.nnz;
    m.ncodes = (int)delta.size();
    uint8_t *d_codes;
    int *d_delta;
    double *d_val;
    RC(upload(ctx, &d_codes, codes.data(), (int64_t)codes.size()));
    RC(upload(ctx, &d_delta, delta.data(), (int64_t)std::max<size_t>(1, delta.size())));
    RC(upload(ctx, &d_val, val.data(), (int64_t)std::max<size_t>(1, val.size())));
    m.codes = reinterpret_cast<const uint2 *>(d_codes);
    m.ctab_delta = d_delta;
    m.ctab_val = d_val;
    ok = true;
    return DFL_OK;
}

// value codes for an ELL-layout matrix with <= 255 distinct values (bitwise)
static int attach_value_codes(dfl_ctx *ctx, DMat &m, const std::vector<double> &val) {
    std::unordered_map<uint64_t, int> dict;
    std::vector<double> tab;
    std::vector<uint8_t> code(val.size());
    for (size_t e = 0; e < val.size(); ++e) {
        uint64_t bits;
        std::memcpy(&bits, &val[e], 8);
        auto it = dict.find(bits);
        if (it == dict.end()) {
            if (dict.size() >= 255) return DFL_OK;  // not value-codable
            it = dict.emplace(bits, (int)tab.size()).first;
            tab.push_back(val[e]);
        }
        code[e] = (uint8_t)it->second;
    }
    uint8_t *d_code;
    double *d_tab;
    RC(upload(ctx, &d_code, code.data(), (int64_t)code.size()));
    RC(upload(ctx, &d_tab, tab.data(), (int64_t)tab.size()));
    m.vcode = d_code;
    m.vtab = d_tab;
    m.nvtab = (int)tab.size();
    return DFL_OK;
}

static constexpr int64_t kSigma = 1024;  // SELL-C-sigma sorting window
// SELL-32-1024 for long-row matrices with enough rows to hide the per-warp
// width imbalance (measured: L0 restriction and L1 operator, profiles/r01);
// short-row (P) and small coarse matrices stay CSR-vector
static constexpr int64_t kSellMinRows = 100000;
static constexpr double kSellMinMean = 12.0;
static constexpr double kShortRowMean = 8.0;  // DFL_SHORT_PAD=x overrides the padding limit below
static double kShortRowPad = 1.7;

static int upload_matrix(dfl_ctx *ctx, const HostRows &h, DMat &m, const std::vector<int64_t> &bounds,
                         std::vector<int64_t> *bound_tiles = nullptr, bool allow_ell = true,
                         const double *colscale = nullptr, DMat *scaled = nullptr, bool allow_sell = true,
                         bool allow_code = true, bool allow_vcode = false) {
    m = DMat{};
    m.nrows = h.nrows;
    m.ncols = h.ncols;
    m.nnz = h.ptr[h.nrows] - h.ptr[0];
    if (h.ncols >= INT32_MAX || m.nnz >= INT32_MAX) {
        ctx->err = "matrix too large for int32 device indices";
        return DFL_E_DIMENSION;
    }
    if (g_use_code && allow_code && allow_ell && h.nrows > 0) {
        bool ok = false;
        RC(try_upload_code(ctx, h, m, ok));
        if (ok) {
            if (colscale) *scaled = m;  // RESID on a coded matrix gathers w .* r instead (k_wr)
            return DFL_OK;
        }
    }
    const int64_t nsl = cdiv(h.nrows, 32);
    auto rlen = [&](int64_t i) { return h.ptr[i + 1] - h.ptr[i]; };
    // slot -> row: identity, or (SELL-C-sigma) rows sorted by length,
    // descending and stable, inside windows of kSigma rows
    std::vector<int> perm;
    auto slice_offsets = [&](const std::vector<int> &pm, int64_t &maxlen) {
        std::vector<int64_t> so(nsl + 1, 0);
        maxlen = 0;
        for (int64_t s = 0; s < nsl; ++s) {
            int64_t wmax = 0;
            for (int64_t j = s * 32; j < std::min(h.nrows, s * 32 + 32); ++j)
                wmax = std::max(wmax, rlen(pm.empty() ? j : pm[j]));
            maxlen = std::max(maxlen, wmax);
            so[s + 1] = so[s] + 32 * wmax;
        }
        return so;
    };
    int64_t maxlen = 0;
    std::vector<int64_t> soff = slice_offsets(perm, maxlen);
    const double mean = h.nrows ? (double)m.nnz / (double)h.nrows : 0.0;
    const double nnzd = (double)m.nnz + 64.0;
    bool ell = false;
    const double upad = mean <= kShortRowMean ? kShortRowPad : 1.03;  // short rows: padding is cheaper than CSR
    if (allow_ell && maxlen <= 8 && (double)(nsl * 32 * maxlen) <= upad * nnzd) {
        // uniform slice width: the kernels compute slice offsets instead of loading them
        ell = true;
        m.ell_w = (int)maxlen;
        for (int64_t s = 0; s <= nsl; ++s) soff[s] = s * 32 * maxlen;
    } else if (allow_ell && (double)soff[nsl] <= 1.03 * nnzd) {
        ell = true;
    } else if (allow_ell && allow_sell && maxlen <= 1024 &&
               (g_allow_sell || (h.nrows >= kSellMinRows && mean >= kSellMinMean))) {
        perm.resize(h.nrows);
        for (int64_t w0 = 0; w0 < h.nrows; w0 += kSigma) {
            const int64_t w1 = std::min(h.nrows, w0 + kSigma);
            for (int64_t j = w0; j < w1; ++j) perm[j] = (int)j;
            std::stable_sort(perm.begin() + w0, perm.begin() + w1, [&](int a, int b) { return rlen(a) > rlen(b); });
        }
        int64_t ml = 0;
        std::vector<int64_t> ss = slice_offsets(perm, ml);
        if ((double)ss[nsl] <= 1.25 * nnzd) {
            ell = true;
            soff = ss;
            maxlen = ml;
        } else {
            perm.clear();
        }
    }
    if (!ell && allow_ell && maxlen <= 32 && (double)soff[nsl] <= 1.2 * nnzd) ell = true;
    // short rows (prolongation, ~4 entries): coalesced sliced ELL beats 1-lane
    // CSR even with ~40% padding (profiles/r01)
    if (!ell && allow_ell && mean <= kShortRowMean && maxlen <= 16 && (double)soff[nsl] <= kShortRowPad * nnzd) {
        ell = true;
        perm.clear();
        soff = slice_offsets(perm, maxlen);
    }
    if (ell) {
        m.fmt = FMT_ELL;
        m.stored = soff[nsl];
        std::vector<int> col(m.stored, 0);
        std::vector<double> val(m.stored, 0.0);
        std::vector<double> sval(colscale ? m.stored : 0, 0.0);
        for (int64_t s = 0; s < nsl; ++s) {
            const int64_t wdt = (soff[s + 1] - soff[s]) / 32;
            for (int64_t j = s * 32; j < std::min(h.nrows, s * 32 + 32); ++j) {
                const int lane = (int)(j - s * 32);
                const int64_t i = perm.empty() ? j : perm[j];
                const int64_t b = h.ptr[i], e = h.ptr[i + 1];
                const int pad_col = e > b ? (int)h.col[e - 1] : 0;
                for (int64_t k = 0; k < wdt; ++k) {
                    const int64_t dst = soff[s] + k * 32 + lane;
                    if (b + k < e) {
                        col[dst] = (int)h.col[b + k];
                        val[dst] = h.val[b + k];
                        if (colscale) sval[dst] = h.val[b + k] * colscale[h.col[b + k]];
                    } else {
                        col[dst] = pad_col;
                    }
                }
            }
        }
        int64_t *d_soff;
        int *d_col;
        double *d_val;
        RC(upload(ctx, &d_soff, soff.data(), nsl + 1));
        RC(upload(ctx, &d_col, col.data(), m.stored));
        RC(upload(ctx, &d_val, val.data(), m.stored));
        m.slice_off = d_soff;
        m.col = d_col;
        m.val = d_val;
        if (!perm.empty()) {
            int *d_perm;
            RC(upload(ctx, &d_perm, perm.data(), h.nrows));
            m.perm = d_perm;
        }
        if (g_use_vcode && allow_vcode) RC(attach_value_codes(ctx, m, val));
        if (perm.empty()) RC(build_pipe(ctx, h, m, soff, bounds, bound_tiles));
        if (colscale) {
            double *d_sval;
            RC(upload(ctx, &d_sval, sval.data(), m.stored));
            *scaled = m;
            scaled->val = d_sval;
        }
    } else {
        m.fmt = FMT_CSR;
        m.stored = m.nnz;
        // lanes per row: about 6 entries per lane, batched kCsrUnroll deep
        int g = 1;
        const int want = (int)std::ceil(mean / (h.nrows < 50000 ? g_small_per_lane : g_csr_per_lane));
        while (g < want && g < 32) g *= 2;
        if (g_csr_g > 0) g = g_csr_g;
        m.group = g;
        // padded by 4 entries so that 16-byte aligned bulk copies may overrun the last row
        std::vector<int> ptr(h.nrows + 1), col(m.nnz + 4, 0);
        std::vector<double> val(m.nnz + 4, 0.0);
        for (int64_t i = 0; i <= h.nrows; ++i) ptr[i] = (int)(h.ptr[i] - h.ptr[0]);
        for (int64_t k = 0; k < m.nnz; ++k) col[k] = (int)h.col[h.ptr[0] + k];
        std::memcpy(val.data(), h.val + h.ptr[0], sizeof(double) * m.nnz);
        int *d_ptr, *d_col;
        double *d_val;
        RC(upload(ctx, &d_ptr, ptr.data(), h.nrows + 1));
        RC(upload(ctx, &d_col, col.data(), m.nnz + 4));
        RC(upload(ctx, &d_val, val.data(), m.nnz + 4));
        m.ptr = d_ptr;
        m.col = d_col;
        m.val = d_val;
        RC(build_pipe(ctx, h, m, soff, bounds, bound_tiles));
        if (colscale) {
            std::vector<double> sval(m.nnz + 4, 0.0);
            for (int64_t k = 0; k < m.nnz; ++k) sval[k] = h.val[h.ptr[0] + k] * colscale[h.col[h.ptr[0] + k]];
            double *d_sval;
            RC(upload(ctx, &d_sval, sval.data(), m.nnz + 4));
            *scaled = m;
            scaled->val = d_sval;
        }
    }
    return DFL_OK;
}

// Row tiles for the TMA pipeline: tiles never straddle `bounds` (subdomain
// starts for the operator); ELL tiles are 256 rows (one per thread), CSR
// tiles ~3K entries in passes of 256/G rows.
static constexpr int kStageBytesMax = 100 * 1024;

static int build_pipe(dfl_ctx *ctx, const HostRows &h, DMat &m, const std::vector<int64_t> &soff,
                      const std::vector<int64_t> &bounds, std::vector<int64_t> *bound_tiles) {
    m.pipe = Pipe{};
    if (bound_tiles) bound_tiles->assign(1, 0);
    if (h.nrows == 0) return DFL_OK;
    int64_t rpt;
    if (m.fmt == FMT_ELL) {
        rpt = kPipeThreads;
    } else {
        const int64_t rpp = kPipeThreads / m.group;
        const double mean = (double)m.nnz / (double)h.nrows;
        const int64_t passes = std::max<int64_t>(1, (int64_t)std::llround(3072.0 / std::max(1.0, mean * rpp)));
        rpt = rpp * passes;
    }
    std::vector<int64_t> r0, r1, e0;
    std::vector<int> ec;
    int64_t cap = 0;
    const int64_t base = h.ptr[0];
    for (size_t bi = 0; bi + 1 < bounds.size(); ++bi) {
        for (int64_t r = bounds[bi]; r < bounds[bi + 1]; r += rpt) {
            const int64_t re = std::min(r + rpt, bounds[bi + 1]);
            int64_t a, b;
            if (m.fmt == FMT_ELL) {
                a = soff[r >> 5];
                b = soff[(re + 31) >> 5];
            } else {
                a = (h.ptr[r] - base) & ~int64_t(3);
                b = ((h.ptr[re] - base) + 3) & ~int64_t(3);
            }
            r0.push_back(r);
            r1.push_back(re);
            e0.push_back(a);
            ec.push_back((int)(b - a));
            cap = std::max(cap, b - a);
        }
        if (bound_tiles) bound_tiles->push_back((int64_t)r0.size());
    }
    cap = (cap + 3) & ~int64_t(3);
    const int64_t stage_bytes = cap * 12;
    int stages = (int)std::min<int64_t>(4, kStageBytesMax / std::max<int64_t>(1, stage_bytes));
    if (stages < 2) return DFL_OK;  // rows too long for staging: register kernels
    int64_t *d0, *d1, *de;
    int *dc;
    RC(upload(ctx, &d0, r0.data(), (int64_t)r0.size()));
    RC(upload(ctx, &d1, r1.data(), (int64_t)r1.size()));
    RC(upload(ctx, &de, e0.data(), (int64_t)e0.size()));
    RC(upload(ctx, &dc, ec.data(), (int64_t)ec.size()));
    m.pipe.row0 = d0;
    m.pipe.row1 = d1;
    m.pipe.e0 = de;
    m.pipe.ecnt = dc;
    m.pipe.ntiles = (int64_t)r0.size();
    m.pipe.cap = (int)cap;
    m.pipe.stages = stages;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// kernel launch helpers

static int rows_per_block(const DMat &A) { return A.fmt == FMT_CSR ? kBlock / A.group : kBlock; }

static int64_t nblocks_for(const DMat &A) { return cdiv(A.nrows, rows_per_block(A)); }

static int g_sm_count = 148;

// grid of the grid-stride FMT_CODE kernels
static int64_t code_grid(const dfl_ctx *, const DMat &A) {
    return std::max<int64_t>(1, std::min<int64_t>(cdiv(A.nrows, kBlock), 8 * (int64_t)g_sm_count));
}

// number of per-block / per-tile partials a row kernel on A produces
static int64_t parts_for(const DMat &A) {
    if (A.fmt == FMT_CODE || A.vcode) return code_grid(nullptr, A);
    return A.pipe.stages ? A.pipe.ntiles : nblocks_for(A);
}

static size_t pipe_smem(const DMat &A) { return 128 + (size_t)A.pipe.stages * A.pipe.cap * 12; }

template <int MODE, bool PART>
static void pipe_attr_one() {
    auto set = [](const void *f) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageBytesMax + 1024);
    };
    set((const void *)k_pipe<0, MODE, PART>);
    set((const void *)k_pipe<1, MODE, PART>);
    set((const void *)k_pipe<2, MODE, PART>);
    set((const void *)k_pipe<4, MODE, PART>);
    set((const void *)k_pipe<8, MODE, PART>);
    set((const void *)k_pipe<16, MODE, PART>);
    set((const void *)k_pipe<32, MODE, PART>);
}

static void pipe_attrs() {
    pipe_attr_one<PMODE_PLAIN, false>();
    pipe_attr_one<PMODE_RESID, false>();
    pipe_attr_one<PMODE_PROLONG, false>();
    pipe_attr_one<PMODE_POST, false>();
    pipe_attr_one<PMODE_POST, true>();
    pipe_attr_one<PMODE_OP, true>();
    pipe_attr_one<PMODE_OPRES, true>();
}

template <int MODE, bool PART>
static bool launch_pipe(dfl_ctx *ctx, const DMat &A, const SpArgs &a) {
    if (A.pipe.stages == 0) return false;
    const size_t smem = pipe_smem(A);
    const int per_sm = smem <= 110 * 1024 ? 2 : 1;
    const unsigned grid = (unsigned)std::min<int64_t>(A.pipe.ntiles, (int64_t)ctx->sm_count * per_sm);
    if (A.fmt == FMT_ELL) {
        k_pipe<0, MODE, PART><<<grid, kPipeThreads, smem, ctx->st>>>(A, a);
    } else {
        switch (A.group) {
            case 1: k_pipe<1, MODE, PART><<<grid, kPipeThreads, smem, ctx->st>>>(A, a); break;
            case 2: k_pipe<2, MODE, PART><<<grid, kPipeThreads, smem, ctx->st>>>(A, a); break;
            case 4: k_pipe<4, MODE, PART><<<grid, kPipeThreads, smem, ctx->st>>>(A, a); break;
            case 8: k_pipe<8, MODE, PART><<<grid, kPipeThreads, smem, ctx->st>>>(A, a); break;
            case 16: k_pipe<16, MODE, PART><<<grid, kPipeThreads, smem, ctx->st>>>(A, a); break;
            default: k_pipe<32, MODE, PART><<<grid, kPipeThreads, smem, ctx->st>>>(A, a); break;
        }
    }
    ctx->launches++;
    return true;
}


template <int MODE, bool DOT>
static void launch_csr_mode(const DMat &A, const RowArgs &a, cudaStream_t st) {
    const dim3 grid((unsigned)nblocks_for(A));
    switch (A.group) {
        case 1: k_csr<1, MODE, DOT><<<grid, kBlock, 0, st>>>(A, a); break;
        case 2: k_csr<2, MODE, DOT><<<grid, kBlock, 0, st>>>(A, a); break;
        case 4: k_csr<4, MODE, DOT><<<grid, kBlock, 0, st>>>(A, a); break;
        case 8: k_csr<8, MODE, DOT><<<grid, kBlock, 0, st>>>(A, a); break;
        case 16: k_csr<16, MODE, DOT><<<grid, kBlock, 0, st>>>(A, a); break;
        default: k_csr<32, MODE, DOT><<<grid, kBlock, 0, st>>>(A, a); break;
    }
}

template <int MODE, bool DOT>
static void launch_rows(dfl_ctx *ctx, const DMat &A, const RowArgs &a) {
    if (A.nrows == 0) return;
    if (A.fmt == FMT_CODE) {
        k_code<MODE, DOT><<<(unsigned)code_grid(ctx, A), kBlock, 0, ctx->st>>>(A, a);
        ctx->launches++;
        return;
    }
    if (A.vcode) {
        k_vell<MODE, DOT><<<(unsigned)code_grid(ctx, A), kBlock, 0, ctx->st>>>(A, a);
        ctx->launches++;
        return;
    }
    if (g_use_pipe) {
        SpArgs s;
        s.x = a.x;
        s.w = a.w;
        s.r = a.r;
        s.xo = a.xo;
        s.out = a.out;
        s.part = a.dot_part;
        s.st = a.st;
        constexpr int PM = MODE == MODE_PLAIN ? PMODE_PLAIN
                           : MODE == MODE_RESID ? PMODE_RESID
                           : MODE == MODE_POST ? PMODE_POST
                                                : PMODE_PROLONG;
        if (launch_pipe<PM, DOT>(ctx, A, s)) return;
    }
    if (A.fmt == FMT_ELL) {
        const unsigned grid = (unsigned)nblocks_for(A);
        switch (A.ell_w) {
            case 3: k_ell<MODE, DOT, 3><<<grid, kBlock, 0, ctx->st>>>(A, a); break;
            case 4: k_ell<MODE, DOT, 4><<<grid, kBlock, 0, ctx->st>>>(A, a); break;
            case 5: k_ell<MODE, DOT, 5><<<grid, kBlock, 0, ctx->st>>>(A, a); break;
            case 6: k_ell<MODE, DOT, 6><<<grid, kBlock, 0, ctx->st>>>(A, a); break;
            case 7: k_ell<MODE, DOT, 7><<<grid, kBlock, 0, ctx->st>>>(A, a); break;
            case 8: k_ell<MODE, DOT, 8><<<grid, kBlock, 0, ctx->st>>>(A, a); break;
            default: k_ell<MODE, DOT, 0><<<grid, kBlock, 0, ctx->st>>>(A, a); break;
        }
    } else
        launch_csr_mode<MODE, DOT>(A, a, ctx->st);
    ctx->launches++;
}

template <int OPMODE>
static void launch_op(dfl_ctx *ctx, const OpArgs &a) {
    const DMat &A = ctx->Aop;
    if (g_use_pipe && !a.skip_rows && !ctx->split) {
        SpArgs s;
        s.x = a.x;
        s.b = a.b;
        s.out = a.y;
        s.part = a.k > 0 ? a.zt_part : nullptr;
        s.zcols = a.zcols;
        s.zn = a.n;
        s.k = a.k;
        s.st = a.st;
        s.need_refresh = a.need_refresh;
        if (launch_pipe<OPMODE == 0 ? PMODE_OP : PMODE_OPRES, true>(ctx, A, s)) return;
    }
    const unsigned grid = (unsigned)ctx->ntiles;
    if (grid == 0) return;
    if (A.fmt == FMT_CODE) {
        k_op_code<OPMODE><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, ctx->subtab, a);
    } else if (A.fmt == FMT_ELL) {
        const SubTable &S = ctx->subtab;
        switch (A.ell_w) {
            case 5: k_op_ell<OPMODE, 5><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, S, a); break;
            case 6: k_op_ell<OPMODE, 6><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, S, a); break;
            case 7: k_op_ell<OPMODE, 7><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, S, a); break;
            default: k_op_ell<OPMODE, 0><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, S, a); break;
        }
    } else {
        switch (A.group) {
            case 1: k_op_csr<1, OPMODE><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, ctx->subtab, a); break;
            case 2: k_op_csr<2, OPMODE><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, ctx->subtab, a); break;
            case 4: k_op_csr<4, OPMODE><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, ctx->subtab, a); break;
            case 8: k_op_csr<8, OPMODE><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, ctx->subtab, a); break;
            case 16: k_op_csr<16, OPMODE><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, ctx->subtab, a); break;
            default: k_op_csr<32, OPMODE><<<grid, kBlock, 0, ctx->st>>>(A, ctx->tiles, ctx->subtab, a); break;
        }
    }
    ctx->launches++;
}

// ---------------------------------------------------------------------------
// communication (no-ops on a single rank)

static int nccl_check(dfl_ctx *ctx, int rc, const char *what) {
    if (rc != 0) {
        ctx->err = std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(rc) : "nccl error");
        return DFL_E_COMM;
    }
    return DFL_OK;
}

static bool multi(const dfl_ctx *ctx) { return ctx->comm != nullptr || ctx->fab != nullptr; }

// allgather of `count` doubles per rank into recv[q * count] (send may alias
// recv + rank * count)
static int comm_allgather(dfl_ctx *ctx, const double *send, double *recv, size_t count) {
    if (ctx->comm) return nccl_check(ctx, g_nccl.AllGather(send, recv, count, ncclDouble_, ctx->comm, ctx->st), "ncclAllGather");
    dfl_fabric *f = ctx->fab;
    CK(cudaStreamSynchronize(ctx->st));
    f->pub[ctx->rank] = send;
    f->barrier();
    for (int q = 0; q < ctx->nranks; ++q) {
        double *dst = recv + (size_t)q * count;
        if (f->pub[q] != dst) CK(cudaMemcpyAsync(dst, f->pub[q], count * sizeof(double), cudaMemcpyDefault, ctx->st));
    }
    CK(cudaStreamSynchronize(ctx->st));
    f->barrier();
    return DFL_OK;
}

// fill the ghost part v[n .. n+n_ghost) from the neighbours (runtime.py:246-271)
// pack on ctx->st; the NCCL transfers run on `xs` (ctx->st, or the comm
// stream when the operator overlaps them with its interior rows)
static int halo(dfl_ctx *ctx, double *v, cudaStream_t xs = nullptr) {
    if (!multi(ctx) || (ctx->nbr.empty() && !ctx->fab)) return DFL_OK;
    if (!xs) xs = ctx->st;
    if (ctx->nsend > 0) {
        k_gather<<<(unsigned)cdiv(ctx->nsend, kBlock), kBlock, 0, ctx->st>>>(v, ctx->send_idx, ctx->nsend,
                                                                              ctx->sendbuf);
        ctx->launches++;
    }
    if (xs != ctx->st && !ctx->fab) {
        CK(cudaEventRecord(ctx->ev_packed, ctx->st));
        CK(cudaStreamWaitEvent(xs, ctx->ev_packed, 0));
    }
    if (ctx->fab) {  // every rank takes part in the barriers, neighbours or not
        dfl_fabric *f = ctx->fab;
        CK(cudaStreamSynchronize(ctx->st));
        f->pub[ctx->rank] = ctx->sendbuf;
        f->barrier();
        int64_t ro = 0;
        for (size_t qi = 0; qi < ctx->nbr.size(); ++qi) {
            const dfl_ctx *peer = f->ctxs[ctx->nbr[qi]];
            int64_t off = 0, cnt = -1;
            for (size_t j = 0; j < peer->nbr.size(); ++j) {
                if (peer->nbr[j] == ctx->rank) {
                    cnt = peer->send_cnt[j];
                    break;
                }
                off += peer->send_cnt[j];
            }
            if (cnt != ctx->recv_cnt[qi]) {
                ctx->err = "halo plan mismatch between ranks";
                f->barrier();
                return DFL_E_COMM;
            }
            if (cnt > 0)
                CK(cudaMemcpyAsync(v + ctx->n + ro, f->pub[ctx->nbr[qi]] + off, cnt * sizeof(double), cudaMemcpyDefault,
                                   ctx->st));
            ro += ctx->recv_cnt[qi];
        }
        CK(cudaStreamSynchronize(ctx->st));
        f->barrier();
        return DFL_OK;
    }
    RC(nccl_check(ctx, g_nccl.GroupStart(), "ncclGroupStart"));
    int64_t so = 0, ro = 0;
    for (size_t q = 0; q < ctx->nbr.size(); ++q) {
        if (ctx->send_cnt[q] > 0)
            RC(nccl_check(ctx, g_nccl.Send(ctx->sendbuf + so, ctx->send_cnt[q], ncclDouble_, ctx->nbr[q], ctx->comm, xs),
                          "ncclSend"));
        if (ctx->recv_cnt[q] > 0)
            RC(nccl_check(ctx, g_nccl.Recv(v + ctx->n + ro, ctx->recv_cnt[q], ncclDouble_, ctx->nbr[q], ctx->comm, xs),
                          "ncclRecv"));
        so += ctx->send_cnt[q];
        ro += ctx->recv_cnt[q];
    }
    RC(nccl_check(ctx, g_nccl.GroupEnd(), "ncclGroupEnd"));
    return DFL_OK;
}

// Z' v partials -> t (global numbering) -> t2 = E^-1 t on every rank
static int zt_to_t2(dfl_ctx *ctx, const KState *st, int need_refresh, bool from_op) {
    const int64_t *sub_tiles =
        (from_op && g_use_pipe && !ctx->split && ctx->Aop.pipe.stages) ? ctx->op_sub_tiles : ctx->sub_tiles;
    if (!multi(ctx)) {
        k_zt_finish<<<ctx->nsub * ctx->k, 512, 0, ctx->st>>>(ctx->zt_part, sub_tiles, ctx->nsub, ctx->k,
                                                             ctx->tvec, 0, ctx->inexact ? nullptr : ctx->Einv,
                                                             ctx->K, ctx->t2, st, need_refresh, ctx->ticket,
                                                             from_op && ctx->split ? ctx->sub_btiles : nullptr,
                                                             ctx->ntiles);
        ctx->launches++;
        if (ctx->inexact) {
            k_egmres<<<1, 256, 0, ctx->st>>>(ctx->Edense, (int)ctx->K, ctx->tvec, ctx->t2, ctx->coarse_tol,
                                             ctx->egm_scr, st, need_refresh);
            ctx->launches++;
        }
        return DFL_OK;
    }
    // local entries into a padded slot, allgather, unpack, solve
    const int64_t slot = (int64_t)ctx->max_nsub * ctx->k;
    double *mine = ctx->tgather + (int64_t)ctx->rank * slot;
    k_zt_finish<<<ctx->nsub * ctx->k, 512, 0, ctx->st>>>(ctx->zt_part, sub_tiles, ctx->nsub, ctx->k, mine, 0,
                                                         nullptr, ctx->K, nullptr, st, need_refresh, ctx->ticket,
                                                         from_op && ctx->split ? ctx->sub_btiles : nullptr,
                                                         ctx->ntiles);
    RC(comm_allgather(ctx, mine, ctx->tgather, slot));
    // unpack rank slots into t: rank q owns a contiguous subdomain range
    int64_t pos = 0;
    for (int q = 0; q < ctx->nranks; ++q) {
        const int64_t cnt = (int64_t)ctx->rank_nsub[q] * ctx->k;
        if (cnt > 0) CK(cudaMemcpyAsync(ctx->tvec + pos, ctx->tgather + q * slot, cnt * sizeof(double),
                                        cudaMemcpyDeviceToDevice, ctx->st));
        pos += cnt;
    }
    if (ctx->inexact)
        k_egmres<<<1, 256, 0, ctx->st>>>(ctx->Edense, (int)ctx->K, ctx->tvec, ctx->t2, ctx->coarse_tol, ctx->egm_scr,
                                         st, need_refresh);
    else
        k_esolve<<<1, 256, 0, ctx->st>>>(ctx->Einv, ctx->K, ctx->tvec, ctx->t2, st, need_refresh);
    ctx->launches += 2;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// Krylov scalar steps (single block).  With several ranks the per-rank sums
// arrive allgathered in `gath` (stride 8) and are added in rank order, which
// mirrors the ascending-order allreduce of runtime.py:214-219.

__device__ __forceinline__ double scalar_in(const double *part, int64_t nparts, const double *gath, int nranks,
                                            int slot) {
    if (gath == nullptr) return reduce_parts(part, nparts);
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += gath[q * 8 + slot];
    return s;
}

// bnorm = ||b|| (deflation.py:266), atol = tol * bnorm
__global__ void k_cg_start(KState *st, const double *part, int64_t nparts, const double *gath, int nranks,
                           double tol, int maxiter, int refresh) {
    const double bb = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    KState s{};
    s.bnorm = sqrt(fmax(bb, 0.0));
    s.target = tol * s.bnorm;
    s.maxiter = maxiter;
    s.refresh_every = refresh;
    if (s.bnorm == 0.0) {
        s.done = 1;
        s.converged = 1;
    }
    *st = s;
}

// ||b'|| of the projected rhs: zero -> zero solution; r = b' meets the target
// -> converged at 0 iterations (krylov.py:101-113)
__global__ void k_cg_init_r(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double bb = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    const double bn = sqrt(fmax(bb, 0.0));
    st->resnorm = bn;
    if (bn == 0.0 || bn <= st->target) {
        st->done = 1;
        st->converged = 1;
    } else if (st->maxiter <= 0) {
        st->done = 1;
    }
}

__global__ void k_cg_init_rz(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double rz = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x == 0) st->rz = rz;
}

// iters += 1; pAp (krylov.py:119-126)
__global__ void k_cg_pq(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double pq = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    st->iters += 1;
    st->pq = pq;
    if (pq <= 0.0 || !isfinite(pq)) {
        st->breakdown = DFL_BRK_CURVATURE;
        st->done = 1;
        return;
    }
    st->alpha = st->rz / pq;
    st->refresh_now = (st->iters % st->refresh_every) == 0;
}

// resnorm test (krylov.py:132-136)
__global__ void k_cg_rr(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double rr = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    st->rr = rr;
    st->resnorm = sqrt(fmax(rr, 0.0));
    if (st->resnorm <= st->target) {
        st->converged = 1;
        st->done = 1;
    }
}

// beta (krylov.py:138-143)
__global__ void k_cg_rz(KState *st, const double *part, int64_t nparts, const double *gath, int nranks) {
    if (st->done) return;
    const double rz = scalar_in(part, nparts, gath, nranks, 0);
    if (threadIdx.x != 0) return;
    if (rz == 0.0 || !isfinite(rz)) {
        st->breakdown = DFL_BRK_RZ;
        st->done = 1;
        return;
    }
    st->beta = rz / st->rz;
    st->rz = rz;
}

// multi-rank: r.r and r.z arrive in one allgather (slots 0 and 1); the
// convergence test uses r.r exactly as k_cg_rr, then beta as k_cg_rz
__global__ void k_cg_rrz(KState *st, const double *gath, int nranks) {
    if (st->done || threadIdx.x != 0) return;
    double rr = 0.0, rz = 0.0;
    for (int q = 0; q < nranks; ++q) {
        rr += gath[q * 8 + 0];
        rz += gath[q * 8 + 1];
    }
    st->rr = rr;
    st->resnorm = sqrt(fmax(rr, 0.0));
    if (st->resnorm <= st->target) {
        st->converged = 1;
        st->done = 1;
        return;
    }
    if (rz == 0.0 || !isfinite(rz)) {
        st->breakdown = DFL_BRK_RZ;
        st->done = 1;
        return;
    }
    st->beta = rz / st->rz;
    st->rz = rz;
}

__global__ void k_cg_end(KState *st, cudaGraphConditionalHandle h, int use_cond) {
    if (threadIdx.x != 0) return;
    if (!st->done && st->iters >= st->maxiter) st->done = 1;
    if (use_cond) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

// ---------------------------------------------------------------------------
// reductions across ranks: returns the pointer the scalar kernel reads
static int rank_scalar(dfl_ctx *ctx, const double *part, int64_t nparts, int slot, const double **gath) {
    *gath = nullptr;
    if (!multi(ctx)) return DFL_OK;
    k_reduce<<<1, 1024, 0, ctx->st>>>(part, nparts, ctx->scal + slot);
    ctx->launches++;
    RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
    *gath = ctx->sgather;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// V-cycle over all groups: z = M r  (deflation.py:239-250 -> amg.py:201-212).
// With dot_part != nullptr the last kernel of every group also emits the
// per-block partials of r.z; *nparts receives their count.
static int vcycle(dfl_ctx *ctx, const double *r, double *z, const KState *st, double *dot_part, int64_t *nparts) {
    int64_t poff = 0;
    for (VGroup &g : ctx->groups) {
        const double *rin = r + g.row0;
        double *zout = z + g.row0;
        const int L = (int)g.lv.size();
        const bool use_coarse = g.lc >= 0 && g_use_coarse;
        const bool use_tiny = !use_coarse && g.lt >= 0 && g_use_tiny;
        const int lc = use_coarse ? g.lc : use_tiny ? g.lt : L + 1;  // first level of the fused tail kernel
        for (int l = 0; l < std::min(L, lc); ++l) {
            DLevel &v = g.lv[l];
            const double *in = l == 0 ? rin : v.rv;
            double *next = (l + 1 < L) ? g.lv[l + 1].rv : g.rb;
            if (v.A.fmt == FMT_CODE) {
                k_wr<<<(unsigned)cdiv(v.n, kBlock), kBlock, 0, ctx->st>>>(v.w, in, v.wr, v.n);
                ctx->launches++;
                RowArgs a{v.wr, v.w, in, nullptr, v.t, nullptr, st};
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
        if (lc <= L) {
            const double *crin = lc == 0 ? rin : g.lv[lc < L ? lc : 0].rv;
            double *cxout = lc == 0 ? zout : g.lv[lc < L ? lc : 0].xv;
            if (lc == L && L > 0) {  // bottom only
                crin = g.rb;
                cxout = g.xb;
            }
            if (use_tiny) {
                k_tiny_cycle<<<kTinyCtas, kTinyThreads, 0, ctx->st>>>(g.targs, crin, cxout);
                ctx->launches++;
                prof_mark(ctx, "tiny L" + std::to_string(lc) + "+");
            } else {
                void *args[] = {(void *)&g.cargs, (void *)&crin, (void *)&cxout};
                cudaLaunchCooperativeKernel((const void *)k_coarse_cycle, g.coarse_grid, 256, args, 0, ctx->st);
                ctx->launches++;
                prof_mark(ctx, "coarse L" + std::to_string(lc) + "+");
            }
        } else {
            const double *rb = L == 0 ? rin : g.rb;
            double *xb = L == 0 ? zout : g.xb;
            k_bottom<<<dim3((unsigned)cdiv(g.max_nb, 32), (unsigned)g.nsub), 256, 0, ctx->st>>>(
                g.binvT, g.binv_off, g.b_off, rb, xb, st);
            ctx->launches++;
            prof_mark(ctx, "bottom");
        }
        for (int l = std::min(L, lc) - 1; l >= 0; --l) {
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
        if ((L == 0 || lc == 0) && dot_part) {
            // the group's finest level ran without a fused dot: explicit partials
            const int64_t rows = g.row1 - g.row0;
            const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(rows, kBlock), 64));
            k_dot<<<nb, kBlock, 0, ctx->st>>>(rin, zout, rows, dot_part + poff, st);
            ctx->launches++;
            poff += nb;
        }
    }
    if (nparts) *nparts = poff;
    return DFL_OK;
}

// y = A x (opmode 0) or y = b - A x (opmode 1); with zt the Z'y tile partials
static int op_apply_dev(dfl_ctx *ctx, double *xin, double *y, int opmode, const double *b, bool zt,
                        const KState *st, int need_refresh) {
    OpArgs a{xin, b, y, ctx->zcols, ctx->n, zt ? ctx->k : 0, ctx->zt_part, st, need_refresh};
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
    if (!ctx->fab) {
        CK(cudaEventRecord(ctx->ev_halo, ctx->st2));
        CK(cudaStreamWaitEvent(ctx->st, ctx->ev_halo, 0));
    }
    a.skip_rows = nullptr;
    if (ctx->nbtiles > 0) {
        if (opmode == 0)
            k_op_bnd<0><<<(unsigned)ctx->nbtiles, kBlock, 0, ctx->st>>>(ctx->Aop, ctx->brows, ctx->bstart, ctx->bcnt,
                                                                         ctx->ntiles, a);
        else
            k_op_bnd<1><<<(unsigned)ctx->nbtiles, kBlock, 0, ctx->st>>>(ctx->Aop, ctx->brows, ctx->bstart, ctx->bcnt,
                                                                         ctx->ntiles, a);
        ctx->launches++;
    }
    return DFL_OK;
}

static ProjArgs proj_args(dfl_ctx *ctx, const double *in, double *out, const KState *st) {
    ProjArgs a{};
    if (ctx->deflation) {
        a.az_ptr = ctx->az_ptr;
        a.az_col = ctx->az_col;
        a.az_val = ctx->az_val;
    }
    a.t2 = ctx->t2;
    a.K = ctx->deflation ? ctx->K : 0;
    a.n = ctx->n;
    a.in = in;
    a.out = out;
    a.st = st;
    return a;
}

template <int MODE>
static void launch_project(dfl_ctx *ctx, const ProjArgs &a) {
    k_project<MODE><<<(unsigned)ctx->nblk, kBlock, sizeof(double) * std::max<int64_t>(1, a.K), ctx->st>>>(a);
    ctx->launches++;
}

// out = project(v) = v - AZ E^-1 Z' v   (deflation.py:230-233)
static int project_dev(dfl_ctx *ctx, const double *v, double *out, const KState *st, int dotmode) {
    k_zt_vec<<<(unsigned)ctx->ntiles, kBlock, 0, ctx->st>>>(ctx->tiles, v, ctx->zcols, ctx->n, ctx->k, ctx->zt_part);
    ctx->launches++;
    RC(zt_to_t2(ctx, nullptr, 0, false));
    ProjArgs a = proj_args(ctx, v, out, st);
    a.dotmode = dotmode;
    a.dot_part = ctx->dpart;
    launch_project<0>(ctx, a);
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// one CG iteration (krylov.py:119-143) on the projected operator
static int cg_body(dfl_ctx *ctx, bool deflated, cudaGraphConditionalHandle h, int use_cond) {
    KState *st = ctx->state;
    const double *gath;
    // w = A p, Z'w ; t2 ; q = w - AZ t2 ; p.q
    RC(op_apply_dev(ctx, ctx->p, ctx->w, 0, nullptr, deflated, st, 0));
    if (deflated) RC(zt_to_t2(ctx, st, 0, true));
    {
        ProjArgs a = proj_args(ctx, ctx->w, ctx->w, st);
        if (!deflated) a.az_ptr = nullptr, a.K = 0;
        a.dotmode = 1;
        a.dotv = ctx->p;
        a.dot_part = ctx->dpart;
        launch_project<0>(ctx, a);
    }
    RC(rank_scalar(ctx, ctx->dpart, ctx->nblk, 0, &gath));
    k_cg_pq<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, gath, ctx->nranks);
    ctx->launches++;
    // x += alpha p ; r -= alpha q (regular iterations)
    k_cg_update<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->x, ctx->r, ctx->p, ctx->w, ctx->n, ctx->dpart, st);
    ctx->launches++;
    // refresh iterations: r = b' - project(A x)   (krylov.py:128-129)
    RC(op_apply_dev(ctx, ctx->x, ctx->tmp, 0, nullptr, deflated, st, 1));
    if (deflated) RC(zt_to_t2(ctx, st, 1, true));
    {
        ProjArgs a = proj_args(ctx, ctx->tmp, ctx->r, st);
        if (!deflated) a.az_ptr = nullptr, a.K = 0;
        a.base = ctx->bp;
        a.dotmode = 2;
        a.dot_part = ctx->dpart;
        a.need_refresh = 1;
        launch_project<1>(ctx, a);
    }
    int64_t np = 0;
    if (multi(ctx)) {
        // one collective for r.r and r.z: the V-cycle runs before the
        // convergence test (its result is discarded on the last iteration)
        k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->dpart, ctx->nblk, ctx->scal + 0);
        RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
        k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->dpart, np, ctx->scal + 1);
        RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
        k_cg_rrz<<<1, 32, 0, ctx->st>>>(st, ctx->sgather, ctx->nranks);
        ctx->launches += 3;
    } else {
        k_cg_rr<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, nullptr, 1);
        ctx->launches++;
        // z = M r, r.z
        RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
        k_cg_rz<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, np, nullptr, 1);
        ctx->launches++;
    }
    k_cg_p<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->p, ctx->z, ctx->n, st);
    ctx->launches++;
    k_cg_end<<<1, 32, 0, ctx->st>>>(st, h, use_cond);
    ctx->launches++;
    return DFL_OK;
}

static int build_loop_graph(dfl_ctx *ctx, bool deflated) {
    const int key = deflated ? 1 : 0;
    if (ctx->loop_exec && ctx->loop_key == key) return DFL_OK;
    if (ctx->loop_exec) {
        cudaGraphExecDestroy(ctx->loop_exec);
        ctx->loop_exec = nullptr;
    }
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(ctx->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t before = ctx->launches;
    int rc = cg_body(ctx, deflated, h, 1);
    cudaGraph_t captured = nullptr;
    cudaError_t ce = cudaStreamEndCapture(ctx->st, &captured);
    if (rc != DFL_OK) return rc;
    CK(ce);
    ctx->body_kernels = ctx->launches - before;
    ctx->launches = before;
    CK(cudaGraphInstantiate(&ctx->loop_exec, g, 0));
    cudaGraphDestroy(g);
    ctx->loop_key = key;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// the whole solve on the device: b, x in ctx->b / ctx->xin
static int lift_dev(dfl_ctx *ctx, const dfl_solve_params *p);

static int cg_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, bool use_graph) {
    KState *st = ctx->state;
    const bool defl = p->deflated != 0;
    const double *gath;
    // x = 0 (y of the deflated system)
    k_fill<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->x, 0.0, ctx->n);
    // ||b||
    k_dot<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->b, ctx->b, ctx->n, ctx->dpart, nullptr);
    ctx->launches += 2;
    RC(rank_scalar(ctx, ctx->dpart, ctx->nblk, 0, &gath));
    k_cg_start<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, gath, ctx->nranks, p->tol, p->maxiter,
                                      std::max(1, p->refresh_every));
    ctx->launches++;
    // b' = project(b) and ||b'||^2
    if (defl) {
        RC(project_dev(ctx, ctx->b, ctx->bp, nullptr, 2));
    } else {
        ProjArgs a = proj_args(ctx, ctx->b, ctx->bp, nullptr);
        a.az_ptr = nullptr;
        a.K = 0;
        a.dotmode = 2;
        a.dot_part = ctx->dpart;
        launch_project<0>(ctx, a);
    }
    RC(rank_scalar(ctx, ctx->dpart, ctx->nblk, 0, &gath));
    k_cg_init_r<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, ctx->nblk, gath, ctx->nranks);
    k_copy<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->r, ctx->bp, ctx->n);
    ctx->launches += 2;
    int64_t np = 0;
    RC(vcycle(ctx, ctx->r, ctx->z, st, ctx->dpart, &np));
    RC(rank_scalar(ctx, ctx->dpart, np, 0, &gath));
    k_cg_init_rz<<<1, 1024, 0, ctx->st>>>(st, ctx->dpart, np, gath, ctx->nranks);
    k_copy<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->p, ctx->z, ctx->n);
    ctx->launches += 2;
    // the loop
    if (use_graph) {
        RC(build_loop_graph(ctx, defl));
        CK(cudaGraphLaunch(ctx->loop_exec, ctx->st));
    } else {
        for (;;) {
            RC(cg_body(ctx, defl, 0, 0));
            CK(cudaMemcpyAsync(ctx->h_state, st, sizeof(KState), cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            if (ctx->h_state->done) break;
        }
    }
    return lift_dev(ctx, p);
}

// x = y + Z E^-1 Z'(b - A y)   (deflation.py:285); y in ctx->x, x -> ctx->xin
static int lift_dev(dfl_ctx *ctx, const dfl_solve_params *p) {
    if (p->deflated) {
        RC(op_apply_dev(ctx, ctx->x, ctx->tmp, 1, ctx->b, true, nullptr, 0));
        RC(zt_to_t2(ctx, nullptr, 0, true));
        k_lift<<<(unsigned)ctx->ntiles, kBlock, 0, ctx->st>>>(ctx->tiles, ctx->tile_sub, ctx->x, ctx->zcols, ctx->n,
                                                              ctx->k, ctx->t2, (int64_t)ctx->first_sub * ctx->k,
                                                              ctx->xin, 1);
    } else {
        k_copy<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->xin, ctx->x, ctx->n);
    }
    ctx->launches++;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// BiCGStab(2) (krylov.py:148-285), right preconditioned: op_hat = op o M with
// op = project o A.  Host-driven: scalars are computed on the host in IEEE
// double with the reference's expressions; every dot is a device reduction
// read back at its branch point.

static int fetch(dfl_ctx *ctx, const double *dev, int n, double *out) {
    CK(cudaMemcpyAsync(ctx->h_dots, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    for (int q = 0; q < n; ++q) out[q] = ctx->h_dots[q];
    return DFL_OK;
}

// global value of nq interleaved (stride 3) or plain (nq == 0 -> 1 stream) partials
static int global_dots(dfl_ctx *ctx, const double *part, int64_t nparts, int nq, bool strided, double *out) {
    if (strided)
        k_reduceq<<<1, 1024, 0, ctx->st>>>(part, nparts, nq, ctx->scal);
    else
        k_reduce<<<1, 1024, 0, ctx->st>>>(part, nparts, ctx->scal);
    ctx->launches++;
    if (multi(ctx)) {
        RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
        k_rank_sum<<<1, 32, 0, ctx->st>>>(ctx->sgather, ctx->nranks, 8, nq, ctx->scal + 8);
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
    k_multidot<<<g, kBlock, 0, ctx->st>>>(a0, b0, a1, b1, a2, b2, a3, b3, nq, ctx->n, ctx->dpart);
    ctx->launches++;
    return global_dots(ctx, ctx->dpart, g, nq, true, out);
}

// out = op_hat(v) = project(A (M v)); with dotv: also returns dot(out, dotv)
static int op_hat(dfl_ctx *ctx, bool defl, const double *v, double *out, const double *dotv, double *dot_out) {
    RC(vcycle(ctx, v, ctx->zx, nullptr, nullptr, nullptr));
    RC(op_apply_dev(ctx, ctx->zx, ctx->w, 0, nullptr, defl, nullptr, 0));
    if (defl) RC(zt_to_t2(ctx, nullptr, 0, true));
    ProjArgs a = proj_args(ctx, ctx->w, out, nullptr);
    if (!defl) a.az_ptr = nullptr, a.K = 0;
    if (dotv) {
        a.dotmode = 1;
        a.dotv = dotv;
        a.dot_part = ctx->dpart;
    }
    launch_project<0>(ctx, a);
    if (dotv) RC(global_dots(ctx, ctx->dpart, ctx->nblk, 1, false, dot_out));
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

static int bicg_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, KState &out) {
    RC(bicg_alloc(ctx));
    const bool defl = p->deflated != 0;
    const int64_t n = ctx->n;
    const unsigned nb = (unsigned)ctx->nblk;
    out = KState{};
    double val[3];
    // ||b|| (deflation.py:266), b' = project(b), ||b'||
    RC(dots(ctx, 1, ctx->b, ctx->b, nullptr, nullptr, nullptr, nullptr, val));
    out.bnorm = std::sqrt(std::max(val[0], 0.0));
    const double target = std::max(0.0, p->tol * out.bnorm);  // max(tol*||b'||, atol) with tol = 0
    out.target = target;
    k_fill<<<nb, kBlock, 0, ctx->st>>>(ctx->bu, 0.0, n);
    ctx->launches++;
    if (out.bnorm == 0.0) {
        out.converged = 1;
        k_fill<<<nb, kBlock, 0, ctx->st>>>(ctx->x, 0.0, n);
        ctx->launches++;
        return DFL_OK;
    }
    if (defl) {
        RC(project_dev(ctx, ctx->b, ctx->bp, nullptr, 0));
    } else {
        k_copy<<<nb, kBlock, 0, ctx->st>>>(ctx->bp, ctx->b, n);
        ctx->launches++;
    }
    RC(dots(ctx, 1, ctx->bp, ctx->bp, nullptr, nullptr, nullptr, nullptr, val));
    const double bpbp = val[0];  // also r[0].shadow of the first step (both are b')
    const double bpn = std::sqrt(std::max(val[0], 0.0));
    if (bpn == 0.0) {  // bicgstab2 returns zeros (krylov.py:270-272)
        out.converged = 1;
        k_fill<<<nb, kBlock, 0, ctx->st>>>(ctx->x, 0.0, n);
        ctx->launches++;
        return DFL_OK;
    }
    double *r[3] = {ctx->br[0], ctx->br[1], ctx->br[2]};
    double *d[3] = {ctx->bd[0], ctx->bd[1], ctx->bd[2]};
    double *u = ctx->bu, *shadow = ctx->bshadow;
    const double *r0init = ctx->bp;
    k_copy<<<nb, kBlock, 0, ctx->st>>>(r[0], r0init, n);
    k_fill<<<nb, kBlock, 0, ctx->st>>>(d[0], 0.0, n);
    k_copy<<<nb, kBlock, 0, ctx->st>>>(shadow, r0init, n);
    ctx->launches += 3;
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
        k_copy<<<nb, kBlock, 0, ctx->st>>>(shadow, r[0], n);
        k_fill<<<nb, kBlock, 0, ctx->st>>>(d[0], 0.0, n);
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
            k_bicg_d<<<nb, kBlock, 0, ctx->st>>>(r[0], d[0], r[1], d[1], j + 1, beta, n);
            ctx->launches++;
            double gd;
            RC(op_hat(ctx, defl, d[j], d[j + 1], shadow, &gd));
            if (gd == 0.0 || !std::isfinite(gd)) {
                brk = fail(DFL_BRK_SHADOW);
                aborted = true;
                break;
            }
            alpha = rho0 / gd;
            k_bicg_r<<<nb, kBlock, 0, ctx->st>>>(r[0], d[1], r[1], d[2], j + 1, u, d[0], alpha, n, ctx->dpart);
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
            k_bicg_mr2<<<g, kBlock, 0, ctx->st>>>(r[2], r[1], r[0], tau12, n, ctx->dpart);
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
        k_bicg_final<<<nb, kBlock, 0, ctx->st>>>(u, r[0], d[0], r[1], r[2], d[1], d[2], g1, gp2, g2, gpp1, gp1, n,
                                                 ctx->dpart);
        ctx->launches++;
        if (iters % refresh == 0) {
            // r[0] = r0 - op_hat(u)   (krylov.py:256-257)
            RC(op_hat(ctx, defl, u, ctx->tmp, nullptr, nullptr));
            ProjArgs a = proj_args(ctx, ctx->tmp, r[0], nullptr);
            a.az_ptr = nullptr;
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

static constexpr int kGmLd = 128;  // max restart + 1

static int gm_alloc(dfl_ctx *ctx, int restart, bool flexible) {
    if (restart < 1 || restart + 1 > kGmLd) {
        ctx->err = "solver.M (GMRES restart) must be in [1, " + std::to_string(kGmLd - 1) + "]";
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
    if (!ctx->gmVp) {
        RC(dalloc(ctx, (double **)&ctx->gmVp, kGmLd));
        RC(dalloc(ctx, (double **)&ctx->gmZp, kGmLd));
        RC(dalloc(ctx, &ctx->gm_h, kGmLd));
        RC(dalloc(ctx, &ctx->gm_e, kGmLd));
        RC(dalloc(ctx, &ctx->gm_y, kGmLd));
        RC(dalloc(ctx, &ctx->gm_loc, kGmLd));
        RC(dalloc(ctx, &ctx->gm_gath, (int64_t)kGmLd * ctx->nranks));
        RC(dalloc(ctx, &ctx->gm_part, (int64_t)kGmLd * 4 * ctx->sm_count));
        CK(cudaMallocHost(&ctx->h_gm, 4 * kGmLd * sizeof(double)));
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
    k_vdots<<<grid, kBlock, 0, ctx->st>>>(ctx->gmVp, nvec, w, ctx->n, ctx->gm_part, kGmLd);
    ctx->launches++;
    if (!multi(ctx)) {
        k_vreduce<<<nvec, 1024, 0, ctx->st>>>(ctx->gm_part, gx, kGmLd, dev_out);
        ctx->launches++;
        return DFL_OK;
    }
    k_vreduce<<<nvec, 1024, 0, ctx->st>>>(ctx->gm_part, gx, kGmLd, ctx->gm_loc);
    RC(comm_allgather(ctx, ctx->gm_loc, ctx->gm_gath, kGmLd));
    k_rank_sum<<<1, kGmLd, 0, ctx->st>>>(ctx->gm_gath, ctx->nranks, kGmLd, nvec, dev_out);
    ctx->launches += 2;
    return DFL_OK;
}

// r = b' - project(A x), returns ||r||   (krylov.py:408)
static int gm_residual(dfl_ctx *ctx, bool defl, double *resnorm) {
    RC(op_apply_dev(ctx, ctx->x, ctx->w, 0, nullptr, defl, nullptr, 0));
    if (defl) RC(zt_to_t2(ctx, nullptr, 0, true));
    ProjArgs a = proj_args(ctx, ctx->w, ctx->r, nullptr);
    if (!defl) a.az_ptr = nullptr, a.K = 0;
    a.base = ctx->bp;
    a.dotmode = 2;
    a.dot_part = ctx->dpart;
    launch_project<1>(ctx, a);
    double v[4];
    RC(global_dots(ctx, ctx->dpart, ctx->nblk, 1, false, v));
    *resnorm = std::sqrt(std::max(v[0], 0.0));
    return DFL_OK;
}

static int gmres_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, bool flexible, KState &out) {
    const bool defl = p->deflated != 0;
    const int M = p->restart > 0 ? p->restart : 50;
    RC(gm_alloc(ctx, M, flexible));
    const int64_t n = ctx->n;
    const unsigned nb = (unsigned)ctx->nblk;
    const unsigned gx = (unsigned)std::min<int64_t>(std::max<int64_t>(1, ctx->nblk), 4 * ctx->sm_count);
    out = KState{};
    double val[4];
    RC(dots(ctx, 1, ctx->b, ctx->b, nullptr, nullptr, nullptr, nullptr, val));
    out.bnorm = std::sqrt(std::max(val[0], 0.0));
    const double target = std::max(0.0, p->tol * out.bnorm);
    out.target = target;
    k_fill<<<nb, kBlock, 0, ctx->st>>>(ctx->x, 0.0, n);
    ctx->launches++;
    if (out.bnorm == 0.0) {
        out.converged = 1;
        return DFL_OK;
    }
    if (defl) {
        RC(project_dev(ctx, ctx->b, ctx->bp, nullptr, 0));
    } else {
        k_copy<<<nb, kBlock, 0, ctx->st>>>(ctx->bp, ctx->b, n);
        ctx->launches++;
    }
    RC(dots(ctx, 1, ctx->bp, ctx->bp, nullptr, nullptr, nullptr, nullptr, val));
    double resnorm = std::sqrt(std::max(val[0], 0.0));
    if (resnorm == 0.0) {
        out.converged = 1;
        return DFL_OK;
    }
    k_copy<<<nb, kBlock, 0, ctx->st>>>(ctx->r, ctx->bp, n);
    ctx->launches++;
    std::vector<double> H((size_t)(M + 1) * M), g(M + 1), cs(M), sn(M), y(M);
    auto h = [&](int i, int j) -> double & { return H[(size_t)i * M + j]; };
    int total = 0;
    while (total < p->maxiter && resnorm > target) {
        const int steps = std::min(M, p->maxiter - total);
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = resnorm;
        k_vdiv<<<nb, kBlock, 0, ctx->st>>>(ctx->gmV[0], ctx->r, resnorm, n);  // V0 = r0 / ||r0||
        ctx->launches++;
        int j = 0;
        while (j < steps) {
            double *w = ctx->w;
            if (flexible) {  // z_j = M(V_j), w = project(A z_j)
                RC(vcycle(ctx, ctx->gmV[j], ctx->gmZ[j], nullptr, nullptr, nullptr));
                RC(op_apply_dev(ctx, ctx->gmZ[j], w, 0, nullptr, defl, nullptr, 0));
                if (defl) RC(zt_to_t2(ctx, nullptr, 0, true));
                ProjArgs a = proj_args(ctx, w, w, nullptr);
                if (!defl) a.az_ptr = nullptr, a.K = 0;
                launch_project<0>(ctx, a);
            } else {  // w = project(A (M V_j))
                RC(op_hat(ctx, defl, ctx->gmV[j], ctx->tmp, nullptr, nullptr));
                w = ctx->tmp;
            }
            // two Gram-Schmidt passes against V_0..V_j, then ||w||
            RC(gm_vdots(ctx, j + 1, w, ctx->gm_h));
            k_vsub<<<gx, kBlock, 0, ctx->st>>>(w, ctx->gmVp, ctx->gm_h, j + 1, n, nullptr);
            RC(gm_vdots(ctx, j + 1, w, ctx->gm_e));
            k_vsub<<<gx, kBlock, 0, ctx->st>>>(w, ctx->gmVp, ctx->gm_e, j + 1, n, ctx->dpart);
            ctx->launches += 2;
            RC(global_dots(ctx, ctx->dpart, gx, 1, false, val));
            CK(cudaMemcpyAsync(ctx->h_gm, ctx->gm_h, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaMemcpyAsync(ctx->h_gm + kGmLd, ctx->gm_e, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost,
                               ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            for (int i = 0; i <= j; ++i) {
                h(i, j) = ctx->h_gm[i];
                h(i, j) += ctx->h_gm[kGmLd + i];
            }
            const double hj1 = std::sqrt(std::max(val[0], 0.0));
            h(j + 1, j) = hj1;
            const bool exact = hj1 == 0.0;
            if (!exact) {
                k_vdiv<<<nb, kBlock, 0, ctx->st>>>(ctx->gmV[j + 1], w, hj1, n);
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
            k_vcombine<<<gx, kBlock, 0, ctx->st>>>(ctx->x, ctx->x, ctx->gmZp, ctx->gm_y, j, n);
            ctx->launches++;
        } else {  // x = x + M(V_0 y_0 + ...)
            k_vcombine<<<gx, kBlock, 0, ctx->st>>>(ctx->tmp, nullptr, ctx->gmVp, ctx->gm_y, j, n);
            RC(vcycle(ctx, ctx->tmp, ctx->zx, nullptr, nullptr, nullptr));
            k_addv<<<nb, kBlock, 0, ctx->st>>>(ctx->x, ctx->zx, n);
            ctx->launches += 2;
        }
        CK(cudaStreamSynchronize(ctx->st));  // y (host vector) was read by the async copy above
        total += j;
        RC(gm_residual(ctx, defl, &resnorm));
    }
    out.iters = total;
    out.resnorm = resnorm;
    out.converged = resnorm <= target;
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// upload helpers for finalize

struct OwnedRows {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> ptr{0}, col;
    std::vector<double> val;
    HostRows view() const { return HostRows{nrows, ncols, ptr.data(), col.data(), val.data()}; }
};

// block-diagonal concatenation: part j contributes rows at row offset, columns
// shifted by col offset
static OwnedRows merge_blocks(const std::vector<const dfl::Csr *> &parts, const std::vector<int64_t> &coff) {
    OwnedRows m;
    int64_t nnz = 0;
    for (auto *p : parts) nnz += p->nnz(), m.nrows += p->nrows;
    m.ncols = coff.back();
    m.ptr.reserve(m.nrows + 1);
    m.col.reserve(nnz);
    m.val.reserve(nnz);
    for (size_t j = 0; j < parts.size(); ++j) {
        const dfl::Csr &p = *parts[j];
        for (int64_t i = 0; i < p.nrows; ++i) {
            for (int64_t k = p.ptr[i]; k < p.ptr[i + 1]; ++k) {
                m.col.push_back(p.col[k] + coff[j]);
                m.val.push_back(p.val[k]);
            }
            m.ptr.push_back((int64_t)m.col.size());
        }
    }
    return m;
}

static int build_groups(dfl_ctx *ctx) {
    ctx->groups.clear();
    int s = 0;
    while (s < ctx->nsub) {
        const size_t depth = ctx->pending[s].levels.size();
        int e = s + 1;
        while (e < ctx->nsub && ctx->pending[e].levels.size() == depth) ++e;
        VGroup g;
        g.sub0 = s;
        g.nsub = e - s;
        g.row0 = ctx->sub_off[s];
        g.row1 = ctx->sub_off[e];
        const int L = (int)depth - 1;
        for (int j = s; j < e; ++j)
            if (ctx->pending[j].levels[0].A.nrows != ctx->sub_off[j + 1] - ctx->sub_off[j]) {
                ctx->err = "hierarchy of subdomain " + std::to_string(j) + " does not match its row range";
                return DFL_E_DIMENSION;
            }
        for (int l = 0; l < L; ++l) {
            DLevel v;
            std::vector<const dfl::Csr *> As, Ps, Rs;
            std::vector<int64_t> fo{0}, co{0};
            std::vector<double> w;
            for (int j = s; j < e; ++j) {
                const dfl::Level &lv = ctx->pending[j].levels[l];
                As.push_back(&lv.A);
                Ps.push_back(&lv.P);
                Rs.push_back(&lv.R);
                fo.push_back(fo.back() + lv.A.nrows);
                co.push_back(co.back() + lv.P.ncols);
                w.insert(w.end(), lv.w.begin(), lv.w.end());
            }
            OwnedRows A = merge_blocks(As, fo), P = merge_blocks(Ps, co), R = merge_blocks(Rs, fo);
            // tiny levels stay CSR: they run inside the k_tiny_cycle cluster kernel
            const bool tiny = g_use_tiny && fo.back() <= kTinyRows;
            RC(upload_matrix(ctx, A.view(), v.A, {0, A.nrows}, nullptr, !tiny, w.data(), &v.Aw));
            if (v.A.fmt == FMT_CODE) RC(dalloc(ctx, &v.wr, A.nrows));
            RC(upload_matrix(ctx, P.view(), v.P, {0, P.nrows}, nullptr, !tiny, nullptr, nullptr, true, true, true));
            RC(upload_matrix(ctx, R.view(), v.R, {0, R.nrows}, nullptr, !tiny, nullptr, nullptr, true, true, true));
            RC(upload(ctx, &v.w, w.data(), (int64_t)w.size()));
            v.n = fo.back();
            v.nc = co.back();
            RC(dalloc(ctx, &v.t, v.n));
            if (l > 0) {
                RC(dalloc(ctx, &v.rv, v.n));
                RC(dalloc(ctx, &v.xv, v.n));
            }
            g.nnzA.push_back(A.ptr.back());
            g.nnzP.push_back(P.ptr.back());
            g.rows.push_back(v.n);
            g.lv.push_back(v);
        }
        // bottom level
        std::vector<int64_t> boff{0}, ioff{0};
        std::vector<double> invT;
        for (int j = s; j < e; ++j) {
            const dfl::Level &bl = ctx->pending[j].levels.back();
            const int64_t nb = bl.A.nrows;
            boff.push_back(boff.back() + nb);
            ioff.push_back(ioff.back() + nb * nb);
            g.max_nb = std::max<int>(g.max_nb, (int)nb);
            for (int64_t c = 0; c < nb; ++c)
                for (int64_t i = 0; i < nb; ++i) invT.push_back(bl.bottom_inv[i * nb + c]);
        }
        g.nb = boff.back();
        g.rows.push_back(g.nb);
        RC(upload(ctx, &g.binvT, invT.data(), (int64_t)invT.size()));
        RC(upload(ctx, &g.binv_off, ioff.data(), (int64_t)ioff.size()));
        RC(upload(ctx, &g.b_off, boff.data(), (int64_t)boff.size()));
        if (L > 0) {
            RC(dalloc(ctx, &g.rb, g.nb));
            RC(dalloc(ctx, &g.xb, g.nb));
        }
        {
            // row-major inverses and the argument block of the cooperative kernel
            std::vector<double> binv;
            for (int j = s; j < e; ++j) {
                const auto &bi = ctx->pending[j].levels.back().bottom_inv;
                binv.insert(binv.end(), bi.begin(), bi.end());
            }
            RC(upload(ctx, &g.binv, binv.data(), (int64_t)binv.size()));
            int lc = L;
            for (int l = 0; l < L; ++l)
                if (g.rows[l] <= kCoarseRows) {
                    lc = l;
                    break;
                }
            if (L - lc <= kMaxCoarse) {
                CoarseArgs ca{};
                ca.nlev = L - lc;
                for (int l = lc; l < L; ++l) {
                    const DLevel &v = g.lv[l];
                    CLevel &cl = ca.lv[l - lc];
                    cl.A = v.A;
                    cl.Aw = v.Aw;
                    cl.P = v.P;
                    cl.R = v.R;
                    cl.w = v.w;
                    cl.rv = v.rv;
                    cl.t = v.t;
                    cl.xv = v.xv;
                }
                ca.binv = g.binv;
                ca.binv_off = g.binv_off;
                ca.b_off = g.b_off;
                ca.nsub = g.nsub;
                ca.nb = g.nb;
                ca.rb = g.rb;
                ca.xb = g.xb;
                RC(upload(ctx, &g.cargs, &ca, 1));
                // tiny tail: levels of <= kTinyRows rows + bottom (all CSR)
                int lt = L;
                for (int l = 0; l < L; ++l)
                    if (g.rows[l] <= kTinyRows) {
                        lt = l;
                        break;
                    }
                if (g_use_tiny && g.nb <= kTinyRows && L - lt <= kMaxCoarse) {
                    CoarseArgs ta = ca;
                    ta.nlev = L - lt;
                    for (int l = lt; l < L; ++l) ta.lv[l - lt] = ca.lv[l - lc];
                    bool csr = true;
                    for (int l = 0; l < ta.nlev; ++l)
                        csr = csr && ta.lv[l].Aw.fmt == FMT_CSR && ta.lv[l].A.fmt == FMT_CSR &&
                              ta.lv[l].P.fmt == FMT_CSR && ta.lv[l].R.fmt == FMT_CSR;
                    if (csr && lt >= lc) {
                        RC(upload(ctx, &g.targs, &ta, 1));
                        g.lt = lt;
                    }
                }
                int bps = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_coarse_cycle, 256, 0));
                g.coarse_grid = (unsigned)(std::max(1, std::min(bps, 2)) * ctx->sm_count);
                g.lc = bps > 0 ? lc : -1;
            }
        }
        if (g.max_nb > (1 << 20)) {
            ctx->err = "bottom level too large for shared-memory staging";
            return DFL_E_DIMENSION;
        }
        ctx->groups.push_back(std::move(g));
        s = e;
    }
    return DFL_OK;
}

static int build_tiles(dfl_ctx *ctx) {
    const int rpt = rows_per_block(ctx->Aop);
    std::vector<int64_t> r0, r1, subt{0};
    std::vector<int> ts;
    for (int s = 0; s < ctx->nsub; ++s) {
        for (int64_t i = ctx->sub_off[s]; i < ctx->sub_off[s + 1]; i += rpt) {
            r0.push_back(i);
            r1.push_back(std::min(i + rpt, ctx->sub_off[s + 1]));
            ts.push_back(s);
        }
        subt.push_back((int64_t)r0.size());
    }
    ctx->ntiles = (int64_t)r0.size();
    int64_t *d0, *d1;
    RC(upload(ctx, &d0, r0.data(), ctx->ntiles));
    RC(upload(ctx, &d1, r1.data(), ctx->ntiles));
    RC(upload(ctx, &ctx->tile_sub, ts.data(), ctx->ntiles));
    RC(upload(ctx, &ctx->sub_tiles, subt.data(), (int64_t)subt.size()));
    ctx->h_sub_tiles = subt;
    ctx->tiles = Tiles{d0, d1, ctx->ntiles};
    ctx->subtab = SubTable{};
    if (ctx->nsub <= kSubTab) {
        ctx->subtab.n = ctx->nsub;
        ctx->subtab.rows_per_tile = rpt;
        for (int s = 0; s <= ctx->nsub; ++s) {
            ctx->subtab.sub_off[s] = ctx->sub_off[s];
            ctx->subtab.tile_start[s] = subt[s];
        }
    }
    return DFL_OK;
}

static int stage_in(dfl_ctx *ctx, double *dst, const double *src, int ptr_kind) {
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * ctx->n,
                       ptr_kind == DFL_PTR_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->st));
    return DFL_OK;
}

static int stage_out(dfl_ctx *ctx, double *dst, const double *src, int ptr_kind) {
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dst, src, sizeof(double) * ctx->n,
                       ptr_kind == DFL_PTR_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return DFL_OK;
}

static int ready(dfl_ctx *ctx) {
    if (!ctx) return DFL_E_STATE;
    if (!ctx->finalized) {
        ctx->err = "context not finalized";
        return DFL_E_STATE;
    }
    CK(cudaSetDevice(ctx->device));
    return DFL_OK;
}

static int rank_dot(dfl_ctx *ctx, const double *a, const double *b, double *out) {
    const unsigned nb = (unsigned)std::min<int64_t>(std::max<int64_t>(1, ctx->nblk), 4 * 148);
    k_dot<<<nb, kBlock, 0, ctx->st>>>(a, b, ctx->n, ctx->dpart, nullptr);
    k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->dpart, nb, ctx->scal);
    ctx->launches += 2;
    if (multi(ctx)) {
        RC(comm_allgather(ctx, ctx->scal, ctx->sgather, 8));
        k_rank_sum<<<1, 32, 0, ctx->st>>>(ctx->sgather, ctx->nranks, 8, 1, ctx->scal + 1);
        ctx->launches++;
        CK(cudaMemcpyAsync(out, ctx->scal + 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    } else {
        CK(cudaMemcpyAsync(out, ctx->scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    }
    CK(cudaStreamSynchronize(ctx->st));
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char *dfl_breakdown_string(int code) {
    switch (code) {
        case DFL_BRK_NONE: return "";
        case DFL_BRK_CURVATURE: return "non-positive curvature p'Ap";
        case DFL_BRK_RZ: return "preconditioned residual product degenerated";
        case DFL_BRK_RHO: return "rho degenerated in the BiCG stage";
        case DFL_BRK_SHADOW: return "shadow product degenerated in the BiCG stage";
        case DFL_BRK_MR: return "minimal-residual basis degenerated";
        case DFL_BRK_OMEGA: return "stabilization weight vanished";
        default: return "unknown breakdown";
    }
}

int dfl_ctx_create(int device, dfl_ctx **out) {
    if (!out) return DFL_E_STATE;
    *out = nullptr;
    auto *ctx = new dfl_ctx;
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_state, sizeof(KState));
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) g_sm_count = ctx->sm_count;
    if (e == cudaSuccess) {
        pipe_attrs();
        const char *np = getenv("DFL_PIPE");
        g_use_pipe = np && np[0] == '1';
        const char *nvc = getenv("DFL_VCODE");
        g_use_vcode = nvc && nvc[0] == '1';
        const char *spl = getenv("DFL_CSR_PER_LANE_SMALL");
        g_small_per_lane = spl ? atof(spl) : 12.0;
        const char *ncd = getenv("DFL_NO_CODE");
        g_use_code = !(ncd && ncd[0] == '1');
        const char *sp = getenv("DFL_SHORT_PAD");
        kShortRowPad = sp ? atof(sp) : 1.7;
        const char *nt = getenv("DFL_TINY");
        g_use_tiny = nt && nt[0] == '1';
        const char *nc = getenv("DFL_COARSE");
        g_use_coarse = nc && nc[0] == '1';
        const char *ns = getenv("DFL_SELL");
        g_allow_sell = ns && ns[0] == '1';
        const char *cg = getenv("DFL_CSR_G");
        g_csr_g = cg ? atoi(cg) : 0;
        const char *cl = getenv("DFL_CSR_PER_LANE");
        g_csr_per_lane = cl ? atof(cl) : 12.0;
    }
    if (e != cudaSuccess) {
        dfl::set_setup_error(std::string("CUDA context creation failed: ") + cudaGetErrorString(e));
        delete ctx;
        return DFL_E_CUDA;
    }
    *out = ctx;
    return DFL_OK;
}

void dfl_ctx_destroy(dfl_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->st) cudaStreamSynchronize(ctx->st);
    if (ctx->loop_exec) cudaGraphExecDestroy(ctx->loop_exec);
    for (void *p : ctx->allocs) cudaFree(p);
    if (ctx->h_state) cudaFreeHost(ctx->h_state);
    if (ctx->h_dots) cudaFreeHost(ctx->h_dots);
    if (ctx->h_gm) cudaFreeHost(ctx->h_gm);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->comm) g_nccl.CommDestroy(ctx->comm);
    if (ctx->st2) cudaStreamDestroy(ctx->st2);
    if (ctx->ev_packed) cudaEventDestroy(ctx->ev_packed);
    if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
    if (ctx->st) cudaStreamDestroy(ctx->st);
    delete ctx;
}

const char *dfl_last_error(const dfl_ctx *ctx) { return ctx ? ctx->err.c_str() : dfl::setup_error(); }

int64_t dfl_ctx_device_bytes(const dfl_ctx *ctx) { return ctx ? ctx->bytes : 0; }

int dfl_nccl_unique_id(void *id) {
    std::string err;
    if (!g_nccl.load(err)) {
        dfl::set_setup_error(err);
        return DFL_E_COMM;
    }
    int rc = g_nccl.GetUniqueId(static_cast<NcclId *>(id));
    if (rc != 0) {
        dfl::set_setup_error(std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(rc));
        return DFL_E_COMM;
    }
    return DFL_OK;
}

int dfl_ctx_set_comm(dfl_ctx *ctx, int nranks, int rank, const void *id) {
    if (!ctx) return DFL_E_STATE;
    if (nranks < 1 || rank < 0 || rank >= nranks) {
        ctx->err = "bad rank / world size";
        return DFL_E_PARTITION;
    }
    ctx->nranks = nranks;
    ctx->rank = rank;
    // a 1-rank NCCL communicator exercises the multi-rank code path on one GPU
    const char *fc = getenv("DFL_FORCE_COMM");
    if (nranks == 1 && !(fc && fc[0] == '1')) return DFL_OK;
    if (!g_nccl.load(ctx->err)) return DFL_E_COMM;
    CK(cudaSetDevice(ctx->device));
    NcclId nid;
    std::memcpy(&nid, id, sizeof nid);
    return nccl_check(ctx, g_nccl.CommInitRank(&ctx->comm, nranks, nid, rank), "ncclCommInitRank");
}

int dfl_fabric_create(int nranks, dfl_fabric **out) {
    if (!out || nranks < 1) return DFL_E_STATE;
    auto *f = new dfl_fabric;
    f->nranks = nranks;
    f->ctxs.assign(nranks, nullptr);
    f->pub.assign(nranks, nullptr);
    *out = f;
    return DFL_OK;
}

void dfl_fabric_destroy(dfl_fabric *f) { delete f; }

int dfl_ctx_set_fabric(dfl_ctx *ctx, dfl_fabric *f, int rank) {
    if (!ctx || !f || rank < 0 || rank >= f->nranks) return DFL_E_STATE;
    ctx->fab = f;
    ctx->nranks = f->nranks;
    ctx->rank = rank;
    f->ctxs[rank] = ctx;
    return DFL_OK;
}

int dfl_ctx_set_operator(dfl_ctx *ctx, const dfl_csr *A, int32_t nsub, const int64_t *sub_offsets, int32_t nnbr,
                         const int32_t *nbr_rank, const int64_t *recv_counts, const int64_t *send_counts,
                         const int64_t *send_idx) {
    if (!ctx || !A || nsub < 1 || !sub_offsets) return DFL_E_STATE;
    CK(cudaSetDevice(ctx->device));
    if (sub_offsets[0] != 0 || sub_offsets[nsub] != A->nrows) {
        ctx->err = "subdomain offsets do not span the operator rows";
        return DFL_E_PARTITION;
    }
    for (int s = 0; s < nsub; ++s)
        if (sub_offsets[s + 1] <= sub_offsets[s]) {
            ctx->err = "empty subdomain";
            return DFL_E_PARTITION;
        }
    ctx->n = A->nrows;
    ctx->n_ghost = A->ncols - A->nrows;
    if (ctx->n_ghost < 0) {
        ctx->err = "operator has fewer columns than rows";
        return DFL_E_DIMENSION;
    }
    ctx->nsub = nsub;
    ctx->sub_off.assign(sub_offsets, sub_offsets + nsub + 1);
    HostRows h{A->nrows, A->ncols, A->row_ptr, A->col_idx, A->values};
    // the operator stays uniform ELL (at the HBM roofline, 99.9%); FMT_CODE only
    // pays off for the V-cycle kernels with longer epilogues (profiles/r01)
    RC(upload_matrix(ctx, h, ctx->Aop, ctx->sub_off, &ctx->op_sub_tiles_h, true, nullptr, nullptr, false, false));
    if (ctx->Aop.pipe.stages) RC(upload(ctx, &ctx->op_sub_tiles, ctx->op_sub_tiles_h.data(), (int64_t)ctx->op_sub_tiles_h.size()));
    ctx->op_nnz = ctx->Aop.nnz;
    int64_t nrecv = 0;
    ctx->nbr.clear();
    ctx->recv_cnt.clear();
    ctx->send_cnt.clear();
    ctx->nsend = 0;
    for (int q = 0; q < nnbr; ++q) {
        ctx->nbr.push_back(nbr_rank[q]);
        ctx->recv_cnt.push_back(recv_counts[q]);
        ctx->send_cnt.push_back(send_counts[q]);
        nrecv += recv_counts[q];
        ctx->nsend += send_counts[q];
    }
    if (nrecv != ctx->n_ghost) {
        ctx->err = "halo plan receives " + std::to_string(nrecv) + " values for " + std::to_string(ctx->n_ghost) +
                   " ghost columns";
        return DFL_E_COMM;
    }
    if (ctx->nsend > 0) {
        std::vector<int> si(send_idx, send_idx + ctx->nsend);
        for (int v : si)
            if (v < 0 || v >= ctx->n) {
                ctx->err = "halo send index out of range";
                return DFL_E_COMM;
            }
        RC(upload(ctx, &ctx->send_idx, si.data(), ctx->nsend));
        RC(dalloc(ctx, &ctx->sendbuf, ctx->nsend));
    }
    // rows with ghost columns (multi-rank only): second pass of the operator
    ctx->split = false;
    if (multi(ctx) && ctx->n_ghost > 0 && !(getenv("DFL_NO_OVERLAP") && getenv("DFL_NO_OVERLAP")[0] == '1')) {
        std::vector<uint8_t> flag(ctx->n, 0);
        std::vector<int> rows, bs, bc;
        std::vector<int64_t> sbt{0};
        for (int s = 0; s < nsub; ++s) {
            const size_t first = rows.size();
            for (int64_t i = sub_offsets[s]; i < sub_offsets[s + 1]; ++i)
                for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; ++e)
                    if (A->col_idx[e] >= ctx->n) {
                        flag[i] = 1;
                        rows.push_back((int)i);
                        break;
                    }
            for (size_t j = first; j < rows.size(); j += kBlock) {
                bs.push_back((int)j);
                bc.push_back((int)std::min<size_t>(kBlock, rows.size() - j));
            }
            sbt.push_back((int64_t)bs.size());
        }
        ctx->nbtiles = (int64_t)bs.size();
        RC(upload(ctx, &ctx->bflag, flag.data(), ctx->n));
        RC(upload(ctx, &ctx->brows, rows.data(), (int64_t)rows.size()));
        RC(upload(ctx, &ctx->bstart, bs.data(), (int64_t)bs.size()));
        RC(upload(ctx, &ctx->bcnt, bc.data(), (int64_t)bc.size()));
        RC(upload(ctx, &ctx->sub_btiles, sbt.data(), (int64_t)sbt.size()));
        if (!ctx->st2) {
            CK(cudaStreamCreateWithFlags(&ctx->st2, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ctx->ev_packed, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
        }
        ctx->split = true;
    }
    ctx->pending.assign(nsub, dfl::Hierarchy{});
    ctx->pending_set.assign(nsub, 0);
    ctx->have_op = true;
    ctx->finalized = false;
    return DFL_OK;
}

int dfl_ctx_add_hierarchy(dfl_ctx *ctx, int32_t sub, const dfl_hier *h) {
    if (!ctx || !h) return DFL_E_STATE;
    if (!ctx->have_op || sub < 0 || sub >= ctx->nsub) {
        ctx->err = "hierarchy for an unknown subdomain (set the operator first)";
        return DFL_E_STATE;
    }
    const dfl::Hierarchy &src = h->h;
    if (sub > 0 && src.relax != ctx->relax) {
        ctx->err = "all subdomains must use the same relaxation";
        return DFL_E_CONFIG;
    }
    ctx->relax = src.relax;
    ctx->pending[sub] = src;
    ctx->pending_set[sub] = 1;
    return DFL_OK;
}

int dfl_ctx_set_deflation(dfl_ctx *ctx, int32_t k, const double *zcols, const dfl_csr *AZ, int64_t K,
                          const double *Einv, int32_t first_sub) {
    if (!ctx || !AZ || !Einv) return DFL_E_STATE;
    if (!ctx->have_op) {
        ctx->err = "set the operator before the deflation basis";
        return DFL_E_STATE;
    }
    if (k < 1 || k > kKmax || K % k != 0 || AZ->nrows != ctx->n || AZ->ncols != K) {
        ctx->err = "inconsistent deflation dimensions";
        return DFL_E_DIMENSION;
    }
    CK(cudaSetDevice(ctx->device));
    ctx->k = k;
    ctx->K = K;
    ctx->first_sub = first_sub;
    const int m = (int)(K / k);
    ctx->rank_nsub.assign(ctx->nranks, 0);
    for (int q = 0; q < ctx->nranks; ++q) ctx->rank_nsub[q] = m / ctx->nranks + (q < m % ctx->nranks ? 1 : 0);
    ctx->max_nsub = *std::max_element(ctx->rank_nsub.begin(), ctx->rank_nsub.end());
    if (ctx->rank_nsub[ctx->rank] != ctx->nsub) {
        ctx->err = "rank owns " + std::to_string(ctx->nsub) + " subdomains, placement expects " +
                   std::to_string(ctx->rank_nsub[ctx->rank]);
        return DFL_E_PARTITION;
    }
    // Z columns 1..k-1, column-major for coalesced loads
    std::vector<double> zc((size_t)std::max(1, k - 1) * ctx->n, 0.0);
    for (int c = 1; c < k; ++c)
        for (int64_t i = 0; i < ctx->n; ++i) zc[(size_t)(c - 1) * ctx->n + i] = zcols[i * (k - 1) + (c - 1)];
    RC(upload(ctx, &ctx->zcols, zc.data(), (int64_t)zc.size()));
    std::vector<int> ptr(ctx->n + 1), col(AZ->row_ptr[ctx->n]);
    for (int64_t i = 0; i <= ctx->n; ++i) ptr[i] = (int)AZ->row_ptr[i];
    for (size_t j = 0; j < col.size(); ++j) col[j] = (int)AZ->col_idx[j];
    ctx->az_nnz = (int64_t)col.size();
    RC(upload(ctx, &ctx->az_ptr, ptr.data(), (int64_t)ptr.size()));
    RC(upload(ctx, &ctx->az_col, col.data(), ctx->az_nnz));
    RC(upload(ctx, &ctx->az_val, AZ->values, ctx->az_nnz));
    RC(upload(ctx, &ctx->Einv, Einv, K * K));
    RC(dalloc(ctx, &ctx->tvec, K));
    RC(dalloc(ctx, &ctx->t2, K));
    RC(dalloc(ctx, &ctx->tgather, (int64_t)ctx->nranks * ctx->max_nsub * k));
    ctx->deflation = true;
    return DFL_OK;
}

int dfl_ctx_set_inexact(dfl_ctx *ctx, const double *E, double coarse_tol) {
    if (!ctx || !ctx->deflation) {
        if (ctx) ctx->err = "set the deflation basis before the inexact coarse solve";
        return DFL_E_STATE;
    }
    if (E == nullptr) {
        ctx->inexact = false;
        return DFL_OK;
    }
    CK(cudaSetDevice(ctx->device));
    const int64_t K = ctx->K;
    if (K > 1024) {
        ctx->err = "inexact coarse solve supports K <= 1024";
        return DFL_E_DIMENSION;
    }
    if (!ctx->Edense) {
        RC(dalloc(ctx, &ctx->Edense, K * K));
        RC(dalloc(ctx, &ctx->egm_scr, 2 * (K + 1) * K + 8 * (K + 1)));
    }
    CK(cudaMemcpy(ctx->Edense, E, sizeof(double) * K * K, cudaMemcpyHostToDevice));
    ctx->coarse_tol = coarse_tol;
    ctx->inexact = true;
    return DFL_OK;
}

int dfl_ctx_finalize(dfl_ctx *ctx) {
    if (!ctx) return DFL_E_STATE;
    if (!ctx->have_op) {
        ctx->err = "no operator uploaded";
        return DFL_E_STATE;
    }
    for (int s = 0; s < ctx->nsub; ++s)
        if (!ctx->pending_set[s]) {
            ctx->err = "missing hierarchy for subdomain " + std::to_string(s);
            return DFL_E_STATE;
        }
    CK(cudaSetDevice(ctx->device));
    RC(build_groups(ctx));
    ctx->pending.clear();
    ctx->pending.shrink_to_fit();
    RC(build_tiles(ctx));
    const int64_t nx = ctx->n + ctx->n_ghost;
    RC(dalloc(ctx, &ctx->b, ctx->n));
    RC(dalloc(ctx, &ctx->bp, ctx->n));
    RC(dalloc(ctx, &ctx->x, nx));
    RC(dalloc(ctx, &ctx->xin, nx));
    RC(dalloc(ctx, &ctx->p, nx));
    RC(dalloc(ctx, &ctx->r, ctx->n));
    RC(dalloc(ctx, &ctx->z, ctx->n));
    RC(dalloc(ctx, &ctx->w, ctx->n));
    RC(dalloc(ctx, &ctx->tmp, ctx->n));
    RC(dalloc(ctx, &ctx->yout, ctx->n));
    ctx->nblk = cdiv(ctx->n, kBlock);
    int64_t vparts = 0;
    for (auto &g : ctx->groups)
        vparts += g.lv.empty() ? std::max<int64_t>(1, std::min<int64_t>(cdiv(g.row1 - g.row0, kBlock), 64))
                               : parts_for(g.lv[0].A);
    // partial-sum scratch: one slot per block of the row kernels, or 3 per
    // block of the multi-dot kernels (grid <= 4 * SMs)
    const int64_t dslots = std::max({ctx->nblk, vparts, kDotStride * std::max<int64_t>(ctx->nblk, 4 * ctx->sm_count)});
    RC(dalloc(ctx, &ctx->dpart, dslots + 64));
    RC(dalloc(ctx, &ctx->zt_part, (std::max(ctx->ntiles, ctx->Aop.pipe.ntiles) + ctx->nbtiles) * kKmax + 64));
    RC(dalloc(ctx, &ctx->scal, 16));
    RC(dalloc(ctx, &ctx->sgather, (int64_t)8 * ctx->nranks));
    RC(dalloc(ctx, &ctx->state, 1));
    CK(cudaMallocHost(&ctx->h_dots, 16 * sizeof(double)));
    RC(dalloc(ctx, &ctx->ticket, 4));
    CK(cudaMemset(ctx->ticket, 0, 4 * sizeof(unsigned int)));
    CK(cudaMemset(ctx->x, 0, sizeof(double) * nx));
    CK(cudaMemset(ctx->xin, 0, sizeof(double) * nx));
    CK(cudaMemset(ctx->p, 0, sizeof(double) * nx));
    CK(cudaDeviceSynchronize());
    ctx->finalized = true;
    return DFL_OK;
}

int dfl_solve(dfl_ctx *ctx, const dfl_solve_params *p, const double *b, double *x, int ptr_kind, dfl_report *rep) {
    RC(ready(ctx));
    if (!p || !rep) return DFL_E_STATE;
    if (p->solver < DFL_SOLVER_CG || p->solver > DFL_SOLVER_FGMRES) {
        ctx->err = "solver must be cg, bicgstab2, gmres or fgmres";
        return DFL_E_CONFIG;
    }
    if (p->deflated && !ctx->deflation) {
        ctx->err = "deflated solve requested but no deflation basis uploaded";
        return DFL_E_STATE;
    }
    std::memset(rep, 0, sizeof *rep);
    ctx->launches = 0;
    cudaEvent_t e_h0, e_h1;
    CK(cudaEventCreate(&e_h0));
    CK(cudaEventCreate(&e_h1));
    CK(cudaEventRecord(e_h0, ctx->st));
    RC(stage_in(ctx, ctx->b, b, ptr_kind));
    CK(cudaEventRecord(ctx->ev0, ctx->st));
    const char *ng = getenv("DFL_NO_GRAPH");
    const bool bicg = p->solver != DFL_SOLVER_CG;  // host-driven solvers
    const bool use_graph = !bicg && !multi(ctx) && !(ng && ng[0] == '1');
    KState bstate{};
    if (p->solver == DFL_SOLVER_BICGSTAB2) {
        RC(bicg_solve_dev(ctx, p, bstate));
        RC(lift_dev(ctx, p));
    } else if (p->solver == DFL_SOLVER_GMRES || p->solver == DFL_SOLVER_FGMRES) {
        RC(gmres_solve_dev(ctx, p, p->solver == DFL_SOLVER_FGMRES, bstate));
        RC(lift_dev(ctx, p));
    } else {
        RC(cg_solve_dev(ctx, p, use_graph));
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev1, ctx->st));
    CK(cudaMemcpyAsync(x, ctx->xin, sizeof(double) * ctx->n,
                       ptr_kind == DFL_PTR_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->st));
    CK(cudaEventRecord(e_h1, ctx->st));
    CK(cudaMemcpyAsync(ctx->h_state, ctx->state, sizeof(KState), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    float ms_h2d = 0, ms_solve = 0, ms_d2h = 0;
    CK(cudaEventElapsedTime(&ms_h2d, e_h0, ctx->ev0));
    CK(cudaEventElapsedTime(&ms_solve, ctx->ev0, ctx->ev1));
    CK(cudaEventElapsedTime(&ms_d2h, ctx->ev1, e_h1));
    cudaEventDestroy(e_h0);
    cudaEventDestroy(e_h1);
    const KState s = bicg ? bstate : *ctx->h_state;
    rep->iterations = s.iters;
    rep->converged = s.converged || (s.resnorm <= s.target);
    if (s.breakdown) rep->converged = 0;
    rep->breakdown = rep->converged ? DFL_BRK_NONE : s.breakdown;
    rep->device_loop = use_graph ? 1 : 0;
    rep->bnorm = s.bnorm;
    rep->resnorm = s.resnorm;
    rep->solve_seconds = ms_solve * 1e-3;
    rep->h2d_seconds = ms_h2d * 1e-3;
    rep->d2h_seconds = ms_d2h * 1e-3;
    rep->kernel_launches = ctx->launches + (use_graph ? ctx->body_kernels * std::max(1, s.iters) : 0);
    // true residual ||b - A x|| / ||b|| (deflation.py:293-297; outside the timed span)
    if (s.bnorm == 0.0) {
        rep->relative_residual = 0.0;
    } else {
        RC(op_apply_dev(ctx, ctx->xin, ctx->tmp, 1, ctx->b, false, nullptr, 0));
        double rr = 0.0;
        RC(rank_dot(ctx, ctx->tmp, ctx->tmp, &rr));
        rep->relative_residual = std::sqrt(std::max(rr, 0.0)) / s.bnorm;
    }
    return DFL_OK;
}

int dfl_op_apply(dfl_ctx *ctx, const double *x, double *y, int ptr_kind) {
    RC(ready(ctx));
    RC(stage_in(ctx, ctx->xin, x, ptr_kind));
    RC(op_apply_dev(ctx, ctx->xin, ctx->yout, 0, nullptr, false, nullptr, 0));
    return stage_out(ctx, y, ctx->yout, ptr_kind);
}

int dfl_precond_apply(dfl_ctx *ctx, const double *r, double *z, int ptr_kind) {
    RC(ready(ctx));
    RC(stage_in(ctx, ctx->tmp, r, ptr_kind));
    RC(vcycle(ctx, ctx->tmp, ctx->yout, nullptr, nullptr, nullptr));
    return stage_out(ctx, z, ctx->yout, ptr_kind);
}

int dfl_project(dfl_ctx *ctx, const double *r, double *out, int ptr_kind) {
    RC(ready(ctx));
    if (!ctx->deflation) {
        ctx->err = "no deflation basis";
        return DFL_E_STATE;
    }
    RC(stage_in(ctx, ctx->tmp, r, ptr_kind));
    RC(project_dev(ctx, ctx->tmp, ctx->yout, nullptr, 0));
    return stage_out(ctx, out, ctx->yout, ptr_kind);
}

int dfl_coarse_lift(dfl_ctx *ctx, const double *r, double *out, int ptr_kind) {
    RC(ready(ctx));
    if (!ctx->deflation) {
        ctx->err = "no deflation basis";
        return DFL_E_STATE;
    }
    RC(stage_in(ctx, ctx->tmp, r, ptr_kind));
    k_zt_vec<<<(unsigned)ctx->ntiles, kBlock, 0, ctx->st>>>(ctx->tiles, ctx->tmp, ctx->zcols, ctx->n, ctx->k,
                                                           ctx->zt_part);
    RC(zt_to_t2(ctx, nullptr, 0, false));
    k_lift<<<(unsigned)ctx->ntiles, kBlock, 0, ctx->st>>>(ctx->tiles, ctx->tile_sub, ctx->tmp, ctx->zcols, ctx->n,
                                                         ctx->k, ctx->t2, (int64_t)ctx->first_sub * ctx->k,
                                                         ctx->yout, 0);
    return stage_out(ctx, out, ctx->yout, ptr_kind);
}

int dfl_dot(dfl_ctx *ctx, const double *a, const double *b, int ptr_kind, double *out) {
    RC(ready(ctx));
    RC(stage_in(ctx, ctx->tmp, a, ptr_kind));
    RC(stage_in(ctx, ctx->yout, b, ptr_kind));
    return rank_dot(ctx, ctx->tmp, ctx->yout, out);
}

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
int dfl_ctx_time(dfl_ctx *ctx, int what, int reps, double *ms, double *bytes) {
    RC(ready(ctx));
    if (reps < 1) reps = 1;
    auto run = [&]() -> int {
        if (what == 0) return op_apply_dev(ctx, ctx->p, ctx->w, 0, nullptr, false, nullptr, 0);
        if (what == 1 || what == 2) return vcycle(ctx, ctx->r, ctx->z, nullptr, nullptr, nullptr);
        ctx->err = "unknown timing target";
        return DFL_E_CONFIG;
    };
    // bytes the stored format must move for one pass over M
    auto mat = [](const DMat &M) -> double {
        const double rows = (double)M.nrows;
        if (M.fmt == FMT_CODE) return 8.0 * rows;
        if (M.fmt == FMT_CSR) return 12.0 * (double)M.nnz + 4.0 * (rows + 1);
        return (M.vcode ? 5.0 : 12.0) * (double)M.stored + (M.perm ? 4.0 * rows : 0.0) +
               (M.ell_w ? 0.0 : 8.0 * (rows / 32 + 1));
    };
    if (what == 0) {
        *bytes = 12.0 * ctx->op_nnz + 4.0 * (ctx->n + 1) + 8.0 * (ctx->n + ctx->n_ghost) + 8.0 * ctx->n;
    } else if (what == 2) {
        double b = 0;
        for (auto &g : ctx->groups) {
            for (size_t l = 0; l < g.lv.size(); ++l) {
                const DLevel &v = g.lv[l];
                const double n = (double)g.rows[l], nc = (double)g.rows[l + 1];
                b += v.A.fmt == FMT_CODE ? 24.0 * n + mat(v.A) + 24.0 * n : mat(v.Aw) + 24.0 * n;  // residual
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
    k_fill<<<(unsigned)cdiv(ctx->n + ctx->n_ghost, kBlock), kBlock, 0, ctx->st>>>(ctx->p, 1.0, ctx->n + ctx->n_ghost);
    k_fill<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->r, 1.0, ctx->n);
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
    k_fill<<<(unsigned)ctx->nblk, kBlock, 0, ctx->st>>>(ctx->r, 1.0, ctx->n);
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
