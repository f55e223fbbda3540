// Internal interface of the device context, shared by the ctx_*.cu units.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/dflb200.h"
#include "host_setup.hpp"
#include "kernels.cuh"

using namespace dfl;

// ---------------------------------------------------------------------------
// minimal NCCL surface, loaded lazily (no link-time dependency)
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
    int (*CommGetAsyncError)(NcclComm, int *) = nullptr;  // optional
    int (*CommAbort)(NcclComm) = nullptr;                 // optional
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
        CommGetAsyncError = reinterpret_cast<decltype(CommGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
        CommAbort = reinterpret_cast<decltype(CommAbort)>(dlsym(h, "ncclCommAbort"));
        return true;
    }
};
extern Nccl g_nccl;

// profiling / layout knobs (defined in ctx.cu, read at context creation)
extern bool g_use_code, g_use_class, g_use_pcode, g_no_sell, g_pdl, g_nccl_graph, g_use_zdict;
extern int g_sm_count;

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
    double timeout_s = 300.0;         // a rank waiting longer declares the collective broken
    bool broken = false;              // a participant dropped out: every later collective fails
    // false: a participant did not arrive within timeout_s (or dropped out earlier)
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const long gen = generation;
        if (++arrived == nranks) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                    [&] { return generation != gen || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
};

struct dfl_ctx {
    int device = 0;
    dfl_fabric *fab = nullptr;
    int sm_count = 148;
    cudaStream_t st = nullptr;
    cudaStream_t st_copy = nullptr;  // x read-back, overlapped with the true-residual kernels
    std::mutex setup_mu;
    std::string err;
    std::vector<void *> allocs;
    int64_t bytes = 0;
    // comm
    int nranks = 1, rank = 0;
    NcclComm comm = nullptr;
    bool comm_dead = false;      // aborted after a failure: every later collective fails
    double comm_timeout_s = 300.0;  // DFL_COMM_TIMEOUT: longest wait for a collective
    // operator
    bool have_op = false, finalized = false;
    int64_t n = 0, n_ghost = 0;
    int nsub = 0;
    std::vector<int64_t> sub_off;
    DMat Aop;
    DMat Abnd;  // split operator (ranks with ghost columns): the rows with ghost columns, one per boundary slot
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
    std::vector<std::shared_ptr<const dfl::Hierarchy>> pending;  // added hierarchies until finalize
    std::vector<int> pending_set;
    std::vector<VGroup> groups;
    int relax = DFL_RELAX_DAMPED_JACOBI;
    // deflation
    bool deflation = false;
    int k = 0;
    int64_t K = 0;
    int first_sub = 0;
    double *zcols = nullptr;
    double *azd = nullptr;                  // own-block AZ values, k x n column-major
    // dictionary-coded copies read by the hot loop (nullptr: > 65536 distinct values, dense)
    int64_t *rank_cnt_d = nullptr;          // coarse values per rank (rank_nsub * k), device
    uint16_t *zcode = nullptr;              // Z columns 1..k-1: zs uint16 per row
    double *ztab = nullptr;
    int ztab_off[kKmax] = {};
    int zs = 0;
    int64_t ztab_n = 0, atab_n = 0;         // table entries (all columns)
    uint16_t *acode = nullptr;              // AZ own block: code_stride(k) uint16 per row
    double *atab = nullptr;
    int atab_off[kKmax] = {};
    int *ax_ptr = nullptr, *ax_col = nullptr;  // AZ entries outside the own block (nullptr: none)
    uint8_t *ax_flag = nullptr;             // rows with such entries
    double *ax_val = nullptr;
    int64_t az_nnz = 0, ax_nnz = 0;
    int64_t *sub_off_d = nullptr;           // nsub + 1 local row offsets
    std::vector<std::unique_ptr<ClassTab>> class_tabs;  // FMT_CLASS tables (DMat::class_id)
    double *Einv = nullptr;
    // inexact coarse solve (deflation.py:166-178): inner GMRES on E
    bool inexact = false;
    double *Edense = nullptr, *egm_scr = nullptr;
    double coarse_tol = 1e-2;
    double *tvec = nullptr, *t2 = nullptr;
    double *zt_part = nullptr;
    double *zt_scratch = nullptr;  // k_zt_finish chunk partials (nsub * zt_chunks * k)
    int zt_chunks = 1;             // k_zt_finish blocks per subdomain
    double *tgather = nullptr;  // nranks * maxsub * k
    unsigned int *ticket = nullptr;
    cudaStream_t st_if = nullptr;  // capture stream of the refresh IF body
    int max_nsub = 0;
    std::vector<int> rank_nsub;  // subdomains per rank (runtime.rank_subdomains)
    // work vectors (n, or n + n_ghost for operator inputs)
    double *b = nullptr, *bp = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr,
           *w = nullptr, *tmp = nullptr, *xin = nullptr, *yout = nullptr;
    double *dpart = nullptr;
    double *x0 = nullptr;  // initial guess of a plain (non-deflated) solve, dfl_solve_params.x0_given
    int64_t nblk = 0;
    int64_t vgrid = 0;  // grid of the grid-stride vector kernels (projection, CG updates, dots)
    // BiCGStab(2) work vectors (allocated on first use)
    double *br[3] = {nullptr, nullptr, nullptr}, *bd[3] = {nullptr, nullptr, nullptr};
    double *bu = nullptr, *bshadow = nullptr, *zx = nullptr;
    double *h_dots = nullptr;  // pinned
    // (F)GMRES (allocated on first use)
    int gm_restart = 0;
    std::vector<double *> gmV, gmZ;
    const double **gmVp = nullptr, **gmZp = nullptr;  // device pointer arrays
    int gm_ld = 0;  // GMRES slot stride (>= restart + 1)
    double *gm_h = nullptr, *gm_e = nullptr, *gm_y = nullptr, *gm_part = nullptr, *gm_loc = nullptr,
           *gm_gath = nullptr, *h_gm = nullptr;
    double *scal = nullptr;     // [0..7] local reduced scalars
    double *sgather = nullptr;  // nranks * 8
    KState *state = nullptr;
    KState *h_state = nullptr;  // pinned
    // graph
    cudaGraphExec_t loop_exec = nullptr;
    int loop_key = -1;
    // the whole single-rank CG solve (prologue, while loop, lift) as one graph
    cudaGraphExec_t solve_exec = nullptr;
    std::string solve_key;
    int64_t solve_fixed_kernels = 0;
    cudaStream_t st_body = nullptr;  // capture stream of the while body
    int64_t body_kernels = 0;
    // several NCCL ranks: the CG body replayed as a graph, done read one iteration late
    cudaGraphExec_t body_exec[2] = {nullptr, nullptr};  // [refresh iteration]
    int body_key = -1;
    int64_t body_graph_kernels[2] = {0, 0};
    KState *h_state2 = nullptr;  // pinned, 2
    cudaEvent_t ev_it[2] = {nullptr, nullptr};
    // BiCGStab(2) device loop (ctx_bicg.cu)
    void *bstate = nullptr, *h_bstate = nullptr;
    cudaGraphExec_t bg_exec = nullptr;
    int bg_key = -1;
    int64_t bg_body_kernels = 0;
    int64_t if_kernels = 0;  // refresh IF body (graph)
    int64_t launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // per-launch profiling of the V-cycle (dfl_ctx_profile_vcycle)
    bool prof_on = false;
    std::vector<cudaEvent_t> prof_ev;
    std::vector<std::string> prof_lab;
    size_t prof_n = 0;
};

inline void prof_mark(dfl_ctx *ctx, const std::string &label) {
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
    std::lock_guard<std::mutex> lk(ctx->setup_mu);
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


// ---------------------------------------------------------------------------
// kernel launch helpers

// Every solve-path kernel is launched with programmatic stream serialization
// (PDL; kernels.cuh DFL_PDL_ENTRY): inside the captured CUDA graphs this
// becomes a programmatic edge, so a kernel's launch overlaps the tail of the
// one before it.  DFL_NO_PDL=1 launches them plainly.
template <typename... KArgs, typename... Args>
inline void launch_k(cudaStream_t st, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (g_pdl) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

inline int rows_per_block(const DMat &A) { return A.fmt == FMT_CSR ? kBlock / A.group : kBlock; }

inline int64_t nblocks_for(const DMat &A) { return cdiv(A.nrows, rows_per_block(A)); }

// resident blocks per SM of a kBlock-thread kernel (grid-stride grids are
// sized to one full wave: a second partial wave would double the tail)
template <class K>
inline int occupancy(K kernel, int threads = kBlock) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess) b = 1;
    return std::max(1, b);
}

// grid of the grid-stride FMT_CODE kernels: one wave of the instance
template <int MODE, bool DOT>
inline int64_t code_grid(const DMat &A) {
    static const int occ = occupancy(k_codep<MODE, DOT>);
    return std::max<int64_t>(1, std::min<int64_t>(cdiv(A.nrows, kBlock), (int64_t)occ * g_sm_count));
}

template <int MODE, bool DOT>
inline int64_t class_grid(const DMat &A) {
    return cdiv(A.nrows, kBlock);  // k_class1: one block per kBlock rows
}

// number of per-block / per-tile partials the POST-with-dot kernel on A produces
inline int64_t parts_for(const DMat &A) {
    if (A.fmt == FMT_PCODE) return cdiv(A.nrows, kBlock);
    if (A.fmt == FMT_CLASS) return class_grid<MODE_POST, true>(A);
    if (A.fmt == FMT_CODE) return code_grid<MODE_POST, true>(A);
    return nblocks_for(A);
}

template <int MODE, bool DOT>
static void launch_csr_mode(const DMat &A, const RowArgs &a, cudaStream_t st) {
    const dim3 grid((unsigned)nblocks_for(A));
    switch (A.group) {
        case 1: launch_k(st, k_csr<1, MODE, DOT>, grid, kBlock, 0, A, a); break;
        case 2: launch_k(st, k_csr<2, MODE, DOT>, grid, kBlock, 0, A, a); break;
        case 4: launch_k(st, k_csr<4, MODE, DOT>, grid, kBlock, 0, A, a); break;
        case 8: launch_k(st, k_csr<8, MODE, DOT>, grid, kBlock, 0, A, a); break;
        case 16: launch_k(st, k_csr<16, MODE, DOT>, grid, kBlock, 0, A, a); break;
        default: launch_k(st, k_csr<32, MODE, DOT>, grid, kBlock, 0, A, a); break;
    }
}

template <int MODE, bool DOT>
static void launch_rows(dfl_ctx *ctx, const DMat &A, const RowArgs &a) {
    if (A.nrows == 0) return;
    if (A.fmt == FMT_PCODE) {
        if (A.pc_wide)
            launch_k(ctx->st, k_pcode<MODE, DOT, true>, (unsigned)cdiv(A.nrows, kBlock), kBlock, 0, A, a);
        else
            launch_k(ctx->st, k_pcode<MODE, DOT>, (unsigned)cdiv(A.nrows, kBlock), kBlock, 0, A, a);
        ctx->launches++;
        return;
    }
    if (A.fmt == FMT_CLASS) {
        static const int occ1 = occupancy(k_class1<MODE, DOT>, kBlock / kOpRpt);
#ifdef DFL_NO_PF
        const int64_t pf = 0;
#else
        const int64_t pf = (int64_t)occ1 * g_sm_count * kBlock;  // next-wave L2 prefetch distance
#endif
        launch_k(ctx->st, k_class1<MODE, DOT>, (unsigned)class_grid<MODE, DOT>(A), kBlock / kOpRpt, 0, A, a,
                 *ctx->class_tabs[A.class_id], pf);
        ctx->launches++;
        return;
    }
    if (A.fmt == FMT_CODE) {
        launch_k(ctx->st, k_codep<MODE, DOT>, (unsigned)code_grid<MODE, DOT>(A), kBlock, 0, A, a);
        ctx->launches++;
        return;
    }
    if (A.fmt == FMT_ELL) {
        const unsigned grid = (unsigned)nblocks_for(A);
        switch (A.ell_w) {
            case 3: launch_k(ctx->st, k_ell<MODE, DOT, 3>, grid, kBlock, 0, A, a); break;
            case 4: launch_k(ctx->st, k_ell<MODE, DOT, 4>, grid, kBlock, 0, A, a); break;
            case 5: launch_k(ctx->st, k_ell<MODE, DOT, 5>, grid, kBlock, 0, A, a); break;
            case 6: launch_k(ctx->st, k_ell<MODE, DOT, 6>, grid, kBlock, 0, A, a); break;
            case 7: launch_k(ctx->st, k_ell<MODE, DOT, 7>, grid, kBlock, 0, A, a); break;
            case 8: launch_k(ctx->st, k_ell<MODE, DOT, 8>, grid, kBlock, 0, A, a); break;
            default: launch_k(ctx->st, k_ell<MODE, DOT, 0>, grid, kBlock, 0, A, a); break;
        }
    } else
        launch_csr_mode<MODE, DOT>(A, a, ctx->st);
    ctx->launches++;
}

template <int OPMODE, int NV>
static void launch_op_nv(dfl_ctx *ctx, const OpArgs &a, unsigned grid) {
    const DMat &A = ctx->Aop;
    const SubTable &S = ctx->subtab;
    if (A.fmt == FMT_CLASS) {
        static const int occ = occupancy(k_op_class<OPMODE, NV, false>, kBlock / kOpRpt);
        OpArgs b = a;
        b.pf = (int64_t)occ * g_sm_count * kBlock;  // next-wave L2 prefetch distance (rows)
#ifdef DFL_NO_PF
        b.pf = 0;
#endif
        if (a.zcode && a.k > 1)
            launch_k(ctx->st, k_op_class<OPMODE, NV, true>, grid, kBlock / kOpRpt, 0, A, ctx->tiles, S, b,
                     *ctx->class_tabs[A.class_id]);
        else
            launch_k(ctx->st, k_op_class<OPMODE, NV, false>, grid, kBlock / kOpRpt, 0, A, ctx->tiles, S, b,
                     *ctx->class_tabs[A.class_id]);
        return;
    }
    if (A.fmt == FMT_CODE) {
        launch_k(ctx->st, k_op_code<OPMODE, NV>, grid, kBlock, 0, A, ctx->tiles, S, a);
        return;
    }
    switch (A.ell_w) {
        case 5: launch_k(ctx->st, k_op_ell<OPMODE, 5, NV>, grid, kBlock, 0, A, ctx->tiles, S, a); break;
        case 6: launch_k(ctx->st, k_op_ell<OPMODE, 6, NV>, grid, kBlock, 0, A, ctx->tiles, S, a); break;
        case 7: launch_k(ctx->st, k_op_ell<OPMODE, 7, NV>, grid, kBlock, 0, A, ctx->tiles, S, a); break;
        default: launch_k(ctx->st, k_op_ell<OPMODE, 0, NV>, grid, kBlock, 0, A, ctx->tiles, S, a); break;
    }
}

template <int OPMODE>
static void launch_op(dfl_ctx *ctx, const OpArgs &a) {
    const DMat &A = ctx->Aop;
    const unsigned grid = (unsigned)ctx->ntiles;
    if (grid == 0) return;
    if (A.fmt == FMT_CODE || A.fmt == FMT_ELL || A.fmt == FMT_CLASS) {
        // Z'y epilogue width: the smallest power of two >= k
        if (a.k <= 1)
            launch_op_nv<OPMODE, 1>(ctx, a, grid);
        else if (a.k <= 2)
            launch_op_nv<OPMODE, 2>(ctx, a, grid);
        else if (a.k <= 4)
            launch_op_nv<OPMODE, 4>(ctx, a, grid);
        else
            launch_op_nv<OPMODE, 8>(ctx, a, grid);
    } else {
        switch (A.group) {
            case 1: launch_k(ctx->st, k_op_csr<1, OPMODE>, grid, kBlock, 0, A, ctx->tiles, ctx->subtab, a); break;
            case 2: launch_k(ctx->st, k_op_csr<2, OPMODE>, grid, kBlock, 0, A, ctx->tiles, ctx->subtab, a); break;
            case 4: launch_k(ctx->st, k_op_csr<4, OPMODE>, grid, kBlock, 0, A, ctx->tiles, ctx->subtab, a); break;
            case 8: launch_k(ctx->st, k_op_csr<8, OPMODE>, grid, kBlock, 0, A, ctx->tiles, ctx->subtab, a); break;
            case 16: launch_k(ctx->st, k_op_csr<16, OPMODE>, grid, kBlock, 0, A, ctx->tiles, ctx->subtab, a); break;
            default: launch_k(ctx->st, k_op_csr<32, OPMODE>, grid, kBlock, 0, A, ctx->tiles, ctx->subtab, a); break;
        }
    }
    ctx->launches++;
}

// ---------------------------------------------------------------------------
// cross-unit entry points (return DFL_OK or a DFL_E_* code, message in ctx->err)

inline bool multi(const dfl_ctx *ctx) { return ctx->comm != nullptr || ctx->fab != nullptr; }
inline ZCode zcode_of(const dfl_ctx *ctx) {
    ZCode z;
    if (ctx->zcode) {
        z.code = ctx->zcode;
        z.tab = ctx->ztab;
        z.stride = ctx->zs;
        for (int c = 0; c < kKmax; ++c) z.off[c] = ctx->ztab_off[c];
    }
    return z;
}
// the plain block-AMG Krylov path starts from x0 (krylov.py:108/275/383)
inline bool use_x0(const dfl_ctx *ctx, const dfl_solve_params *p) { return p->x0_given && !p->deflated && ctx->x0; }

inline ProjArgs proj_args(dfl_ctx *ctx, const double *in, double *out, const KState *st) {
    ProjArgs a{};
    if (ctx->deflation) {
        a.azd = ctx->azd;
        a.ax_ptr = ctx->ax_ptr;
        a.ax_flag = ctx->ax_flag;
        a.ax_col = ctx->ax_col;
        a.ax_val = ctx->ax_val;
        a.acode = ctx->acode;
        a.atab = ctx->atab;
        for (int c = 0; c < kKmax; ++c) a.atab_off[c] = ctx->atab_off[c];
        a.sub_off = ctx->sub_off_d;
        a.nsub = ctx->nsub;
        a.k = ctx->k;
        a.own_base = (int64_t)ctx->first_sub * ctx->k;
    }
    a.t2 = ctx->t2;
    a.K = ctx->deflation ? ctx->K : 0;
    a.n = ctx->n;
    a.in = in;
    a.out = out;
    a.st = st;
    return a;
}

// deflation columns per subdomain -> the k_project instance (KZ >= k)
template <int MODE>
static void launch_project(dfl_ctx *ctx, const ProjArgs &a) {
    const unsigned g = (unsigned)ctx->vgrid;
    if (!a.azd || a.k <= 1)
        launch_k(ctx->st, k_project<MODE, 1>, g, kBlock, 0, a);
    else if (a.k <= 2)
        launch_k(ctx->st, k_project<MODE, 2>, g, kBlock, 0, a);
    else if (a.k <= 4)
        launch_k(ctx->st, k_project<MODE, 4>, g, kBlock, 0, a);
    else
        launch_k(ctx->st, k_project<MODE, 8>, g, kBlock, 0, a);
    ctx->launches++;
}


// ctx_layout.cu
int upload_matrix(dfl_ctx *ctx, const HostRows &h, DMat &m, const std::vector<int64_t> &bounds,
                  std::vector<int64_t> *bound_tiles = nullptr, bool allow_ell = true,
                  const double *colscale = nullptr, DMat *scaled = nullptr, bool allow_sell = true,
                  bool allow_code = true, bool allow_class = true);
int build_groups(dfl_ctx *ctx);
std::vector<uint8_t> class_exceptions(const HostRows &h, const std::function<bool(int64_t)> &skip);
int build_tiles(dfl_ctx *ctx);

// ctx_comm.cu
int comm_allgather(dfl_ctx *ctx, const double *send, double *recv, size_t count);
int halo(dfl_ctx *ctx, double *v, cudaStream_t xs = nullptr);
// fold (several ranks, CG, exact E^-1): also pAp = p.w - t.E^-1 t and the alpha step
// (the rank's p.w partials in extra_part)
int zt_to_t2(dfl_ctx *ctx, const KState *st, int need_refresh, bool from_op, const double *extra_part = nullptr,
             int64_t extra_n = 0, KState *fold = nullptr);
int rank_scalar(dfl_ctx *ctx, const double *part, int64_t nparts, int slot, const double **gath);
// wait for a stream / event; with NCCL, poll the communicator's asynchronous
// error and a timeout instead of blocking, abort the communicator on either
// (a participant that dropped out would otherwise hang the solve) and return
// DFL_E_COMM -> CommunicatorError (runtime.py:191-212)
int comm_wait(dfl_ctx *ctx, cudaStream_t s);
int comm_wait_event(dfl_ctx *ctx, cudaEvent_t e);
// ctx_cycle.cu
int vcycle(dfl_ctx *ctx, const double *r, double *z, const KState *st, double *dot_part, int64_t *nparts);
int op_apply_dev(dfl_ctx *ctx, double *xin, double *y, int opmode, const double *b, bool zt, const KState *st,
                 int need_refresh);
int project_dev(dfl_ctx *ctx, const double *v, double *out, const KState *st, int dotmode, double *out2 = nullptr);
int lift_dev(dfl_ctx *ctx, const dfl_solve_params *p);
// ctx_cg.cu / ctx_krylov.cu
int cg_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, bool use_graph);
int bicg_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, KState &out);
int bicg_prologue(dfl_ctx *ctx, const dfl_solve_params *p, KState &out);
int bicg_solve_graph(dfl_ctx *ctx, const dfl_solve_params *p, KState &out);  // ctx_bicg.cu
int gmres_solve_dev(dfl_ctx *ctx, const dfl_solve_params *p, bool flexible, KState &out);
// ctx.cu
int ready(dfl_ctx *ctx);
