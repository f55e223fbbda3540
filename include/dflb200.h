/*
 * dflb200 -- B200-native solve phase of subdomain-deflated Krylov solvers
 * preconditioned by per-subdomain smoothed-aggregation AMG (arXiv 1710.03940).
 *
 * C ABI of libdflb200.so.  Plain pointers and sizes only; no torch / C++
 * types cross this boundary.  Every function returns 0 on success or a
 * negative DFL_E_* status; the message of the last failure of a context is
 * returned by dfl_last_error(ctx) (dfl_last_setup_error() for context-free
 * setup calls).  Status codes map 1:1 onto the reference's exception classes
 * (pkg/src/deflamg/errors.py:4-37).
 *
 * The entry points replace, in the reference package deflamg 0.1.0:
 *
 *   host setup (stays on the CPU, timed separately, native C++ here):
 *     dfl_hier_build        <- amg.py:217-250 build_hierarchy (+ strength_filter :70-84,
 *                              aggregate :87-125, smooth_prolongation :136-157,
 *                              spai0_weights :160-166, dense_lu sparse.py:226-244)
 *     dfl_basis_az          <- deflation.py:140-149 (AZ = spgemm(A, Z) and the
 *                              per-subdomain rows of E = Z'AZ)
 *     dfl_dense_inverse     <- sparse.py:226-244 dense_lu (+ singularity check)
 *
 *   device solve (sm_100a kernels):
 *     dfl_ctx_set_operator  <- runtime.py:117-152 split_matrix output (SubdomainView)
 *                              and runtime.py:246-271 halo_exchange plan
 *     dfl_ctx_add_hierarchy <- deflation.py:208 (one AmgHierarchy per subdomain)
 *     dfl_ctx_set_deflation <- deflation.py:83-163 DeflationBasis (Z, AZ, E factor)
 *     dfl_solve             <- deflation.py:254-312 DeflatedSolver.solve, with
 *                              krylov.py:95-145 cg / krylov.py:148-285 bicgstab2 /
 *                              krylov.py:288-414 gmres, fgmres
 *     dfl_op_apply          <- runtime.py:283-292 DistributedOperator.apply
 *     dfl_precond_apply     <- deflation.py:239-250 preconditioner -> amg.py:201-212
 *     dfl_project           <- deflation.py:230-233 DeflatedSolver.project
 *     dfl_coarse_lift       <- deflation.py:235-237 DeflatedSolver.coarse_lift
 *     dfl_dot               <- runtime.py:297-304 partition_dot
 *     dfl_spmv_csr          <- _kernels.pyx:11-23 spmv_rows (the reference's plugin
 *                              seam, backend.py:126-146, as one device call)
 */
#ifndef DFLB200_H
#define DFLB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFLB200_ABI_VERSION 1

/* status codes */
#define DFL_OK 0
#define DFL_E_DIMENSION (-1)   /* DimensionError */
#define DFL_E_STRUCTURE (-2)   /* StructureError */
#define DFL_E_SINGULAR (-3)    /* SingularMatrixError */
#define DFL_E_PARTITION (-4)   /* PartitionError */
#define DFL_E_COMM (-5)        /* CommunicatorError (NCCL / halo) */
#define DFL_E_CONFIG (-6)      /* ConfigError */
#define DFL_E_CUDA (-7)        /* CUDA runtime failure */
#define DFL_E_STATE (-8)       /* call out of order (e.g. solve before finalize) */
#define DFL_E_PARSE (-9)       /* ParseError (input files) */

/* relaxation kinds (precond.relax.type) */
#define DFL_RELAX_DAMPED_JACOBI 0
#define DFL_RELAX_SPAI0 1

/* solver kinds (solver.type) */
#define DFL_SOLVER_CG 0
#define DFL_SOLVER_BICGSTAB2 1
#define DFL_SOLVER_GMRES 2     /* restarted, right preconditioned (krylov.py:401-406) */
#define DFL_SOLVER_FGMRES 3    /* flexible (krylov.py:409-414) */

/* which matrix of a hierarchy level */
#define DFL_LEVEL_A 0
#define DFL_LEVEL_P 1
#define DFL_LEVEL_R 2

/* pointer residency for dfl_solve / unit ops */
#define DFL_PTR_HOST 0
#define DFL_PTR_DEVICE 1

/* breakdown codes of dfl_report.breakdown (strings: dfl_breakdown_string) */
#define DFL_BRK_NONE 0
#define DFL_BRK_CURVATURE 1      /* cg: non-positive curvature p'Ap */
#define DFL_BRK_RZ 2             /* cg: preconditioned residual product degenerated */
#define DFL_BRK_RHO 3            /* bicgstab2: rho degenerated in the BiCG stage */
#define DFL_BRK_SHADOW 4         /* bicgstab2: shadow product degenerated */
#define DFL_BRK_MR 5             /* bicgstab2: minimal-residual basis degenerated */
#define DFL_BRK_OMEGA 6          /* bicgstab2: stabilization weight vanished */

/* host CSR view: int64 indices, fp64 values (the reference's SparseMatrix
 * layout, sparse.py:50-58) */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    const int64_t *row_ptr; /* nrows + 1 */
    const int64_t *col_idx; /* row_ptr[nrows] */
    const double *values;   /* row_ptr[nrows] */
} dfl_csr;

/* AmgOptions (amg.py:43-67) */
typedef struct {
    double eps_strong;     /* 0.08 */
    double omega;          /* 2/3 */
    double damping;        /* 0.8 */
    int32_t relax;         /* DFL_RELAX_* */
    int32_t max_levels;    /* 25 */
    int64_t coarse_enough; /* 500 */
} dfl_amg_options;

typedef struct {
    int32_t solver;       /* DFL_SOLVER_* */
    int32_t maxiter;      /* solver.maxiter */
    int32_t refresh_every;/* 50 (krylov.py:41) */
    int32_t deflated;     /* 0: plain block-AMG Krylov (deflation.py:287-290) */
    double tol;           /* solver.tol: atol = tol * ||b|| (deflation.py:266-270) */
    int32_t restart;      /* solver.M: (F)GMRES restart length (deflation.py:275-276) */
    int32_t x0_given;     /* 1: x holds the initial guess on entry (plain block-AMG Krylov only:
                             krylov.py:108/275/383 r = b - A x0; the deflated path ignores x0,
                             deflation.py:284) */
} dfl_solve_params;

typedef struct {
    int32_t iterations;
    int32_t converged;
    int32_t breakdown;          /* DFL_BRK_* */
    int32_t device_loop;        /* 1: the Krylov loop ran as a device-side graph loop */
    double bnorm;
    double resnorm;             /* final recurrence residual norm */
    double relative_residual;   /* true ||b - A x|| / ||b|| (deflation.py:293-297) */
    double solve_seconds;       /* device time of the solve phase (Krylov + lift) */
    double h2d_seconds;
    double d2h_seconds;
    int64_t kernel_launches;    /* kernels of this library launched by the solve */
    double breakdown_value;     /* CG: the p'Ap / r'z that broke down (krylov.py:124,140) */
} dfl_report;

/* structured test problems (problems.py make_problem; reference problems.py:143-171 for the
 * Poisson kind, BASELINE.md §4 for the other two) */
#define DFL_GEN_POISSON 0
#define DFL_GEN_JUMP 1
#define DFL_GEN_CONVDIFF 2
typedef struct {
    int64_t shape[3]; /* grid nodes per axis */
    int64_t boxes[3]; /* subdomain boxes per axis (box-contiguous unknown ordering) */
    int32_t kind;     /* DFL_GEN_* */
    int32_t cells;    /* jump: checkerboard blocks per axis */
    double contrast;  /* jump: kappa on odd blocks */
    double conv[3];   /* convdiff: c per axis */
} dfl_gen_params;

typedef struct dfl_matrix dfl_matrix; /* host CSR produced by setup */
typedef struct dfl_hier dfl_hier;     /* host AMG hierarchy */
typedef struct dfl_ctx dfl_ctx;       /* device solve context (one rank) */
typedef struct dfl_fabric dfl_fabric; /* in-process communicator (tests) */

/* exported entry points; everything else in the library has hidden visibility */
#if defined(__GNUC__)
#define DFL_API __attribute__((visibility("default")))
#else
#define DFL_API
#endif

/* ---- library ----------------------------------------------------------- */
DFL_API int dfl_abi_version(void);
DFL_API const char *dfl_last_setup_error(void);
DFL_API const char *dfl_breakdown_string(int code);

/* ---- host setup (C++) ----------------------------------------------------- */
DFL_API int dfl_hier_build(const dfl_csr *A, const dfl_amg_options *opts, dfl_hier **out);
/* device >= 0: later dfl_hier_build calls on the calling thread run the strength filter,
 * smoothed prolongation, transpose and Galerkin products on that GPU (setup_dev.cu; the
 * hierarchy is bit-identical to the host build; greedy aggregation and the bottom LU stay
 * on the host).  -1 (default): all on the host. */
DFL_API int dfl_setup_device(int device);

/* ---- problem generation on the GPU (gen_dev.cu; problems.py local_rows / node_coords /
 *      make_problem's unknown_of_node, bit-identical) ---------------------------------- */
/* CSR rows [r0, r1) with global columns into host arrays: row_ptr[r1-r0+1], col_idx and values
 * with room for 7 (r1-r0) entries; *nnz = entries written; coords[(r1-r0)*3] or NULL */
DFL_API int dfl_gen_rows(int device, const dfl_gen_params *p, int64_t r0, int64_t r1, int64_t *row_ptr,
                         int64_t *col_idx, double *values, int64_t *nnz, double *coords);
/* natural (x-fastest) node k -> unknown index, for every node of the grid */
DFL_API int dfl_gen_unknown_of_node(int device, const dfl_gen_params *p, int64_t *uon);
DFL_API int dfl_hier_num_levels(const dfl_hier *h);
/* shape of level l's A / P / R (P and R absent at the bottom level: nnz = -1) */
DFL_API int dfl_hier_level_shape(const dfl_hier *h, int level, int which, int64_t *nrows,
                         int64_t *ncols, int64_t *nnz);
DFL_API int dfl_hier_level_copy(const dfl_hier *h, int level, int which, int64_t *row_ptr,
                        int64_t *col_idx, double *values);
/* relaxation weights w of level l: (damping * 1/a_ii) or SPAI-0 a_ii / sum a_ij^2 */
DFL_API int dfl_hier_level_weights(const dfl_hier *h, int level, double *w);
/* bottom level: dense inverse (n x n, row-major) of the LU-factorised block */
DFL_API int dfl_hier_bottom_inverse(const dfl_hier *h, double *inv);
DFL_API void dfl_hier_free(dfl_hier *h);

/* AZ rows of this rank (deflation.py:140) and its rows of E = Z'AZ.
 *   A      : n_local x n_ext rows of the global operator, columns [0, n_local)
 *            own, [n_local, n_ext) ghosts, entries in the global CSR order
 *   zext   : n_ext x k values of Z on every extended column (row-major)
 *   owner  : n_ext global subdomain index of every extended column
 *   rowsub : n_local global subdomain index of every own row
 *   K      : global coarse dimension m*k
 * Outputs: *AZ (n_local x K, exact zeros dropped unless keep_zeros) and
 * E_rows (nsub_local*k x K, row-major) for subdomains [sub0, sub0+nsub). */
DFL_API int dfl_basis_az(const dfl_csr *A, int32_t k, const double *zext, const int32_t *owner,
                 const int32_t *rowsub, int64_t K, int32_t sub0, int32_t nsub, int32_t keep_zeros,
                 dfl_matrix **AZ, double *E_rows);
DFL_API int dfl_matrix_shape(const dfl_matrix *m, int64_t *nrows, int64_t *ncols, int64_t *nnz);
DFL_API int dfl_matrix_copy(const dfl_matrix *m, int64_t *row_ptr, int64_t *col_idx, double *values);
DFL_API void dfl_matrix_free(dfl_matrix *m);

/* ---- input files (mmio.py:29-157; native readers, csrc/mmio.cpp) -----------------------
 * dfl_mm_read: MatrixMarket coordinate real|integer, general|symmetric ->
 *   CSR (1-based indices converted, symmetric entries mirrored, entries in
 *   (row, col) order with duplicates summed in file order) -- replaces
 *   mmio.read_matrix_market (mmio.py:29-101).
 * dfl_vec_read: one float per line (mask = 0, mmio.read_vector :115-131) or
 *   one 0/1 per line (mask != 0, mmio.read_mask :140-157) -> n x 1 matrix.
 * Failures: DFL_E_PARSE, "<path>:<line>: <reason>" in dfl_last_setup_error(). */
DFL_API int dfl_mm_read(const char *path, dfl_matrix **out);
DFL_API int dfl_vec_read(const char *path, int32_t mask, dfl_matrix **out);

/* LU with partial pivoting; DFL_E_SINGULAR with the reference's criterion
 * (min |u_ii| <= 1e-14 max |u_ii|, sparse.py:236-241); writes inv (n x n). */
DFL_API int dfl_dense_inverse(int64_t n, const double *a, double *inv);

/* ---- device context ----------------------------------------------------------- */
DFL_API int dfl_ctx_create(int device, dfl_ctx **out);
DFL_API void dfl_ctx_destroy(dfl_ctx *ctx);
DFL_API const char *dfl_last_error(const dfl_ctx *ctx);

/* multi-process (one rank per GPU) communicator over NCCL; nccl_id is the
 * 128-byte ncclUniqueId produced on rank 0 by dfl_nccl_unique_id */
DFL_API int dfl_nccl_unique_id(void *nccl_id_128);
DFL_API int dfl_ctx_set_comm(dfl_ctx *ctx, int nranks, int rank, const void *nccl_id_128);
/* in-process communicator: ranks are contexts driven by different host
 * threads; collectives synchronise at a host barrier and copy from the peers'
 * device buffers.  Exercises the multi-rank path (halo plan, allgathers,
 * rank-ordered sums, host-driven loop) without NCCL, e.g. on one GPU. */
DFL_API int dfl_fabric_create(int nranks, dfl_fabric **out);
DFL_API void dfl_fabric_destroy(dfl_fabric *f);
/* a rank that waits longer than `seconds` in a collective declares the
 * fabric broken: its call and every later collective return DFL_E_COMM
 * (CommunicatorError, "a participant dropped out", runtime.py:191-212).
 * NCCL ranks use DFL_COMM_TIMEOUT (seconds, default 300) and also poll
 * ncclCommGetAsyncError; either failure aborts the communicator. */
DFL_API int dfl_fabric_set_timeout(dfl_fabric *f, double seconds);
DFL_API int dfl_ctx_set_fabric(dfl_ctx *ctx, dfl_fabric *f, int rank);

/* Operator rows of this rank (all its subdomains), columns renumbered as in
 * dfl_basis_az, entries in the global CSR order.
 *   sub_offsets : nsub+1 rank-local row offsets of the rank's subdomains
 *   halo plan   : for each neighbour rank q (ascending): recv_counts[q] ghost
 *                 values arrive (they fill the ghost columns in ascending
 *                 global order), send_counts[q] values go out, taken from own
 *                 rows send_idx[...] (concatenated in neighbour order). */
DFL_API int dfl_ctx_set_operator(dfl_ctx *ctx, const dfl_csr *A, int32_t nsub, const int64_t *sub_offsets,
                         int32_t nnbr, const int32_t *nbr_rank, const int64_t *recv_counts,
                         const int64_t *send_counts, const int64_t *send_idx);
/* the AMG hierarchy of local subdomain `sub` (uploaded, host copy not kept) */
DFL_API int dfl_ctx_add_hierarchy(dfl_ctx *ctx, int32_t sub, const dfl_hier *h);
/* deflation data of this rank: k columns per subdomain; zcols = n_local x (k-1)
 * non-constant columns (row-major, NULL when k == 1); AZ = n_local x K;
 * Einv = K x K inverse of E (row-major); first_sub = global index of the
 * rank's first subdomain. */
DFL_API int dfl_ctx_set_deflation(dfl_ctx *ctx, int32_t k, const double *zcols, const dfl_csr *AZ,
                          int64_t K, const double *Einv, int32_t first_sub);
/* inexact coarse solve (deflation.inexact, deflation.py:166-178): every
 * E-solve of the projector becomes restarted GMRES on the dense E (K x K,
 * row-major) to relative tolerance coarse_tol (restart K, maxiter 4K+20);
 * E == NULL switches back to the exact E^{-1}.  The caller runs FGMRES. */
DFL_API int dfl_ctx_set_inexact(dfl_ctx *ctx, const double *E, double coarse_tol);
/* converts layouts, builds launch plans; call once after the uploads */
DFL_API int dfl_ctx_finalize(dfl_ctx *ctx);

/* device bytes held by the context */
DFL_API int64_t dfl_ctx_device_bytes(const dfl_ctx *ctx);

/* ---- solve phase ------------------------------------------------------------------- */
/* Stream ordering for device-pointer inputs (DFL_PTR_DEVICE): the context
 * works on a private stream, so a b (or x0) just written by work queued on
 * another stream must be ordered first: dfl_ctx_wait_stream(ctx, s) makes
 * the context's next operations wait for everything queued on the CUDA
 * stream s (a cudaStream_t; NULL = the legacy default stream).  dfl_solve and
 * the unit operations return only after their outputs are complete. */
DFL_API int dfl_ctx_wait_stream(dfl_ctx *ctx, void *stream);
DFL_API int dfl_solve(dfl_ctx *ctx, const dfl_solve_params *p, const double *b, double *x, int ptr_kind,
              dfl_report *rep);

/* page-locked host buffers for solve results (cached: a freed block is reused by the next
 * allocation of the same size, so x can be read back at full copy speed without pinning
 * memory on every solve).  NULL when the driver refuses the allocation. */
DFL_API void *dfl_host_alloc(int64_t bytes);
DFL_API void dfl_host_free(void *ptr);

/* unit operations on this rank's vectors (n_local), host or device pointers */
DFL_API int dfl_op_apply(dfl_ctx *ctx, const double *x, double *y, int ptr_kind);
DFL_API int dfl_precond_apply(dfl_ctx *ctx, const double *r, double *z, int ptr_kind);
DFL_API int dfl_project(dfl_ctx *ctx, const double *r, double *out, int ptr_kind);
DFL_API int dfl_coarse_lift(dfl_ctx *ctx, const double *r, double *out, int ptr_kind);
DFL_API int dfl_dot(dfl_ctx *ctx, const double *a, const double *b, int ptr_kind, double *out);

/* stand-alone CSR SpMV on the device (rows of A; x has A->ncols entries) --
 * the per-kernel seam of the reference (backend.py:126-146) */
DFL_API int dfl_spmv_csr(const dfl_csr *A, const double *x, double *y, int device);

/* timing of the unit operations for the roofline: runs `reps` back-to-back
 * launches of the named kernel family on the context's data and returns the
 * mean device milliseconds per launch and the algorithmic bytes per launch.
 *   what: 0 = operator SpMV (fine A; CSR fp64/int32 algorithmic bytes),
 *         1 = V-cycle (bytes of SURVEY §8(d): CSR layouts),
 *         2 = V-cycle (bytes the stored layouts actually need: ELL padding,
 *             1-byte codes of FMT_CODE matrices, the w.*r pass),
 *         3 = V-cycle captured once and replayed as a CUDA graph, as inside
 *             the solve (bytes as 1),
 *         4 = operator SpMV with the fused Z'y tile partials (as in CG),
 *         5 = projection q = w - AZ t2 with the fused p.q partials,
 *         6 = the finest level's restriction t -> R t (group 0; the V-cycle's
 *             largest single kernel at 150^3)
 *   flags or-ed into what:
 *     DFL_TIME_FLUSH_L2: cold L2 before every launch (a 256 MB buffer is
 *         written in between; each launch timed by its own event pair) --
 *         for 0 / 4 / 5 / 6, whose working set would otherwise fit in L2;
 *     DFL_TIME_FORMAT_BYTES: for 0 / 4 / 5 / 6, return the bytes the stored layout
 *         must move (each stored matrix byte once, each vector read once and
 *         written once) instead of the CSR algorithmic bytes */
#define DFL_TIME_FLUSH_L2 0x100
#define DFL_TIME_FORMAT_BYTES 0x200
DFL_API int dfl_ctx_time(dfl_ctx *ctx, int what, int reps, double *ms_per_launch, double *bytes_per_launch);

/* per-launch device times of one V-cycle, mean over reps; labels is a
 * cap x 32 char buffer ("L<l> resid|restrict|prolong|post", "bottom");
 * returns the number of launches (or a negative status) */
DFL_API int dfl_ctx_profile_vcycle(dfl_ctx *ctx, int reps, int cap, double *ms, char *labels);

/* ---- pressure-Schur block solver (schur.py, paper §4.2) -------------------------------
 * Saddle-point systems split by a pressure mask into [K G; D S] (schur.py:84-120,
 * split on the host).  Outer FGMRES on the monolithic matrix, right
 * preconditioned by the pressure-correction sweep (schur.py:235-251):
 * GMRES on K (SPAI-0), FGMRES on the matrix-free S - D diag(K)^-1 G with the
 * deflated block AMG of S as preconditioner, GMRES on K again. */
typedef struct dfl_block dfl_block;

typedef struct {
    int64_t n;                     /* unknowns of the monolithic system */
    int64_t n_u;                   /* velocity unknowns (mask false); n_p = n - n_u */
    const dfl_csr *A;              /* monolithic matrix (outer operator) */
    const dfl_csr *K, *G, *D, *S;  /* blocks, fields in their original relative order */
    const int32_t *u_idx;          /* n_u positions of the velocity unknowns, ascending */
    const int32_t *p_idx;          /* n_p positions of the pressure unknowns, ascending */
    const double *wK;              /* SPAI-0 weights of K (amg.py:160-166) */
    const double *invKdiag;        /* 1 / diag(K) */
} dfl_block_desc;

typedef struct {
    double tol;        /* solver.tol: outer target tol ||b|| (schur.py:337-345) */
    int32_t maxiter;   /* solver.maxiter */
    int32_t restart;   /* solver.M */
    int32_t usolver;   /* precond.usolver.solver.type: DFL_SOLVER_GMRES or _FGMRES */
    int32_t umaxiter;
    double utol;
    int32_t psolver;   /* precond.psolver.isolver.type: DFL_SOLVER_GMRES or _FGMRES */
    int32_t pmaxiter;
    double ptol;
} dfl_block_params;

typedef struct {
    int32_t iterations;           /* outer FGMRES steps */
    int32_t converged;
    double relative_residual;     /* ||b - A x|| / ||b|| */
    double solve_seconds;         /* device time of the outer solve */
    int64_t velocity_iterations;  /* cumulative inner counts (schur.py:188-190) */
    int64_t pressure_iterations;
    int64_t kernel_launches;
} dfl_block_report;

/* pctx: finalized single-rank context holding the deflated AMG solver of S
 * (schur.py:210-217), shared with the block (same stream); NULL when n_p == 0
 * or when only the operators are needed -- the block then creates its own
 * context on `device`.  The block must be freed before pctx is destroyed. */
DFL_API int dfl_block_create(dfl_ctx *pctx, int device, const dfl_block_desc *desc, dfl_block **out);
DFL_API void dfl_block_free(dfl_block *b);
DFL_API const char *dfl_block_last_error(const dfl_block *b);
DFL_API int64_t dfl_block_device_bytes(const dfl_block *b);
/* schur.py:254-360 SchurSolver.solve */
DFL_API int dfl_block_solve(dfl_block *b, const dfl_block_params *p, const double *rhs, double *x, int ptr_kind,
                            dfl_block_report *rep);
/* schur.py:235-251 one sweep (u, p) = M(b_u, b_p); cumulative inner counts of this call */
DFL_API int dfl_block_precond(dfl_block *b, const dfl_block_params *p, const double *b_u, const double *b_p,
                              double *u, double *pp, int ptr_kind, int64_t *velocity_iterations,
                              int64_t *pressure_iterations);
/* schur.py:145-152 out = S p - D diag(K)^-1 G p */
DFL_API int dfl_block_schur_apply(dfl_block *b, const double *p, double *out, int ptr_kind);
/* y = A x on the monolithic matrix */
DFL_API int dfl_block_apply(dfl_block *b, const double *x, double *y, int ptr_kind);

#ifdef __cplusplus
}
#endif
#endif /* DFLB200_H */
