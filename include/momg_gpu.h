/* momg_gpu -- C ABI of the B200-native NMG / fast-sweeping hot path.
 *
 * This is the drop-in boundary.  The reference has no FFI
 * or plugin registry: its boundary is the set of C++ free functions in
 * namespace momg that the host driver calls.  Each entry point below replaces
 * exactly one of them (reference file:line cited); plain pointers, sizes and
 * status codes only -- no C++ or torch types cross this line.
 *
 * Device residency: a momg_field is one grid level living in B200 HBM
 * (coefficients [cells][NP] cell-major with NP = N rounded up to 4 doubles,
 * params [cells][4]).  Host arrays passed to upload/download use the
 * reference's host order: coeffs[(j*nx+i)*N + k], params[(j*nx+i)*4 + q]
 * (grid.hpp:64, moment_rep.hpp:16-32).  All work is FP64 and runs on the
 * library's CUDA stream (momg_set_stream); calls are stream-ordered and only
 * the ones that return host scalars or report errors synchronise.
 *
 * Errors: every function returns a momg status (0 = OK) and fills *err
 * (nullable).  Codes mirror the reference exception hierarchy
 * (types.hpp:20-57); the host wrappers rethrow the matching exception type so
 * solve_steady's catch logic (multigrid.cpp:289-300) is unchanged.
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns MOMG_ERR_NO_DEVICE.
 */
#ifndef MOMG_GPU_H
#define MOMG_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

enum momg_status {
  MOMG_OK = 0,
  MOMG_NONPHYSICAL_STATE = 1, /* NonphysicalState   (types.hpp:33) */
  MOMG_SOLVER_ERROR = 2,      /* SolverError        (types.hpp:54) */
  MOMG_ERROR = 3,             /* Error              (types.hpp:20), e.g. grad_normalize cap */
  MOMG_NON_SPD = 4,           /* NonSpdTensor       (types.hpp:46) */
  MOMG_CONFIG = 5,            /* ConfigError        (types.hpp:26) */
  MOMG_NONCONVERGENCE = 6,    /* NonConvergence     (multigrid.hpp:89-97) */
  MOMG_ERR_NO_DEVICE = 100,   /* no CUDA device / extension unusable */
  MOMG_ERR_CUDA = 101,        /* CUDA runtime failure */
  MOMG_ERR_ARG = 102          /* invalid argument (null handle, shape mismatch) */
};

typedef struct momg_err {
  int code;
  int i, j;        /* failing cell when known, else -1 */
  char msg[256];
} momg_err;

/* Grid2D (grid.hpp:12-37): per-cell sizes and centres, host pointers. */
typedef struct momg_grid {
  int nx, ny;
  double Lx, Ly;
  const double *dx, *dy, *xc, *yc;
} momg_grid;

enum { MOMG_BGK = 0, MOMG_ES_BGK = 1, MOMG_SHAKHOV = 2 };

/* SolveContext (single_level.hpp:27-34): walls left, right, bottom, top. */
typedef struct momg_ctx {
  int M;               /* moment order (IndexSet order) */
  int space_order;     /* SpatialScheme.order, 1 or 2 (spatial.hpp:16-22) */
  double c_bound;      /* SpatialScheme.c_bound = max_hermite_root(M+1) */
  double cfl;          /* CflPolicy.cfl */
  double cfl_c_bound;  /* CflPolicy.c_bound */
  int collision;       /* CollisionModel.kind */
  double prandtl;      /* CollisionModel.prandtl */
  double knudsen;      /* GasParams.knudsen */
  double viscosity_index; /* GasParams.viscosity_index */
  double wall_speed[4];
  double wall_theta[4];
  int threads;         /* SolveContext.threads: > 1 selects the blocked-parallel sweep (band-aligned blocks, first order) */
} momg_ctx;

/* CyclePolicy + SolverOptions (multigrid.hpp:30-35, 101-107). */
typedef struct momg_solver_opts {
  int kind;            /* 0 euler, 1 fs, 2 nmg (SolverKind) */
  double tol;
  int max_iterations;  /* 0: 200 nmg, 100000 fs/euler */
  int levels;          /* 0: auto (GridHierarchy::build) */
  int s1, s2, s3, gamma;
} momg_solver_opts;

/* SolveReport (multigrid.hpp:78-87); history = rel_residual per iteration. */
typedef struct momg_report {
  int converged;
  int iterations;
  double r0_norm;
  double final_norm;
  double final_ratio;
  long long work;      /* fast-sweeping cell evaluations (WorkStats) */
  double seconds;
  int history_len;
  double* history;     /* caller buffer, capacity history_cap (nullable) */
  int history_cap;
  double* history_seconds; /* nullable, capacity history_cap: elapsed seconds at each
                              iteration (HistoryEntry.seconds, multigrid.cpp:303) */
} momg_report;

typedef struct momg_field momg_field; /* opaque device-resident level */

/* ---- runtime ---------------------------------------------------------- */
int momg_init(int device, momg_err* err);          /* select device, create stream */
int momg_set_stream(void* cuda_stream);            /* use an external stream (nullable = own) */
void* momg_get_stream(void);
int momg_synchronize(momg_err* err);
const char* momg_version(void);
int momg_supported_order(int M);                   /* 1 if kernels are instantiated for M */
/* Hermite bound C_{M+1}: max_hermite_root (tables.cpp:22-41, hermite.hpp:23-26) */
double momg_max_hermite_root(int degree);

/* ---- fields (CellField, grid.hpp:54-85) -------------------------------- */
int momg_field_create(const momg_grid* grid, int M, momg_field** out, momg_err* err);
void momg_field_destroy(momg_field* f);
int momg_field_shape(const momg_field* f, int* nx, int* ny, int* M, int* N, int* NP);
int momg_field_upload(momg_field* f, const double* coeffs, const double* params, momg_err* err);
int momg_field_download(const momg_field* f, double* coeffs, double* params, momg_err* err);
int momg_field_upload_async(momg_field* f, const double* coeffs, const double* params, momg_err* err);
int momg_field_download_async(const momg_field* f, double* coeffs, double* params, momg_err* err);
/* Overlapped transfers for streaming many solves through double-buffered
 * fields: the upload runs on the library's H2D copy stream once the field's
 * previous overlapped download has finished, and every kernel enqueued after
 * the call waits for it; the download runs on the D2H copy stream after the
 * kernels enqueued before the call.  Host buffers should be pinned.  Finish
 * with momg_synchronize (which also waits for both copy streams). */
int momg_field_upload_overlapped(momg_field* f, const double* coeffs, const double* params, momg_err* err);
int momg_field_download_overlapped(momg_field* f, double* coeffs, double* params, momg_err* err);
/* make later work on the library stream wait for every overlapped transfer enqueued so far */
int momg_copy_barrier(momg_err* err);
int momg_field_copy(momg_field* dst, const momg_field* src, momg_err* err);   /* CellField copy (multigrid.cpp:188) */
int momg_field_fill_maxwellian(momg_field* f, double rho, const double u[3], double theta,
                               momg_err* err);                               /* uniform_field (grid.hpp:79-85) */
/* device pointers for zero-copy interop (coeffs [cells][NP], params [cells][4]) */
int momg_field_device_ptrs(momg_field* f, double** coeffs, double** params);

/* ---- the hot path ------------------------------------------------------ */
/* residual (spatial.cpp:135-159): out <- R(field), out params <- field params */
int momg_residual(const momg_ctx* ctx, const momg_field* field, momg_field* out, momg_err* err);
/* fast_sweep_step (single_level.cpp:121-166): exact lexicographic Gauss-Seidel
   order via anti-diagonal wavefronts; rhs nullable (empty RhsField);
   sweep_order nullable ({0,1,2,3}); evals += cell updates (WorkStats) */
int momg_fast_sweep(const momg_ctx* ctx, momg_field* field, const momg_field* rhs,
                    const int* sweep_order, long long* evals, momg_err* err);
/* fast_sweep_step (no rhs) followed by residual into `out`, the sequence of
 * nmg_cycle (multigrid.cpp:170-176) and of the C5 step: identical results to
 * the two calls, run as one launch (the residual follows the last sweep's
 * wavefront on otherwise idle SMs) where the band kernels apply */
int momg_fast_sweep_residual(const momg_ctx* ctx, momg_field* field, const int* sweep_order, momg_field* out,
                             long long* evals, momg_err* err);
/* euler_step (single_level.cpp:74-97; single_level.hpp:55-58): f += dt (R - rhs)
   with the single global dt (global_dt, :31-38), re-normalisation and the dt/2
   retry.  residuals = residual(field) on the incoming field (nullable: evaluated
   here); rhs nullable (empty RhsField) */
int momg_euler_step(const momg_ctx* ctx, momg_field* field, const momg_field* residuals,
                    const momg_field* rhs, momg_err* err);
/* total_mass / mass_correction (single_level.cpp:168-183) */
int momg_total_mass(const momg_field* field, double* out, momg_err* err);
int momg_mass_correction(momg_field* field, double target_mass, momg_err* err);
/* restrict_solution (multigrid.cpp:67-112): coarse <- R_sol(fine) */
int momg_restrict_solution(const momg_field* fine, momg_field* coarse, momg_err* err);
/* restrict_residual (multigrid.cpp:114-142): out <- sum (a_c/S) project(arrays_c -> coarse basis) */
int momg_restrict_residual(const momg_field* fine_arrays, const momg_field* coarse,
                           momg_field* out, momg_err* err);
/* fas_correct (multigrid.cpp:144-164) */
int momg_fas_correct(momg_field* fine, const momg_field* coarse_before,
                     const momg_field* coarse_after, momg_err* err);
/* residual_norm (multigrid.cpp:202-218); theta from field params */
int momg_residual_norm(const momg_field* res, const momg_field* field, double* out, momg_err* err);
/* residual_scale (multigrid.cpp:224-239) */
int momg_residual_scale(const momg_ctx* ctx, const momg_field* field, double* out, momg_err* err);
/* defect of nmg_cycle (multigrid.cpp:178-185): out <- project(rhs -> res basis) - res,
   or -res when rhs is null */
int momg_defect(const momg_field* res, const momg_field* rhs, momg_field* out, momg_err* err);
/* coarse_rhs += coarse_res (multigrid.cpp:192-193): dst.coeffs += src.coeffs */
int momg_axpy(momg_field* dst, const momg_field* src, momg_err* err);
/* f.coeffs *= factor: mass_correction's rescale (single_level.cpp:176-183) with the
   factor target / total mass computed by the caller (strips of a partitioned level) */
int momg_field_scale(momg_field* f, double factor, momg_err* err);

/* ---- the host driver (kept as host C++, multigrid.cpp:44-65, 166-320) --- */
/* nmg_cycle on the hierarchy GridHierarchy::build(field grid, levels) */
int momg_nmg_cycle(const momg_ctx* ctx, momg_field* field, int levels, int s1, int s2, int s3,
                   int gamma, long long* work, momg_err* err);
/* nmg_cycle for R(f) = rhs (rhs nullable) on GridHierarchy::build(field grid, levels):
   the coarse problem of a cycle whose finer level runs elsewhere (strips) */
int momg_nmg_cycle_rhs(const momg_ctx* ctx, momg_field* field, const momg_field* rhs, int levels, int s1,
                       int s2, int s3, int gamma, long long* work, momg_err* err);
/* solve_steady: NonConvergence -> MOMG_NONCONVERGENCE with the partial report */
int momg_solve_steady(const momg_ctx* ctx, momg_field* field, const momg_solver_opts* opts,
                      momg_report* report, momg_err* err);

/* ---- front-end output (scenario.cpp:372-399) ---- */
/* UnitScales (scenario.hpp:76-84, scenario.cpp:313-319) and GasParams.molecule_mass:
   lengths scale by `length`, densities by `density`, temperatures (specific-energy
   form) by `theta`, speeds by `speed`. */
typedef struct momg_units {
  double length, density, theta, speed, molecule_mass;
} momg_units;
/* export_field's table in laboratory units: per cell, row-major with j outermost,
   the 11 columns x y rho u1 u2 T sigma11 sigma12 sigma22 q1 q2 (extract_macro,
   moment_rep.hpp:116-146, evaluated on the device) into the host buffer `out` of
   nx*ny*11 doubles.  A cell with rho <= 0 is NonphysicalState ("extract_macro:
   nonpositive density", err->i/j = the first such cell in row order);
   *rows_ok (nullable) = the rows before it. */
int momg_field_table(const momg_field* f, const momg_units* u, double* out, long long* rows_ok,
                     momg_err* err);
/* export_field (scenario.cpp:372-399): the table as TSV at `path` (header row, values
   %.17g, tab-separated).  MOMG_ERROR "export_field: cannot open '<path>'" / "write
   failed"; NonphysicalState after writing the rows before the first rejected cell. */
int momg_export_field(const momg_field* f, const momg_units* u, const char* path, momg_err* err);

/* ---- strip partition: multi-GPU ------------------ */
/* A level of `grid` split into n <= 8 column strips [bounds[r], bounds[r+1])
   (widths multiples of 32; nx a multiple of 32).  This process owns strips
   [first, last]: they are allocated here (momg_strips_field gives each as an
   ordinary momg_field on its sub-grid, plus its residual field); the other
   strips belong to peer ranks and are attached with momg_strips_import from
   the handle their owner exported (CUDA IPC: peer memory over NVLink).  The
   fused FS iteration + residual then runs this process's band tasks and reads
   / polls the neighbouring strips' cells in place, so the Gauss-Seidel
   wavefront (single_level.cpp:121-166) pipelines across strips with no
   collective.  Ranks must call it in the same sequence, and fields are only
   written by other entry points while no rank is inside it (the host layer,
   paper_2206_13164_b200/strips.py, brackets it with barriers).  With all
   strips owned by one process it is one kernel over every strip (the
   single-GPU emulation of the ranks). */
typedef struct momg_strips momg_strips;
#define MOMG_STRIP_HANDLE_BYTES 320
int momg_strips_create(const momg_grid* grid, int M, int n, const int* bounds, int first, int last,
                       momg_strips** out, momg_err* err);
void momg_strips_destroy(momg_strips* s);
int momg_strips_field(momg_strips* s, int r, momg_field** field, momg_field** residual);
int momg_strips_export(momg_strips* s, int r, void* handle /* MOMG_STRIP_HANDLE_BYTES */, momg_err* err);
int momg_strips_import(momg_strips* s, int r, const void* handle, momg_err* err);
/* fast_sweep_step (no rhs, first order, M <= 5) + residual into the strips'
   residual fields, over the partition (nmg_cycle multigrid.cpp:170-176; the
   C5 step); evals += the owned strips' cell updates */
int momg_strips_fast_sweep_residual(const momg_ctx* ctx, momg_strips* s, const int* sweep_order,
                                    long long* evals, momg_err* err);
/* `iters` (<= 4) consecutive fast_sweep_step calls (no rhs) over the partition,
   first or second order: one band launch */
int momg_strips_fast_sweep(const momg_ctx* ctx, momg_strips* s, const int* sweep_order, int iters,
                           long long* evals, momg_err* err);
/* residual (spatial.cpp:135-159) of the owned strips into their residual fields:
   each strip plus its neighbours' 1 (first order) or 2 (second order) columns,
   copied from peer memory, then the single-field residual on that */
int momg_strips_residual(const momg_ctx* ctx, momg_strips* s, momg_err* err);
/* every strip's field (which = 0) or residual field (1) -> a full-level field
   (own and peer memory): the agglomeration of a level on every rank */
int momg_strips_gather(momg_strips* s, int which, momg_field* full, momg_err* err);
/* the owned strips' columns of a full-level field -> their fields (0) / residual fields (1) */
int momg_strips_scatter(momg_strips* s, int which, const momg_field* full, momg_err* err);

/* ---- execution strategy of fast_sweep (same results either way) -------- */
/* 1 (default): one persistent dataflow kernel per call (the band kernels for
   M <= 6 -- residuals and ES-BGK of M = 6 thread-per-face --, warp-per-cell
   M = 7, 8); 2: the same without
   the band kernels (thread-per-face / warp-per-cell for every M); 0: one launch
   per anti-diagonal (the simple reference strategy; env MOMG_SWEEP=diag). */
int momg_set_sweep_mode(int mode);
/* band kernel of the exact-order sweeps (first / second order, with or
   without an FAS right-hand side) and first-order residuals: 1 (default; env
   MOMG_RB=0 selects 0) the register-resident kernels (one thread per face
   side, moment vectors in registers: k8_band, k9_band; M <= 5 on 32-column
   bands, M = 6 on 16-column bands); 0 the split kernels of M <= 5 (each face
   cut 4 ways across warps through shared memory; thread-per-face for M = 6).
   Results agree to rounding (the two halves of a face flux are summed after
   the back projection). */
int momg_set_band_kernel(int kind);

/* ---- instrumentation --------------------------------------------------- */
/* debug: %globaltimer stamps of the first cap band tasks of the band sweep
   ([task][32]: loop start / end, steps, per-phase sums; tools/trace_band.py) */
int momg_debug_trace(long long cap);
long long momg_debug_trace_read(unsigned long long* host, long long n);
/* number of kernels this library has launched since load (gpu_launches) */
long long momg_launch_count(void);
/* solve_steady iterations replayed from a captured CUDA graph since load */
long long momg_graph_replays(void);

#ifdef __cplusplus
}
#endif
#endif /* MOMG_GPU_H */
