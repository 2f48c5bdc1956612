/* CPU oracle C API -- TEST INFRASTRUCTURE ONLY.
 *
 * Two libraries export this exact API:
 *   oracle/liboracle.so        the plain-C restatement (momg_oracle.c), and
 *   oracle/_ref/libmomg_ref.so the reference itself (/root/reference/proj/src,
 *                              compiled against oracle/shim) behind
 *                              ref_harness.cpp.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load either; the product (paper_2206_13164_b200) never does.
 *
 * Layout (host, row-major, i fastest, flat cell index = j*nx + i):
 *   coeffs[cell*N + k]  Hermite coefficients, k in graded-lex order
 *                       (multi_index.hpp:25-34), N = (M+1)(M+2)(M+3)/6
 *   params[cell*4 + q]  basis (mean_x, mean_y, mean_z, spread)  (moment_rep.hpp:16-20)
 * Residual arrays use the cell params of the field they were evaluated on
 * (spatial.cpp:128); rhs / defect arrays carry their own params
 * (single_level.hpp:42-45).
 */
#ifndef MOMG_ORACLE_H
#define MOMG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: the reference's exception hierarchy (types.hpp:20-57). */
enum {
  MO_OK = 0,
  MO_NONPHYSICAL_STATE = 1, /* NonphysicalState */
  MO_SOLVER_ERROR = 2,      /* SolverError */
  MO_ERROR = 3,             /* plain Error (e.g. grad_normalize cap, projection.hpp:118) */
  MO_NON_SPD = 4,           /* NonSpdTensor */
  MO_CONFIG = 5,            /* ConfigError */
  MO_NONCONVERGENCE = 6     /* NonConvergence (multigrid.hpp:89-97) */
};

typedef struct mo_err {
  int code;
  char msg[256];
} mo_err;

/* Grid2D (grid.hpp:12-37): per-cell sizes and centres. */
typedef struct mo_grid {
  int nx, ny;
  double Lx, Ly;
  const double *dx, *dy, *xc, *yc;
} mo_grid;

enum { MO_BGK = 0, MO_ES_BGK = 1, MO_SHAKHOV = 2 };
enum { MO_WALL_LEFT = 0, MO_WALL_RIGHT = 1, MO_WALL_BOTTOM = 2, MO_WALL_TOP = 3 };

/* SolveContext (single_level.hpp:27-34) flattened. */
typedef struct mo_ctx {
  int M;               /* moment order */
  int space_order;     /* SpatialScheme.order: 1 or 2 */
  double c_bound;      /* SpatialScheme.c_bound */
  double cfl;          /* CflPolicy.cfl */
  double cfl_c_bound;  /* CflPolicy.c_bound */
  int collision;       /* MO_BGK / MO_ES_BGK / MO_SHAKHOV */
  double prandtl;
  double knudsen;
  double viscosity_index;
  double wall_speed[4]; /* left, right, bottom, top */
  double wall_theta[4];
  int threads;
} mo_ctx;

/* Solver report (multigrid.hpp:78-87). history holds rel_residual per iter. */
typedef struct mo_report {
  int converged;
  int iterations;
  double r0_norm;
  double final_norm;
  double final_ratio;
  long long work;
  double seconds;
  int history_len;
  double* history; /* caller-provided, capacity history_cap */
  int history_cap;
} mo_report;

int mo_index_count(int M);
/* a[3N], down[3N] (down[d*N+k]), up[3N], degree[N], factorial[N] */
void mo_index_tables(int M, int* a, int* down, int* up, int* degree, double* factorial);
double mo_max_hermite_root(int degree);

/* ---- per-rep primitives (params = 4 doubles) ---- */
int mo_project(int M, const double* coeffs, const double* from, const double* to,
               double* out, mo_err* err);
int mo_grad_normalize(int M, double* coeffs, double* params, mo_err* err);
double mo_grad_defect(int M, const double* coeffs);
void mo_half_range_table(int pmax, double a, double* upper /* (pmax+1)^2 */,
                         double* lower);
int mo_half_flux(int M, const double* coeffs, const double* params, int axis,
                 int positive_side, double* out, mo_err* err);
void mo_full_flux(int M, const double* coeffs, const double* params, int axis,
                  double* out);
int mo_face_flux(int M, const double* lc, const double* lp, const double* rc,
                 const double* rp, int axis, double c_bound, double* out,
                 double* out_params, mo_err* err);
int mo_wall_flux(int M, const double* c, const double* p, int axis, int high_side,
                 double speed, double theta, double* out, double* out_params,
                 mo_err* err);
int mo_collision(const mo_ctx* ctx, const double* coeffs, const double* params,
                 double* out, mo_err* err);

/* ---- field operations (the hot path) ---- */
int mo_residual(const mo_ctx* ctx, const mo_grid* g, const double* coeffs,
                const double* params, double* res_out, mo_err* err);
int mo_fast_sweep(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                  const double* rhs_coeffs /* NULL = empty rhs */,
                  const double* rhs_params, const int* sweep_order /* NULL = 0123 */,
                  long long* evals, mo_err* err);
double mo_total_mass(const mo_grid* g, int M, const double* coeffs);
int mo_mass_correction(const mo_grid* g, int M, double* coeffs, double target,
                       mo_err* err);
int mo_restrict_solution(int M, const mo_grid* fine, const double* fc, const double* fp,
                         const mo_grid* coarse, double* cc, double* cp, mo_err* err);
int mo_restrict_residual(int M, const mo_grid* fine, const double* arr_c,
                         const double* arr_p, const double* fine_params,
                         const mo_grid* coarse, const double* coarse_params,
                         double* out, mo_err* err);
int mo_fas_correct(int M, const mo_grid* fine, double* fc, double* fp,
                   const mo_grid* coarse, const double* bc, const double* bp,
                   const double* ac, const double* ap, mo_err* err);
double mo_residual_norm(int M, const mo_grid* g, const double* res,
                        const double* field_params);
/* solver: 0 euler, 1 fs, 2 nmg (SolverKind, multigrid.hpp:99) */
int mo_solve_steady(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                    int solver, double tol, int max_iterations, int levels, int s1,
                    int s2, int s3, int gamma, mo_report* report, mo_err* err);
int mo_nmg_cycle(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                 int levels, int s1, int s2, int s3, int gamma, long long* work,
                 mo_err* err);
int mo_sweep_cells(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                   const double* rhs_coeffs, const double* rhs_params, const int* cells, int n,
                   mo_err* err);
int mo_euler_step(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                  mo_err* err);
/* euler_step with an rhs (single_level.cpp:74-97, update_delta :63-70); rhs nullable */
int mo_euler_step_rhs(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                      const double* rhs_coeffs, const double* rhs_params, mo_err* err);

#ifdef __cplusplus
}
#endif
#endif
