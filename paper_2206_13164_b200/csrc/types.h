// Plain types shared by host and device code of momg_gpu (no device code).
#pragma once

#include <stddef.h>
#include <stdint.h>

#ifdef __CUDACC__
#define MOMG_HD __host__ __device__
#else
#define MOMG_HD
#endif

namespace momg_gpu {

MOMG_HD constexpr int tet(int d) { return d * (d + 1) * (d + 2) / 6; }
MOMG_HD constexpr int tri(int r) { return r * (r + 1) / 2; }
// Graded-lex flat index of (a1,a2,a3) (multi_index.hpp:31-40 in closed form).
MOMG_HD constexpr int flat3(int a1, int a2, int a3) {
  return tet(a1 + a2 + a3) + tri(a2 + a3) + a3;
}

// Error codes (match include/momg_gpu.h).
enum : int {
  E_OK = 0,
  E_NONPHYSICAL = 1,
  E_SOLVER = 2,
  E_ERROR = 3,
  E_NONSPD = 4,
  E_CONFIG = 5,
};

// Which failure inside a cell evaluation (for the message).
enum : int {
  W_NONE = 0,
  W_GRAD_RHO = 1,      // grad_normalize: nonpositive/non-finite density
  W_GRAD_THETA = 2,    // grad_normalize: nonpositive/non-finite temperature
  W_GRAD_U = 3,        // grad_normalize: non-finite velocity
  W_GRAD_CAP = 4,      // grad_normalize: iteration cap (plain Error)
  W_PROJ_SPREAD = 5,   // project_coeffs: target spread <= 0
  W_MACRO_RHO = 6,     // extract_macro / maxwellian: nonpositive density
  W_WALL_DEGEN = 7,    // wall_flux: degenerate incoming flux
  W_WALL_RHO = 8,      // wall_flux: nonpositive wall density
  W_HALF_SPREAD = 9,   // half_flux: nonpositive spread
  W_DT_THETA = 10,     // local_dt: nonpositive temperature
  W_DT_HALVING = 11,   // apply_update: failed after dt halving (SolverError)
  W_FAS = 12,          // fas_correct: nonphysical after correction (SolverError)
  W_RESTRICT = 13,     // restrict_solution: nonphysical coarse state
  W_ES_UNSUPPORTED = 14,
  W_DEADLOCK = 15,     // persistent sweep: dependency wait timed out (bug guard)
  W_MASS = 16,         // mass_correction: nonpositive / non-finite total mass
  W_NON_SPD = 17,      // equilibrium_rep: ES-BGK tensor not SPD (NonSpdTensor)
};

// Problem constants (SolveContext, single_level.hpp:27-34), by value per launch.
struct DevCtx {
  int order;           // spatial reconstruction order (1/2)
  int collision;       // 0 bgk, 1 es-bgk, 2 shakhov
  double c_bound;      // SpatialScheme.c_bound
  double cfl;          // CflPolicy.cfl
  double cfl_c_bound;  // CflPolicy.c_bound
  double nu_coef;      // beta*sqrt(pi/2)/Kn (collision.hpp:41-43)
  double nu_exp;       // 1 - viscosity_index
  double shakhov_w;    // (1 - Pr)/5 (collision.hpp:99)
  double prandtl;
  int threads;         // SolveContext.threads (blocked-parallel sweeps when > 1)
  double wall_speed[4];  // left, right, bottom, top
  double wall_theta[4];
};

// One level's device-resident field: coefficients [cells][NP] (cell-major,
// coefficient-minor; 32 B-aligned rows) and basis params [cells][4].
struct DevField {
  int nx, ny;
  double* c;
  double* p;
  const double* dx;
  const double* dy;
  const double* xc;
  const double* yc;
};

// Device error record: first failure wins (atomicCAS on code).
struct DevErr {
  int code;
  int what;
  int i, j;
  double value;
};

}  // namespace momg_gpu
