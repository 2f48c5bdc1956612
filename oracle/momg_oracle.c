/* CPU restatement of the reference's NMG / fast-sweeping path -- TEST
 * INFRASTRUCTURE ONLY (the checker, never the product; see momg_oracle.h).
 *
 * Plain C11, serial, written from the reference's algorithm with the same
 * operation order so that it reproduces the reference bit for bit on baseline
 * x86-64 (no FMA contraction: -ffp-contract=off).  Every function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * Exceptions become mo_err codes; the C++ catch sites (safe_face_state,
 * apply_update's dt/2 retry, solve_steady's NonConvergence mapping) are
 * reproduced explicitly.
 *
 * PINNING: tests/test_oracle_pin.py checks this library against (a) the
 * reference itself compiled here (oracle/_ref/libmomg_ref.so; bitwise on the
 * field operations) and (b) the reference unit tests' known answers and the
 * committed golden vectors in tests/golden/.
 */
#include "momg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXM 24

/* ------------------------------------------------------------------ errors */

static int fail(mo_err* err, int code, const char* fmt, ...) {
  if (err) {
    va_list ap;
    va_start(ap, fmt);
    err->code = code;
    vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}
static void clear(mo_err* err) {
  if (err) {
    err->code = MO_OK;
    err->msg[0] = 0;
  }
}
#define TRY(x)              \
  do {                      \
    int rc_ = (x);          \
    if (rc_ != MO_OK) return rc_; \
  } while (0)

/* --------------------------------------------------------------- index set */
/* IndexSet, multi_index.hpp:25-103: graded lex, ascending degree, descending
 * lexicographic within a degree; flat lookup; down/up neighbours; alpha!. */
typedef struct iset {
  int M, n;
  int* a;       /* 3n */
  int* flat;    /* (M+1)^3 */
  int* down[3]; /* n each */
  int* up[3];
  int* deg;
  double* fact;
} iset;

static iset g_sets[MAXM + 1];

static double fact_int(int n) { /* multi_index.hpp:88-92 */
  double r = 1;
  for (int i = 2; i <= n; ++i) r *= i;
  return r;
}

static int iset_find(const iset* s, int a1, int a2, int a3) { /* :66-70 */
  const int side = s->M + 1;
  if (a1 < 0 || a2 < 0 || a3 < 0 || a1 + a2 + a3 > s->M) return -1;
  return s->flat[(a1 * side + a2) * side + a3];
}

static const iset* get_set(int M) {
  if (M < 0 || M > MAXM) return NULL;
  iset* s = &g_sets[M];
  if (s->a) return s;
  const int n = (M + 1) * (M + 2) * (M + 3) / 6; /* count, :82-84 */
  const int side = M + 1;
  s->M = M;
  s->n = n;
  s->a = (int*)malloc(sizeof(int) * 3 * n);
  s->flat = (int*)malloc(sizeof(int) * side * side * side);
  for (int i = 0; i < side * side * side; ++i) s->flat[i] = -1;
  int k = 0;
  for (int deg = 0; deg <= M; ++deg) /* :31-34 */
    for (int a1 = deg; a1 >= 0; --a1)
      for (int a2 = deg - a1; a2 >= 0; --a2) {
        s->a[3 * k] = a1;
        s->a[3 * k + 1] = a2;
        s->a[3 * k + 2] = deg - a1 - a2;
        s->flat[(a1 * side + a2) * side + (deg - a1 - a2)] = k;
        ++k;
      }
  for (int d = 0; d < 3; ++d) { /* :41-52 */
    s->down[d] = (int*)malloc(sizeof(int) * n);
    s->up[d] = (int*)malloc(sizeof(int) * n);
    for (k = 0; k < n; ++k) {
      int a[3] = {s->a[3 * k], s->a[3 * k + 1], s->a[3 * k + 2]};
      --a[d];
      s->down[d][k] = iset_find(s, a[0], a[1], a[2]);
      a[d] += 2;
      s->up[d][k] = iset_find(s, a[0], a[1], a[2]);
    }
  }
  s->deg = (int*)malloc(sizeof(int) * n);
  s->fact = (double*)malloc(sizeof(double) * n);
  for (k = 0; k < n; ++k) { /* :53-58 */
    s->deg[k] = s->a[3 * k] + s->a[3 * k + 1] + s->a[3 * k + 2];
    s->fact[k] = fact_int(s->a[3 * k]) * fact_int(s->a[3 * k + 1]) * fact_int(s->a[3 * k + 2]);
  }
  return s;
}

int mo_index_count(int M) { return (M + 1) * (M + 2) * (M + 3) / 6; }

void mo_index_tables(int M, int* a, int* down, int* up, int* degree, double* factorial) {
  const iset* s = get_set(M);
  const int n = s->n;
  memcpy(a, s->a, sizeof(int) * 3 * n);
  for (int d = 0; d < 3; ++d) {
    memcpy(down + d * n, s->down[d], sizeof(int) * n);
    memcpy(up + d * n, s->up[d], sizeof(int) * n);
  }
  memcpy(degree, s->deg, sizeof(int) * n);
  memcpy(factorial, s->fact, sizeof(double) * n);
}

/* max_hermite_root, tables.cpp:22-41.  The reference takes the top eigenvalue
 * of the Jacobi matrix; restated here as Newton on He_n from the Gershgorin
 * upper bound 2*sqrt(n-1) (monotone convergence to the largest root), polished
 * to a fixed point.  Agrees with the reference to ~1 ulp (tested). */
static double he_eval(int n, double x, double* dprime) { /* hermite.hpp:10-21 */
  double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0;
  if (n == 0) {
    if (dprime) *dprime = 0.0;
    return 1.0;
  }
  for (int k = 1; k < n; ++k) {
    const double p2 = x * p1 - k * p0;
    const double d2 = p1 + x * d1 - k * d0;
    p0 = p1;
    p1 = p2;
    d0 = d1;
    d1 = d2;
  }
  if (dprime) *dprime = d1;
  return p1;
}
double mo_max_hermite_root(int degree) {
  if (degree < 1) return NAN;
  if (degree == 1) return 0.0;
  double x = 2.0 * sqrt((double)degree) + 1.0;
  for (int it = 0; it < 200; ++it) {
    double d;
    const double p = he_eval(degree, x, &d);
    const double nx = x - p / d;
    if (nx == x || fabs(nx - x) <= 1e-16 * fabs(x)) {
      x = nx;
      break;
    }
    x = nx;
  }
  return x;
}

/* -------------------------------------------------------------- projection */
/* shift_mean_coeffs, projection.hpp:16-30 */
static void shift_mean(const iset* s, double* c, int axis, double delta) {
  if (delta == 0.0) return;
  for (int k = s->n - 1; k >= 0; --k) {
    double acc = c[k];
    double w = 1.0;
    int n = 1;
    for (int j = s->down[axis][k]; j >= 0; j = s->down[axis][j]) {
      w *= -delta / (double)(n++);
      acc += w * c[j];
    }
    c[k] = acc;
  }
}

/* shift_spread_coeffs, projection.hpp:35-57 */
static void shift_spread(const iset* s, double* c, double delta) {
  if (delta == 0.0) return;
  const int n = s->n;
  double cur[1 << 12], nxt[1 << 12];
  memcpy(cur, c, sizeof(double) * n);
  double w = 1.0;
  for (int k = 1; 2 * k <= s->M; ++k) {
    w *= -delta / (2.0 * (double)k);
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int d = 0; d < 3; ++d) {
        int j = s->down[d][i];
        if (j >= 0) j = s->down[d][j];
        if (j >= 0) acc += cur[j];
      }
      nxt[i] = acc;
    }
    for (int i = 0; i < n; ++i) c[i] += w * nxt[i];
    memcpy(cur, nxt, sizeof(double) * n);
  }
}

/* project_coeffs, projection.hpp:64-73 */
static int project_coeffs(const iset* s, double* c, const double* from, const double* to,
                          mo_err* err) {
  if (!(to[3] > 0.0))
    return fail(err, MO_NONPHYSICAL_STATE, "project_coeffs: target spread must be positive");
  for (int d = 0; d < 3; ++d) shift_mean(s, c, d, to[d] - from[d]);
  shift_spread(s, c, to[3] - from[3]);
  return MO_OK;
}

/* project, projection.hpp:83-89 (copy + project_in_place) */
static int project_to(const iset* s, const double* c, const double* from, const double* to,
                      double* out, mo_err* err) {
  if (out != c) memcpy(out, c, sizeof(double) * s->n);
  return project_coeffs(s, out, from, to, err);
}

int mo_project(int M, const double* coeffs, const double* from, const double* to,
               double* out, mo_err* err) {
  clear(err);
  return project_to(get_set(M), coeffs, from, to, out, err);
}

/* std::max / std::min semantics: max(a,b) = (a < b) ? b : a */
static double smax(double a, double b) { return (a < b) ? b : a; }
static double smin(double a, double b) { return (b < a) ? b : a; }

/* rep_velocity, moment_rep.hpp:69-76 */
static void rep_velocity(const iset* s, const double* c, const double* p, double* u) {
  const double rho = c[0];
  for (int d = 0; d < 3; ++d) u[d] = p[d] + c[1 + d] / rho;
  (void)s;
}
/* rep_temperature, moment_rep.hpp:80-93 */
static double rep_temperature(const iset* s, const double* c, const double* p) {
  const double rho = c[0];
  double trace = 0.0, fe2 = 0.0;
  for (int d = 0; d < 3; ++d) {
    trace += c[s->up[d][1 + d]];
    fe2 += c[1 + d] * c[1 + d];
  }
  return p[3] + (2.0 * trace - fe2 / rho) / (3.0 * rho);
}
/* grad_defect, moment_rep.hpp:97-110 */
static double grad_defect(const iset* s, const double* c) {
  double defect = 0.0, trace = 0.0;
  for (int d = 0; d < 3; ++d) {
    defect = smax(defect, fabs(c[1 + d]));
    trace += c[s->up[d][1 + d]];
  }
  defect = smax(defect, fabs(trace));
  return defect / fabs(c[0]);
}
double mo_grad_defect(int M, const double* coeffs) { return grad_defect(get_set(M), coeffs); }

/* grad_normalize, projection.hpp:96-121 (rel_tol 1e-12, max_iter 30) */
static int grad_normalize(const iset* s, double* c, double* p, mo_err* err) {
  const double rel_tol = 1e-12;
  for (int iter = 0; iter < 30; ++iter) {
    const double rho = c[0];
    if (!isfinite(rho) || !(rho > 0.0))
      return fail(err, MO_NONPHYSICAL_STATE,
                  "grad_normalize: nonpositive or non-finite density %f", rho);
    if (grad_defect(s, c) <= rel_tol) return MO_OK;
    double to[4];
    rep_velocity(s, c, p, to);
    to[3] = rep_temperature(s, c, p);
    if (!isfinite(to[3]) || !(to[3] > 0.0))
      return fail(err, MO_NONPHYSICAL_STATE,
                  "grad_normalize: nonpositive or non-finite temperature %f", to[3]);
    for (int d = 0; d < 3; ++d)
      if (!isfinite(to[d]))
        return fail(err, MO_NONPHYSICAL_STATE, "grad_normalize: non-finite velocity");
    TRY(project_coeffs(s, c, p, to, err));
    memcpy(p, to, sizeof(double) * 4);
  }
  if (grad_defect(s, c) > rel_tol)
    return fail(err, MO_ERROR, "grad_normalize: tolerance not reached within iteration cap");
  return MO_OK;
}
int mo_grad_normalize(int M, double* coeffs, double* params, mo_err* err) {
  clear(err);
  return grad_normalize(get_set(M), coeffs, params, err);
}

/* -------------------------------------------------------------- collision */
/* extract_macro, moment_rep.hpp:116-146 */
typedef struct macro_state {
  double rho, u[3], theta, sigma[3][3], q[3];
} macro_state;

static int extract_macro(const iset* s, const double* c, const double* p, macro_state* m,
                         mo_err* err) {
  if (s->M < 3) return fail(err, MO_ERROR, "extract_macro: order must be >= 3");
  if (!(c[0] > 0.0)) return fail(err, MO_NONPHYSICAL_STATE, "extract_macro: nonpositive density");
  m->rho = c[0];
  for (int d = 0; d < 3; ++d) m->u[d] = p[d];
  m->theta = p[3];
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      const int k = s->up[j][1 + i];
      const double delta = (i == j) ? 1.0 : 0.0;
      m->sigma[i][j] = (1.0 + delta) * c[k];
      m->sigma[j][i] = m->sigma[i][j];
    }
  for (int i = 0; i < 3; ++i) {
    double q = 2.0 * c[iset_find(s, i == 0 ? 3 : 0, i == 1 ? 3 : 0, i == 2 ? 3 : 0)];
    for (int d = 0; d < 3; ++d) {
      int a[3] = {0, 0, 0};
      a[d] += 2;
      a[i] += 1;
      q += c[iset_find(s, a[0], a[1], a[2])];
    }
    m->q[i] = q;
  }
  return MO_OK;
}

/* Symmetric 3x3 minimum eigenvalue by cyclic Jacobi (only the ES-BGK SPD
 * check uses it, collision.hpp:88-92). */
static double min_eig3(const double A[3][3]) {
  double a[3][3];
  memcpy(a, A, sizeof(a));
  for (int sweep = 0; sweep < 60; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    if (off == 0.0) break;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = cs * akp - sn * akq;
          a[k][q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = cs * apk - sn * aqk;
          a[q][k] = sn * apk + cs * aqk;
        }
      }
  }
  return smin(smin(a[0][0], a[1][1]), a[2][2]);
}

/* collision_frequency, collision.hpp:36-44 */
static double collision_frequency(const mo_ctx* ctx, double rho, double theta) {
  const double root_half_pi = sqrt(atan(1.0) * 2.0);
  const double beta = ctx->collision == MO_ES_BGK ? ctx->prandtl : 1.0;
  return beta * root_half_pi / ctx->knudsen * rho * pow(theta, 1.0 - ctx->viscosity_index);
}

/* equilibrium_rep, collision.hpp:78-114 (+ maxwellian_rep moment_rep.hpp:47-59,
 * gaussian_rep collision.hpp:52-71) into eq[] in the basis (u, theta). */
static int equilibrium(const mo_ctx* ctx, const iset* s, const macro_state* m, double* eq,
                       mo_err* err) {
  if (!(m->rho > 0.0) || !(m->theta > 0.0))
    return fail(err, MO_NONPHYSICAL_STATE, "maxwellian_rep: rho and theta must be positive");
  memset(eq, 0, sizeof(double) * s->n);
  eq[0] = m->rho;
  if (ctx->collision == MO_BGK) return MO_OK;
  if (ctx->collision == MO_SHAKHOV) {
    if (s->M >= 3) {
      const double w = (1.0 - ctx->prandtl) / 5.0;
      for (int d = 0; d < 3; ++d)
        for (int dd = 0; dd < 3; ++dd) {
          int a[3] = {0, 0, 0};
          a[dd] += 2;
          a[d] += 1;
          eq[iset_find(s, a[0], a[1], a[2])] = w * m->q[d];
        }
    }
    return MO_OK;
  }
  /* ES-BGK */
  const double corr = 1.0 - 1.0 / ctx->prandtl;
  double lambda[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      lambda[i][j] = m->theta * (i == j ? 1.0 : 0.0) + corr / m->rho * m->sigma[i][j];
  const double me = min_eig3(lambda);
  if (!(me > 1e-12 * m->theta))
    return fail(err, MO_NON_SPD, "equilibrium_rep: anisotropic-Gaussian tensor not SPD");
  double cmat[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) cmat[i][j] = lambda[i][j] - m->theta * (i == j ? 1.0 : 0.0);
  for (int k = 1; k < s->n; ++k) {
    if (s->deg[k] % 2 == 1) continue;
    int d = 0;
    while (s->down[d][k] < 0) ++d;
    const int mu = s->down[d][k];
    double acc = 0.0;
    for (int j = 0; j < 3; ++j) {
      const int i = s->down[j][mu];
      if (i >= 0) acc += cmat[d][j] * eq[i];
    }
    eq[k] = acc / (double)(s->a[3 * mu + d] + 1);
  }
  return MO_OK;
}

/* collision_coeffs, collision.hpp:120-127 */
static int collision(const mo_ctx* ctx, const iset* s, const double* c, const double* p,
                     double* out, mo_err* err) {
  macro_state m = {0};
  TRY(extract_macro(s, c, p, &m, err));
  if (!(ctx->knudsen > 0.0))
    return fail(err, MO_CONFIG, "collision_frequency: Kn must be positive");
  const double nu = collision_frequency(ctx, m.rho, m.theta);
  double eq[1 << 12];
  TRY(equilibrium(ctx, s, &m, eq, err));
  for (int k = 0; k < s->n; ++k) out[k] = nu * (eq[k] - c[k]);
  return MO_OK;
}
int mo_collision(const mo_ctx* ctx, const double* coeffs, const double* params, double* out,
                 mo_err* err) {
  clear(err);
  return collision(ctx, get_set(ctx->M), coeffs, params, out, err);
}

/* ------------------------------------------------------------------ fluxes */
/* HalfRangeTable, halfspace.hpp:18-57: upper (pmax+1)^2 row-major [m][p]. */
static void half_range(int pmax, double a, double* up, double* fullmn) {
  const int n = pmax + 1;
  double he[MAXM + 4];
  he[0] = 1.0;
  if (pmax >= 1) he[1] = a;
  for (int k = 1; k + 1 <= pmax; ++k) he[k + 1] = a * he[k] - (double)k * he[k - 1];
  const double g = exp(-a * a / 2.0) / sqrt(8.0 * atan(1.0));
  for (int i = 0; i < n * n; ++i) up[i] = 0.0;
  fullmn[0] = 1.0;
  for (int k = 1; k <= pmax; ++k) fullmn[k] = fullmn[k - 1] * (double)k;
  up[0] = erfc(a / sqrt(2.0)) / 2.0;
  for (int p = 1; p <= pmax; ++p) up[p] = he[p - 1] * g;
  for (int m = 0; m + 1 <= pmax; ++m)
    for (int p = 0; p <= pmax; ++p)
      up[(m + 1) * n + p] = (p > 0 ? (double)p * up[m * n + p - 1] : 0.0) + he[m] * he[p] * g;
}
void mo_half_range_table(int pmax, double a, double* upper, double* lower) {
  double fullmn[MAXM + 4];
  half_range(pmax, a, upper, fullmn);
  const int n = pmax + 1;
  for (int m = 0; m < n; ++m)
    for (int p = 0; p < n; ++p)
      lower[m * n + p] = (m == p ? fullmn[p] : 0.0) - upper[m * n + p];
}

/* full_flux_coeffs, flux.cpp:10-27 */
static void full_flux(const iset* s, const double* c, const double* p, int axis, double* out) {
  const double mean_n = p[axis];
  const double spread = p[3];
  for (int k = 0; k < s->n; ++k) {
    double g = mean_n * c[k];
    const int down = s->down[axis][k];
    if (down >= 0) g += spread * c[down];
    const int up = s->up[axis][k];
    if (up >= 0) g += (double)(s->a[3 * k + axis] + 1) * c[up];
    out[k] = g;
  }
}
void mo_full_flux(int M, const double* coeffs, const double* params, int axis, double* out) {
  full_flux(get_set(M), coeffs, params, axis, out);
}

/* half_flux_coeffs, flux.cpp:29-75 */
static int half_flux(const iset* s, const double* c, const double* p, int axis, int positive,
                     double* out, mo_err* err) {
  const int M = s->M;
  const double spread = p[3];
  if (!(spread > 0.0))
    return fail(err, MO_NONPHYSICAL_STATE, "half_flux_coeffs: nonpositive basis spread");
  const double rs = sqrt(spread);
  const double a = -p[axis] / rs;
  const int pmax = M + 1, tn = pmax + 1;
  double up[(MAXM + 3) * (MAXM + 3)], fullmn[MAXM + 4];
  half_range(pmax, a, up, fullmn);
  double rs_pow[2 * MAXM + 4];
  const int off = M;
  rs_pow[off] = 1.0;
  for (int e = 1; e <= M + 1; ++e) rs_pow[off + e] = rs_pow[off + e - 1] * rs;
  for (int e = -1; e >= -M; --e) rs_pow[off + e] = rs_pow[off + e + 1] / rs;
  const double mean_n = p[axis];
  double fact[MAXM + 2];
  fact[0] = 1.0;
  for (int q = 1; q <= M; ++q) fact[q] = fact[q - 1] * (double)q;
#define PAIR(m, q) \
  (positive ? up[(m) * tn + (q)] : (((m) == (q) ? fullmn[q] : 0.0) - up[(m) * tn + (q)]))
  for (int k = 0; k < s->n; ++k) {
    int idx[3] = {s->a[3 * k], s->a[3 * k + 1], s->a[3 * k + 2]};
    const int q = idx[axis];
    const int tan_deg = s->deg[k] - q;
    double acc = 0.0;
    for (int m = 0; m + tan_deg <= M; ++m) {
      idx[axis] = m;
      const double f = c[iset_find(s, idx[0], idx[1], idx[2])];
      if (f == 0.0) continue;
      double kernel = mean_n * PAIR(m, q) + rs * PAIR(m + 1, q);
      if (m > 0) kernel += rs * (double)m * PAIR(m - 1, q);
      acc += rs_pow[off + (q - m)] * f * kernel;
    }
    out[k] = acc / fact[q];
  }
#undef PAIR
  return MO_OK;
}
int mo_half_flux(int M, const double* coeffs, const double* params, int axis,
                 int positive_side, double* out, mo_err* err) {
  clear(err);
  return half_flux(get_set(M), coeffs, params, axis, positive_side, out, err);
}

/* face_flux, flux.cpp:77-97 -> out in the face basis fp */
static int face_flux(const iset* s, const double* lc, const double* lp, const double* rc,
                     const double* rp, int axis, double c_bound, double* out, double* fp,
                     mo_err* err) {
  double ulv[3], urv[3];
  rep_velocity(s, lc, lp, ulv);
  rep_velocity(s, rc, rp, urv);
  const double ul = ulv[axis], ur = urv[axis];
  const double cl = c_bound * sqrt(rep_temperature(s, lc, lp));
  const double cr = c_bound * sqrt(rep_temperature(s, rc, rp));
  const double lambda_minus = smin(ul - cl, ur - cr);
  const double lambda_plus = smax(ul + cl, ur + cr);
  for (int d = 0; d < 3; ++d) fp[d] = 0.5 * (lp[d] + rp[d]);
  fp[3] = 0.5 * (lp[3] + rp[3]);
  double tmp[1 << 12];
  if (lambda_minus >= 0.0) {
    TRY(project_to(s, lc, lp, fp, tmp, err));
    full_flux(s, tmp, fp, axis, out);
    return MO_OK;
  }
  if (lambda_plus <= 0.0) {
    TRY(project_to(s, rc, rp, fp, tmp, err));
    full_flux(s, tmp, fp, axis, out);
    return MO_OK;
  }
  double low[1 << 12];
  TRY(project_to(s, lc, lp, fp, tmp, err));
  TRY(half_flux(s, tmp, fp, axis, 1, out, err));
  TRY(project_to(s, rc, rp, fp, tmp, err));
  TRY(half_flux(s, tmp, fp, axis, 0, low, err));
  for (int k = 0; k < s->n; ++k) out[k] += low[k];
  return MO_OK;
}
int mo_face_flux(int M, const double* lc, const double* lp, const double* rc, const double* rp,
                 int axis, double c_bound, double* out, double* out_params, mo_err* err) {
  clear(err);
  return face_flux(get_set(M), lc, lp, rc, rp, axis, c_bound, out, out_params, err);
}

/* wall_flux, flux.cpp:105-130 -> out in the wall basis wp */
static int wall_flux(const iset* s, const double* c, const double* p, int axis, int high,
                     double speed, double theta, double* out, double* wp, mo_err* err) {
  wp[0] = wp[1] = wp[2] = 0.0;
  wp[axis == 0 ? 1 : 0] = speed;
  wp[3] = theta;
  double inside_w[1 << 12], unit[1 << 12], in_unit[1 << 12];
  TRY(project_to(s, c, p, wp, inside_w, err));
  memset(unit, 0, sizeof(double) * s->n);
  unit[0] = 1.0;
  TRY(half_flux(s, inside_w, wp, axis, high, out, err));
  TRY(half_flux(s, unit, wp, axis, !high, in_unit, err));
  if (in_unit[0] == 0.0)
    return fail(err, MO_NONPHYSICAL_STATE, "wall_flux: degenerate incoming wall flux");
  const double wall_rho = -out[0] / in_unit[0];
  if (!(wall_rho > 0.0))
    return fail(err, MO_NONPHYSICAL_STATE, "wall_flux: nonpositive wall density");
  for (int k = 0; k < s->n; ++k) out[k] += wall_rho * in_unit[k];
  out[0] = 0.0;
  return MO_OK;
}
int mo_wall_flux(int M, const double* c, const double* p, int axis, int high_side, double speed,
                 double theta, double* out, double* out_params, mo_err* err) {
  clear(err);
  return wall_flux(get_set(M), c, p, axis, high_side, speed, theta, out, out_params, err);
}

/* ----------------------------------------------------------------- spatial */
typedef struct fieldv {
  const mo_grid* g;
  const iset* s;
  double* c; /* cells * n */
  double* p; /* cells * 4 */
} fieldv;

#define CELL(f, i, j) ((size_t)(j) * (f)->g->nx + (i))

/* safe_face_state(face_state(slope_along)), spatial.cpp:34-80: writes the
 * reconstructed state of cell (i,j) on its +/-axis face into wc/wp. */
static void safe_face_state(const mo_ctx* ctx, const fieldv* f, int i, int j, int axis,
                            int high, double* wc, double* wp) {
  const iset* s = f->s;
  const size_t k = CELL(f, i, j);
  const double* cc = f->c + k * s->n;
  const double* cp = f->p + k * 4;
  memcpy(wc, cc, sizeof(double) * s->n);
  memcpy(wp, cp, sizeof(double) * 4);
  if (ctx->space_order == 1) return;
  const mo_grid* g = f->g;
  const int m = axis == 0 ? i : j;
  const int last = (axis == 0 ? g->nx : g->ny) - 1;
  const double off = (high ? 0.5 : -0.5) * (axis == 0 ? g->dx[i] : g->dy[j]);
  double sm[3] = {0, 0, 0}, ss = 0.0;
  if (m == 0 || m == last) {
    /* zero slope (spatial.cpp:39-42): w = cell + off * 0 */
    for (int d = 0; d < 3; ++d) wp[d] += off * 0.0;
    wp[3] += off * 0.0;
    for (int q = 0; q < s->n; ++q) wc[q] += off * 0.0;
  } else {
    const size_t klo = axis == 0 ? CELL(f, i - 1, j) : CELL(f, i, j - 1);
    const size_t khi = axis == 0 ? CELL(f, i + 1, j) : CELL(f, i, j + 1);
    const double h = axis == 0 ? g->xc[i + 1] - g->xc[i - 1] : g->yc[j + 1] - g->yc[j - 1];
    const double* lp = f->p + klo * 4;
    const double* hp = f->p + khi * 4;
    for (int d = 0; d < 3; ++d) sm[d] = (hp[d] - lp[d]) / h;
    ss = (hp[3] - lp[3]) / h;
    for (int d = 0; d < 3; ++d) wp[d] += off * sm[d];
    wp[3] += off * ss;
    const double* lc = f->c + klo * s->n;
    const double* hc = f->c + khi * s->n;
    for (int q = 0; q < s->n; ++q) wc[q] += off * ((hc[q] - lc[q]) / h);
  }
  if (!(wp[3] > 0.0)) { /* NonphysicalReconstruction -> first-order fallback */
    memcpy(wc, cc, sizeof(double) * s->n);
    memcpy(wp, cp, sizeof(double) * 4);
  }
}

/* face lambda of cell_residual, spatial.cpp:106-124: flux through the
 * (axis, high) face of (i,j) projected into the cell basis. */
static int cell_face(const mo_ctx* ctx, const fieldv* f, int i, int j, int axis, int high,
                     double* out, mo_err* err) {
  const iset* s = f->s;
  const mo_grid* g = f->g;
  const size_t k = CELL(f, i, j);
  const double* cc = f->c + k * s->n;
  const double* cp = f->p + k * 4;
  const int at_wall = axis == 0 ? (high ? i == g->nx - 1 : i == 0)
                                : (high ? j == g->ny - 1 : j == 0);
  double flux[1 << 12], fp[4];
  if (at_wall) {
    const int w = axis == 0 ? (high ? MO_WALL_RIGHT : MO_WALL_LEFT)
                            : (high ? MO_WALL_TOP : MO_WALL_BOTTOM);
    TRY(wall_flux(s, cc, cp, axis, high, ctx->wall_speed[w], ctx->wall_theta[w], flux, fp, err));
    return project_to(s, flux, fp, cp, out, err);
  }
  const int ni = axis == 0 ? (high ? i + 1 : i - 1) : i;
  const int nj = axis == 1 ? (high ? j + 1 : j - 1) : j;
  double loc[1 << 12], lop[4], hic[1 << 12], hip[4];
  safe_face_state(ctx, f, high ? i : ni, high ? j : nj, axis, 1, loc, lop);
  safe_face_state(ctx, f, high ? ni : i, high ? nj : j, axis, 0, hic, hip);
  TRY(face_flux(s, loc, lop, hic, hip, axis, ctx->c_bound, flux, fp, err));
  return project_to(s, flux, fp, cp, out, err);
}

/* cell_residual, spatial.cpp:98-133 */
static int cell_residual(const mo_ctx* ctx, const fieldv* f, int i, int j, double* r,
                         mo_err* err) {
  const iset* s = f->s;
  const size_t k = CELL(f, i, j);
  TRY(collision(ctx, s, f->c + k * s->n, f->p + k * 4, r, err));
  double fp_[1 << 12], fm_[1 << 12];
  TRY(cell_face(ctx, f, i, j, 0, 1, fp_, err));
  TRY(cell_face(ctx, f, i, j, 0, 0, fm_, err));
  for (int q = 0; q < s->n; ++q) r[q] -= (fp_[q] - fm_[q]) / f->g->dx[i];
  TRY(cell_face(ctx, f, i, j, 1, 1, fp_, err));
  TRY(cell_face(ctx, f, i, j, 1, 0, fm_, err));
  for (int q = 0; q < s->n; ++q) r[q] -= (fp_[q] - fm_[q]) / f->g->dy[j];
  return MO_OK;
}

/* residual, spatial.cpp:135-159 (serial; first failure in row-major order) */
static int residual(const mo_ctx* ctx, const fieldv* f, double* out, mo_err* err) {
  for (int j = 0; j < f->g->ny; ++j)
    for (int i = 0; i < f->g->nx; ++i)
      TRY(cell_residual(ctx, f, i, j, out + CELL(f, i, j) * f->s->n, err));
  return MO_OK;
}
int mo_residual(const mo_ctx* ctx, const mo_grid* g, const double* coeffs, const double* params,
                double* res_out, mo_err* err) {
  clear(err);
  fieldv f = {g, get_set(ctx->M), (double*)coeffs, (double*)params};
  return residual(ctx, &f, res_out, err);
}

/* ------------------------------------------------------------ single level */
/* local_dt, single_level.cpp:18-24 */
static int local_dt(const mo_ctx* ctx, const double* p, double dx, double dy, double* dt,
                    mo_err* err) {
  const double theta = p[3];
  if (!(theta > 0.0))
    return fail(err, MO_NONPHYSICAL_STATE, "local_dt: nonpositive temperature %f", theta);
  const double c = ctx->cfl_c_bound * sqrt(theta);
  *dt = ctx->cfl / ((fabs(p[0]) + c) / dx + (fabs(p[1]) + c) / dy);
  return MO_OK;
}

/* apply_update, single_level.cpp:44-62 */
static int apply_update(const iset* s, double* c, double* p, const double* delta, double dt,
                        int i, int j, mo_err* err) {
  double saved_c[1 << 12], saved_p[4];
  memcpy(saved_c, c, sizeof(double) * s->n);
  memcpy(saved_p, p, sizeof(double) * 4);
  for (int q = 0; q < s->n; ++q) c[q] += dt * delta[q];
  int rc = grad_normalize(s, c, p, err);
  if (rc == MO_OK) return MO_OK;
  if (rc != MO_NONPHYSICAL_STATE) return rc; /* plain Error propagates */
  memcpy(c, saved_c, sizeof(double) * s->n);
  memcpy(p, saved_p, sizeof(double) * 4);
  const double half = 0.5 * dt;
  for (int q = 0; q < s->n; ++q) c[q] += half * delta[q];
  clear(err);
  rc = grad_normalize(s, c, p, err);
  if (rc == MO_OK) return MO_OK;
  if (rc != MO_NONPHYSICAL_STATE) return rc;
  char what[256];
  snprintf(what, sizeof(what), "%s", err ? err->msg : "");
  memcpy(c, saved_c, sizeof(double) * s->n);
  memcpy(p, saved_p, sizeof(double) * 4);
  return fail(err, MO_SOLVER_ERROR,
              "update left cell (%d,%d) nonphysical after dt halving: %s", i, j, what);
}

/* update_delta, single_level.cpp:64-70 */
static int update_delta(const iset* s, const double* cp, const double* res,
                        const double* rhs_c, const double* rhs_p, double* delta, mo_err* err) {
  memcpy(delta, res, sizeof(double) * s->n);
  if (!rhs_c) return MO_OK;
  double pr[1 << 12];
  TRY(project_to(s, rhs_c, rhs_p, cp, pr, err));
  for (int q = 0; q < s->n; ++q) delta[q] -= pr[q];
  return MO_OK;
}

/* sweep_cell, single_level.cpp:103-111 */
static int sweep_cell(const mo_ctx* ctx, fieldv* f, int i, int j, const double* rhs_c,
                      const double* rhs_p, mo_err* err) {
  const iset* s = f->s;
  const size_t k = CELL(f, i, j);
  double* c = f->c + k * s->n;
  double* p = f->p + k * 4;
  double dt, res[1 << 12], delta[1 << 12];
  TRY(local_dt(ctx, p, f->g->dx[i], f->g->dy[j], &dt, err));
  TRY(cell_residual(ctx, f, i, j, res, err));
  TRY(update_delta(s, p, res, rhs_c ? rhs_c + k * s->n : NULL, rhs_c ? rhs_p + k * 4 : NULL,
                   delta, err));
  return apply_update(s, c, p, delta, dt, i, j, err);
}

/* fast_sweep_step, single_level.cpp:116-166 (threads = 1: exact serial GS) */
static int fast_sweep(const mo_ctx* ctx, fieldv* f, const double* rhs_c, const double* rhs_p,
                      const int* order, long long* evals, mo_err* err) {
  static const int dirs[4][2] = {{1, 1}, {0, 1}, {0, 0}, {1, 0}}; /* :116-117 */
  const int nx = f->g->nx, ny = f->g->ny;
  long long n = 0;
  int rc = MO_OK;
  for (int si = 0; si < 4 && rc == MO_OK; ++si) {
    const int* dir = dirs[order ? order[si] : si];
    for (int step = 0; step < nx && rc == MO_OK; ++step) {
      const int i = dir[0] ? step : nx - 1 - step;
      for (int jj = 0; jj < ny; ++jj) {
        const int j = dir[1] ? jj : ny - 1 - jj;
        rc = sweep_cell(ctx, f, i, j, rhs_c, rhs_p, err);
        if (rc != MO_OK) break;
        ++n;
      }
    }
  }
  if (evals) *evals += n;
  return rc;
}
int mo_fast_sweep(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                  const double* rhs_coeffs, const double* rhs_params, const int* sweep_order,
                  long long* evals, mo_err* err) {
  clear(err);
  fieldv f = {g, get_set(ctx->M), coeffs, params};
  if (evals) *evals = 0;
  return fast_sweep(ctx, &f, rhs_coeffs, rhs_params, sweep_order, evals, err);
}

/* sweep_cell (single_level.cpp:103-111) applied to an explicit list of cells
 * in the given order: the building block of the distributed (row-strip)
 * sweep tests, where each rank updates its own cells of a global-size array
 * whose rows outside its strip + halo are stale. */
int mo_sweep_cells(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                   const double* rhs_coeffs, const double* rhs_params, const int* cells, int n,
                   mo_err* err) {
  clear(err);
  fieldv f = {g, get_set(ctx->M), coeffs, params};
  for (int q = 0; q < n; ++q) {
    const int i = cells[2 * q], j = cells[2 * q + 1];
    TRY(sweep_cell(ctx, &f, i, j, rhs_coeffs, rhs_params, err));
  }
  return MO_OK;
}

/* global_dt, single_level.cpp:31-38 */
static int global_dt(const mo_ctx* ctx, const fieldv* f, double* dt_out, mo_err* err) {
  double dt = INFINITY;
  for (int j = 0; j < f->g->ny; ++j)
    for (int i = 0; i < f->g->nx; ++i) {
      double d;
      TRY(local_dt(ctx, f->p + CELL(f, i, j) * 4, f->g->dx[i], f->g->dy[j], &d, err));
      dt = smin(dt, d);
    }
  *dt_out = dt;
  return MO_OK;
}

/* euler_step, single_level.cpp:74-97 (rhs_c == NULL: empty rhs) */
static int euler_step_rhs(const mo_ctx* ctx, fieldv* f, const double* res, const double* rhs_c,
                          const double* rhs_p, mo_err* err) {
  double dt;
  TRY(global_dt(ctx, f, &dt, err));
  const iset* s = f->s;
  double* delta = (double*)malloc(sizeof(double) * s->n);
  int rc = MO_OK;
  for (int j = 0; j < f->g->ny && rc == MO_OK; ++j)
    for (int i = 0; i < f->g->nx && rc == MO_OK; ++i) {
      const size_t k = CELL(f, i, j);
      rc = update_delta(s, f->p + k * 4, res + k * s->n, rhs_c ? rhs_c + k * s->n : NULL,
                        rhs_c ? rhs_p + k * 4 : NULL, delta, err);
      if (rc == MO_OK) rc = apply_update(s, f->c + k * s->n, f->p + k * 4, delta, dt, i, j, err);
    }
  free(delta);
  return rc;
}
static int euler_step(const mo_ctx* ctx, fieldv* f, const double* res, mo_err* err) {
  return euler_step_rhs(ctx, f, res, NULL, NULL, err);
}
int mo_euler_step(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                  mo_err* err) {
  clear(err);
  fieldv f = {g, get_set(ctx->M), coeffs, params};
  double* res = (double*)malloc(sizeof(double) * (size_t)g->nx * g->ny * f.s->n);
  int rc = residual(ctx, &f, res, err);
  if (rc == MO_OK) rc = euler_step(ctx, &f, res, err);
  free(res);
  return rc;
}

int mo_euler_step_rhs(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                      const double* rhs_coeffs, const double* rhs_params, mo_err* err) {
  clear(err);
  fieldv f = {g, get_set(ctx->M), coeffs, params};
  double* res = (double*)malloc(sizeof(double) * (size_t)g->nx * g->ny * f.s->n);
  int rc = residual(ctx, &f, res, err);
  if (rc == MO_OK) rc = euler_step_rhs(ctx, &f, res, rhs_coeffs, rhs_params, err);
  free(res);
  return rc;
}

/* total_mass, single_level.cpp:168-174 */
static double total_mass(const mo_grid* g, const iset* s, const double* c) {
  double mass = 0.0;
  for (int j = 0; j < g->ny; ++j)
    for (int i = 0; i < g->nx; ++i)
      mass += c[((size_t)j * g->nx + i) * s->n] * (g->dx[i] * g->dy[j]);
  return mass;
}
double mo_total_mass(const mo_grid* g, int M, const double* coeffs) {
  return total_mass(g, get_set(M), coeffs);
}
/* mass_correction, single_level.cpp:176-183 */
static int mass_correction(const mo_grid* g, const iset* s, double* c, double target,
                           mo_err* err) {
  const double current = total_mass(g, s, c);
  if (!(current > 0.0) || !isfinite(current))
    return fail(err, MO_NONPHYSICAL_STATE, "mass_correction: nonpositive total mass %f", current);
  const double f = target / current;
  const size_t total = (size_t)g->nx * g->ny * s->n;
  for (size_t q = 0; q < total; ++q) c[q] *= f;
  return MO_OK;
}
int mo_mass_correction(const mo_grid* g, int M, double* coeffs, double target, mo_err* err) {
  clear(err);
  return mass_correction(g, get_set(M), coeffs, target, err);
}

/* --------------------------------------------------------------- multigrid */
typedef struct grid_store {
  mo_grid g;
  double *dx, *dy, *xc, *yc;
} grid_store;

/* coarsen, multigrid.cpp:12-35 */
static void coarsen(const mo_grid* fine, grid_store* out) {
  out->g.nx = fine->nx / 2;
  out->g.ny = fine->ny / 2;
  out->g.Lx = fine->Lx;
  out->g.Ly = fine->Ly;
  out->dx = (double*)malloc(sizeof(double) * out->g.nx);
  out->xc = (double*)malloc(sizeof(double) * out->g.nx);
  out->dy = (double*)malloc(sizeof(double) * out->g.ny);
  out->yc = (double*)malloc(sizeof(double) * out->g.ny);
  double x = 0.0;
  for (int i = 0; i < out->g.nx; ++i) {
    out->dx[i] = fine->dx[2 * i] + fine->dx[2 * i + 1];
    out->xc[i] = x + 0.5 * out->dx[i];
    x += out->dx[i];
  }
  double y = 0.0;
  for (int j = 0; j < out->g.ny; ++j) {
    out->dy[j] = fine->dy[2 * j] + fine->dy[2 * j + 1];
    out->yc[j] = y + 0.5 * out->dy[j];
    y += out->dy[j];
  }
  out->g.dx = out->dx;
  out->g.dy = out->dy;
  out->g.xc = out->xc;
  out->g.yc = out->yc;
}
static int can_coarsen(const mo_grid* g) { /* multigrid.cpp:37-40 */
  return g->nx % 2 == 0 && g->ny % 2 == 0 && g->nx / 2 >= 8 && g->ny / 2 >= 8;
}

/* GridHierarchy::build, multigrid.cpp:44-65.  levels[0] = coarsest. */
typedef struct hierarchy {
  int n;
  grid_store lv[32];
} hierarchy;

static void free_hierarchy(hierarchy* h) {
  for (int k = 0; k < h->n; ++k) {
    free(h->lv[k].dx);
    free(h->lv[k].dy);
    free(h->lv[k].xc);
    free(h->lv[k].yc);
  }
  h->n = 0;
}
static int build_hierarchy(const mo_grid* finest, int levels, hierarchy* h, mo_err* err) {
  if (levels < 0) return fail(err, MO_CONFIG, "hierarchy: level count must be positive");
  /* store finest-first, reverse at the end */
  grid_store tmp[32];
  int n = 0;
  tmp[n].g = *finest;
  tmp[n].dx = tmp[n].dy = tmp[n].xc = tmp[n].yc = NULL;
  ++n;
  if (levels == 0) {
    while (can_coarsen(&tmp[n - 1].g) && n < 32) {
      coarsen(&tmp[n - 1].g, &tmp[n]);
      ++n;
    }
  } else {
    for (int k = 1; k < levels; ++k) {
      const mo_grid* top = &tmp[n - 1].g;
      if (top->nx % 2 != 0 || top->ny % 2 != 0 || !can_coarsen(top)) {
        h->n = n;
        for (int q = 0; q < n; ++q) h->lv[q] = tmp[q];
        h->lv[0].dx = h->lv[0].dy = h->lv[0].xc = h->lv[0].yc = NULL;
        free_hierarchy(h);
        if (top->nx % 2 != 0 || top->ny % 2 != 0)
          return fail(err, MO_CONFIG,
                      "hierarchy: %d levels need cell counts divisible by 2 at each split",
                      levels);
        return fail(err, MO_CONFIG,
                    "hierarchy: %d levels would make the coarsest grid smaller than 8 cells",
                    levels);
      }
      coarsen(top, &tmp[n]);
      ++n;
    }
  }
  h->n = n;
  for (int q = 0; q < n; ++q) h->lv[q] = tmp[n - 1 - q];
  return MO_OK;
}

/* restrict_solution, multigrid.cpp:67-112 */
static int restrict_solution(const iset* s, const fieldv* fine, const mo_grid* coarse,
                             double* cc, double* cp, mo_err* err) {
  const mo_grid* fg = fine->g;
  if (fg->nx != 2 * coarse->nx || fg->ny != 2 * coarse->ny)
    return fail(err, MO_CONFIG, "restrict_solution: grids are not a 2x2 refinement pair");
  const int n = s->n;
  double proj[1 << 12];
  for (int J = 0; J < coarse->ny; ++J)
    for (int I = 0; I < coarse->nx; ++I) {
      size_t child[4];
      double area[4];
      for (int c = 0; c < 4; ++c) {
        const int i = 2 * I + c % 2, j = 2 * J + c / 2;
        child[c] = (size_t)j * fg->nx + i;
        area[c] = fg->dx[i] * fg->dy[j];
      }
      double S = 0.0, mass = 0.0, energy = 0.0, mom[3] = {0, 0, 0};
      for (int c = 0; c < 4; ++c) {
        const double rho = fine->c[child[c] * n];
        const double* u = fine->p + child[c] * 4;
        const double theta = u[3];
        S += area[c];
        mass += rho * area[c];
        for (int d = 0; d < 3; ++d) mom[d] += rho * u[d] * area[c];
        const double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
        energy += rho * (3.0 * theta + usq) * area[c];
      }
      double basis[4];
      const double rho_H = mass / S;
      for (int d = 0; d < 3; ++d) basis[d] = mom[d] / mass;
      const double msq = basis[0] * basis[0] + basis[1] * basis[1] + basis[2] * basis[2];
      basis[3] = (energy / S - rho_H * msq) / (3.0 * rho_H);
      if (!(rho_H > 0.0) || !(basis[3] > 0.0))
        return fail(err, MO_NONPHYSICAL_STATE,
                    "restrict_solution: nonphysical coarse state at (%d,%d)", I, J);
      const size_t K = (size_t)J * coarse->nx + I;
      double* out = cc + K * n;
      double* op = cp + K * 4;
      memcpy(op, basis, sizeof(basis));
      for (int q = 0; q < n; ++q) out[q] = 0.0;
      for (int c = 0; c < 4; ++c) {
        TRY(project_to(s, fine->c + child[c] * n, fine->p + child[c] * 4, basis, proj, err));
        const double w = area[c] / S;
        for (int q = 0; q < n; ++q) out[q] += w * proj[q];
      }
      TRY(grad_normalize(s, out, op, err));
    }
  return MO_OK;
}
int mo_restrict_solution(int M, const mo_grid* fine, const double* fc, const double* fp,
                         const mo_grid* coarse, double* cc, double* cp, mo_err* err) {
  clear(err);
  fieldv f = {fine, get_set(M), (double*)fc, (double*)fp};
  return restrict_solution(f.s, &f, coarse, cc, cp, err);
}

/* restrict_residual, multigrid.cpp:114-142 */
static int restrict_residual(const iset* s, const mo_grid* fg, const double* arr_c,
                             const double* arr_p, const mo_grid* cg,
                             const double* coarse_params, double* out, mo_err* err) {
  if (fg->nx != 2 * cg->nx || fg->ny != 2 * cg->ny)
    return fail(err, MO_CONFIG, "restrict_residual: grids are not a 2x2 refinement pair");
  const int n = s->n;
  double proj[1 << 12];
  for (int J = 0; J < cg->ny; ++J)
    for (int I = 0; I < cg->nx; ++I) {
      const size_t K = (size_t)J * cg->nx + I;
      const double* basis = coarse_params + K * 4;
      double* r = out + K * n;
      for (int q = 0; q < n; ++q) r[q] = 0.0;
      double S = 0.0;
      for (int c = 0; c < 4; ++c) {
        const int i = 2 * I + c % 2, j = 2 * J + c / 2;
        S += fg->dx[i] * fg->dy[j];
      }
      for (int c = 0; c < 4; ++c) {
        const int i = 2 * I + c % 2, j = 2 * J + c / 2;
        const size_t k = (size_t)j * fg->nx + i;
        TRY(project_to(s, arr_c + k * n, arr_p + k * 4, basis, proj, err));
        const double w = (fg->dx[i] * fg->dy[j]) / S;
        for (int q = 0; q < n; ++q) r[q] += w * proj[q];
      }
    }
  return MO_OK;
}
int mo_restrict_residual(int M, const mo_grid* fine, const double* arr_c, const double* arr_p,
                         const double* fine_params, const mo_grid* coarse,
                         const double* coarse_params, double* out, mo_err* err) {
  clear(err);
  (void)fine_params;
  return restrict_residual(get_set(M), fine, arr_c, arr_p, coarse, coarse_params, out, err);
}

/* fas_correct, multigrid.cpp:144-164 */
static int fas_correct(const iset* s, fieldv* fine, const mo_grid* cg, const double* bc,
                       const double* bp, const double* ac, const double* ap, mo_err* err) {
  const mo_grid* fg = fine->g;
  if (fg->nx != 2 * cg->nx || fg->ny != 2 * cg->ny)
    return fail(err, MO_CONFIG, "fas_correct: grids are not a 2x2 refinement pair");
  const int n = s->n;
  double pa[1 << 12], pb[1 << 12];
  for (int j = 0; j < fg->ny; ++j)
    for (int i = 0; i < fg->nx; ++i) {
      const size_t k = (size_t)j * fg->nx + i;
      const size_t K = (size_t)(j / 2) * cg->nx + (i / 2);
      double* c = fine->c + k * n;
      double* p = fine->p + k * 4;
      TRY(project_to(s, ac + K * n, ap + K * 4, p, pa, err));
      TRY(project_to(s, bc + K * n, bp + K * 4, p, pb, err));
      for (int q = 0; q < n; ++q) c[q] += pa[q] - pb[q];
      const int rc = grad_normalize(s, c, p, err);
      if (rc == MO_NONPHYSICAL_STATE) {
        char what[256];
        snprintf(what, sizeof(what), "%s", err ? err->msg : "");
        return fail(err, MO_SOLVER_ERROR, "coarse-grid correction left cell (%d,%d) nonphysical: %s",
                    i, j, what);
      }
      if (rc != MO_OK) return rc;
    }
  return MO_OK;
}
int mo_fas_correct(int M, const mo_grid* fine, double* fc, double* fp, const mo_grid* coarse,
                   const double* bc, const double* bp, const double* ac, const double* ap,
                   mo_err* err) {
  clear(err);
  fieldv f = {fine, get_set(M), fc, fp};
  return fas_correct(f.s, &f, coarse, bc, bp, ac, ap, err);
}

/* residual_norm, multigrid.cpp:202-218 */
static double residual_norm(const iset* s, const mo_grid* g, const double* res,
                            const double* fp) {
  double total = 0.0;
  for (int j = 0; j < g->ny; ++j)
    for (int i = 0; i < g->nx; ++i) {
      const size_t k = (size_t)j * g->nx + i;
      const double theta = fp[k * 4 + 3];
      const double* r = res + k * s->n;
      double cell = 0.0;
      for (int q = 0; q < s->n; ++q) cell += s->fact[q] * pow(theta, s->deg[q]) * r[q] * r[q];
      total += cell * (g->dx[i] * g->dy[j]);
    }
  return sqrt(total / (g->Lx * g->Ly));
}
double mo_residual_norm(int M, const mo_grid* g, const double* res, const double* field_params) {
  return residual_norm(get_set(M), g, res, field_params);
}

/* residual_scale, multigrid.cpp:224-239 */
static double residual_scale(const mo_ctx* ctx, const fieldv* f) {
  double sc = 0.0;
  for (int j = 0; j < f->g->ny; ++j)
    for (int i = 0; i < f->g->nx; ++i) {
      const size_t k = CELL(f, i, j);
      const double rho = f->c[k * f->s->n];
      const double theta = f->p[k * 4 + 3];
      const double nu = collision_frequency(ctx, rho, theta);
      sc = smax(sc, rho * (ctx->cfl_c_bound * sqrt(theta) *
                               (1.0 / f->g->dx[i] + 1.0 / f->g->dy[j]) +
                           nu));
    }
  return sc;
}

/* nmg_cycle, multigrid.cpp:166-200.  rhs_c == NULL is the empty rhs. */
static int nmg_cycle(const mo_ctx* ctx, const hierarchy* h, int level, fieldv* f,
                     const double* rhs_c, const double* rhs_p, int s1, int s2, int s3,
                     int gamma, long long* work, mo_err* err) {
  if (level == 0) {
    for (int s = 0; s < s3; ++s) TRY(fast_sweep(ctx, f, rhs_c, rhs_p, NULL, work, err));
    return MO_OK;
  }
  for (int s = 0; s < s1; ++s) TRY(fast_sweep(ctx, f, rhs_c, rhs_p, NULL, work, err));
  const iset* st = f->s;
  const int n = st->n;
  const size_t fc = (size_t)f->g->nx * f->g->ny;
  const mo_grid* cg = &h->lv[level - 1].g;
  const size_t cc = (size_t)cg->nx * cg->ny;
  double* res = (double*)malloc(sizeof(double) * fc * n);
  double* defect = (double*)malloc(sizeof(double) * fc * n);
  double* coarse_c = (double*)malloc(sizeof(double) * cc * n);
  double* coarse_p = (double*)malloc(sizeof(double) * cc * 4);
  double* before_c = (double*)malloc(sizeof(double) * cc * n);
  double* before_p = (double*)malloc(sizeof(double) * cc * 4);
  double* crhs_c = (double*)malloc(sizeof(double) * cc * n);
  double* crhs_p = (double*)malloc(sizeof(double) * cc * 4);
  double* cres = (double*)malloc(sizeof(double) * cc * n);
  int rc = residual(ctx, f, res, err);
  for (size_t k = 0; rc == MO_OK && k < fc; ++k) {
    double* d = defect + k * n;
    const double* r = res + k * n;
    if (!rhs_c) {
      for (int q = 0; q < n; ++q) d[q] = -r[q];
    } else {
      rc = project_to(st, rhs_c + k * n, rhs_p + k * 4, f->p + k * 4, d, err);
      if (rc == MO_OK)
        for (int q = 0; q < n; ++q) d[q] = d[q] - r[q];
    }
  }
  if (rc == MO_OK) rc = restrict_solution(st, f, cg, coarse_c, coarse_p, err);
  if (rc == MO_OK) {
    memcpy(before_c, coarse_c, sizeof(double) * cc * n);
    memcpy(before_p, coarse_p, sizeof(double) * cc * 4);
    /* defect params = residual params = fine cell params */
    rc = restrict_residual(st, f->g, defect, f->p, cg, coarse_p, crhs_c, err);
    memcpy(crhs_p, coarse_p, sizeof(double) * cc * 4);
  }
  fieldv coarse = {cg, st, coarse_c, coarse_p};
  if (rc == MO_OK) rc = residual(ctx, &coarse, cres, err);
  if (rc == MO_OK)
    for (size_t q = 0; q < cc * n; ++q) crhs_c[q] += cres[q];
  for (int g = 0; rc == MO_OK && g < gamma; ++g)
    rc = nmg_cycle(ctx, h, level - 1, &coarse, crhs_c, crhs_p, s1, s2, s3, gamma, work, err);
  if (rc == MO_OK) rc = fas_correct(st, f, cg, before_c, before_p, coarse_c, coarse_p, err);
  for (int s = 0; rc == MO_OK && s < s2; ++s)
    rc = fast_sweep(ctx, f, rhs_c, rhs_p, NULL, work, err);
  free(res);
  free(defect);
  free(coarse_c);
  free(coarse_p);
  free(before_c);
  free(before_p);
  free(crhs_c);
  free(crhs_p);
  free(cres);
  return rc;
}
int mo_nmg_cycle(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params, int levels,
                 int s1, int s2, int s3, int gamma, long long* work, mo_err* err) {
  clear(err);
  hierarchy h;
  TRY(build_hierarchy(g, levels, &h, err));
  fieldv f = {g, get_set(ctx->M), coeffs, params};
  long long w = 0;
  const int rc = nmg_cycle(ctx, &h, h.n - 1, &f, NULL, NULL, s1, s2, s3, gamma, &w, err);
  if (work) *work = w;
  h.lv[h.n - 1].dx = h.lv[h.n - 1].dy = h.lv[h.n - 1].xc = h.lv[h.n - 1].yc = NULL;
  free_hierarchy(&h);
  return rc;
}

/* solve_steady, multigrid.cpp:243-320 */
int mo_solve_steady(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                    int solver, double tol, int max_iterations, int levels, int s1, int s2,
                    int s3, int gamma, mo_report* rep, mo_err* err) {
  clear(err);
  const iset* s = get_set(ctx->M);
  fieldv f = {g, s, coeffs, params};
  mo_report local;
  memset(&local, 0, sizeof(local));
  if (!rep) rep = &local;
  rep->converged = 0;
  rep->iterations = 0;
  rep->history_len = 0;
  rep->work = 0;
  const int cap = max_iterations > 0 ? max_iterations : (solver == 2 ? 200 : 100000);
  double* res = (double*)malloc(sizeof(double) * (size_t)g->nx * g->ny * s->n);
  int rc = residual(ctx, &f, res, err);
  if (rc != MO_OK) {
    free(res);
    return rc;
  }
  rep->r0_norm = residual_norm(s, g, res, params);
  if (rep->r0_norm <= 1e-12 * residual_scale(ctx, &f)) {
    rep->converged = 1;
    rep->final_norm = rep->r0_norm;
    rep->final_ratio = 0.0;
    free(res);
    return MO_OK;
  }
  hierarchy h;
  h.n = 0;
  if (solver == 2) {
    rc = build_hierarchy(g, levels, &h, err);
    if (rc != MO_OK) {
      free(res);
      return rc;
    }
  }
  const double target = total_mass(g, s, coeffs);
  long long work = 0;
  rc = MO_NONCONVERGENCE;
  for (int n = 1; n <= cap; ++n) {
    int step = MO_OK;
    if (solver == 0)
      step = euler_step(ctx, &f, res, err);
    else if (solver == 1)
      step = fast_sweep(ctx, &f, NULL, NULL, NULL, &work, err);
    else
      step = nmg_cycle(ctx, &h, h.n - 1, &f, NULL, NULL, s1, s2, s3, gamma, &work, err);
    if (step == MO_OK) step = mass_correction(g, s, coeffs, target, err);
    if (step == MO_OK) step = residual(ctx, &f, res, err);
    if (step != MO_OK) {
      rep->work = work;
      char what[256];
      snprintf(what, sizeof(what), "%s", err ? err->msg : "");
      if (step == MO_SOLVER_ERROR)
        rc = fail(err, MO_NONCONVERGENCE, "iteration step failed: %s", what);
      else if (step == MO_NONPHYSICAL_STATE)
        rc = fail(err, MO_NONCONVERGENCE, "iteration left the field nonphysical: %s", what);
      else
        rc = step; /* other Errors propagate unchanged */
      goto done;
    }
    rep->iterations = n;
    rep->final_norm = residual_norm(s, g, res, params);
    rep->final_ratio = rep->final_norm / rep->r0_norm;
    if (rep->history && rep->history_len < rep->history_cap)
      rep->history[rep->history_len] = rep->final_ratio;
    rep->history_len++;
    rep->work = work;
    if (!isfinite(rep->final_ratio) || rep->final_ratio > 1e6) {
      rc = fail(err, MO_NONCONVERGENCE, "residual diverged: ratio %f at iteration %d",
                rep->final_ratio, n);
      goto done;
    }
    if (rep->final_ratio <= tol) {
      rep->converged = 1;
      rc = MO_OK;
      goto done;
    }
  }
  rc = fail(err, MO_NONCONVERGENCE, "iteration cap %d reached at ratio %f", cap, rep->final_ratio);
done:
  if (h.n > 0) {
    h.lv[h.n - 1].dx = h.lv[h.n - 1].dy = h.lv[h.n - 1].xc = h.lv[h.n - 1].yc = NULL;
    free_hierarchy(&h);
  }
  free(res);
  return rc;
}
