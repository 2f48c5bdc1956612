// Thread-granular FP64 cell math (v3 of the hot path, moment orders 3..6).
//
// One thread evaluates one face flux (or one cell update) with straight-line
// code from gen/simplex_gen.cuh: every multi-index chain is a compile-time
// immediate offset, each thread's N-vectors live in shared memory interleaved
// with the other threads' (element k of thread t at buf[k*VS + t]) so every
// access is bank-conflict free, and nothing inside a face needs a barrier.
// A block of 64 threads works on a segment of 16 independent cells: warp 0
// evaluates their x faces (lanes 0-15 low side, 16-31 high side), warp 1
// their y faces; after one block barrier 16 threads combine the four fluxes
// with the collision term and update / normalise the cells.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "es_bgk.cuh"
#include "gen/simplex_gen.cuh"
#include "types.h"

namespace momg_gpu {

namespace tc {

constexpr int VS = 64;     // threads per block (vector interleave stride)
constexpr int SEG = 16;    // cells per block segment

__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ constexpr double rcp(int n) { return 1.0 / (double)n; }

struct P4 {
  double v[4];
};

template <bool CG>
__device__ __forceinline__ double ld(const double* p) {
  if (CG) return __ldcg(p);
  return __ldg(p);
}
template <bool CG>
__device__ __forceinline__ P4 ldp(const double* p) {
  P4 r;
  if (CG) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = b.x; r.v[3] = b.y;
  } else {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = b.x; r.v[3] = b.y;
  }
  return r;
}

// Copies a global record (N doubles, 16 B aligned) into a thread vector.
template <int M, bool CG>
__device__ __forceinline__ void load_vec(const double* __restrict__ src, double* __restrict__ v) {
  constexpr int N = Gen<M>::N;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    const double2 x = CG ? __ldcg(reinterpret_cast<const double2*>(src + k))
                         : __ldg(reinterpret_cast<const double2*>(src + k));
    v[k * VS] = x.x;
    v[(k + 1) * VS] = x.y;
  }
  if (N & 1) v[(N - 1) * VS] = ld<CG>(src + N - 1);
}

template <int M>
__device__ __forceinline__ void store_vec(const double* __restrict__ v, double* __restrict__ dst) {
  constexpr int N = Gen<M>::N;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) __stcg(reinterpret_cast<double2*>(dst + k), make_double2(v[k * VS], v[(k + 1) * VS]));
  if (N & 1) __stcg(dst + N - 1, v[(N - 1) * VS]);
}

// ---------------------------------------------------------- rep scalars
// rep_velocity (moment_rep.hpp:69-76), rep_temperature (:80-93),
// grad_defect (:97-110) on a thread vector; 2e_d at positions 4, 7, 9.
__device__ __forceinline__ double rep_u(const double* v, const P4& p, int axis) {
  return p.v[axis] + v[(1 + axis) * VS] / v[0];
}
__device__ __forceinline__ double rep_theta(const double* v, const P4& p) {
  const double rho = v[0];
  double trace = 0.0, fe2 = 0.0;
  const double c1 = v[1 * VS], c2 = v[2 * VS], c3 = v[3 * VS];
  trace += v[4 * VS];
  fe2 += c1 * c1;
  trace += v[7 * VS];
  fe2 += c2 * c2;
  trace += v[9 * VS];
  fe2 += c3 * c3;
  return p.v[3] + (2.0 * trace - fe2 / rho) / (3.0 * rho);
}
__device__ __forceinline__ double grad_defect(const double* v) {
  double defect = 0.0, trace = 0.0;
  defect = smax(defect, fabs(v[1 * VS]));
  trace += v[4 * VS];
  defect = smax(defect, fabs(v[2 * VS]));
  trace += v[7 * VS];
  defect = smax(defect, fabs(v[3 * VS]));
  trace += v[9 * VS];
  defect = smax(defect, fabs(trace));
  return defect / fabs(v[0]);
}

// ---------------------------------------------------------- projection
// project (projection.hpp:64-89) in place: the product over axes of the
// Toeplitz factors T_d = sum_n c_n down_d^n, c_n the coefficients of
// exp(a t + b t^2), a = -(to_d - from_d), b = -(to_theta - from_theta)/2,
// from the recurrence n c_n = a c_{n-1} + 2 b c_{n-2}.  An axis whose mean
// and the spread are both unchanged is the identity (projection.hpp:18, 36).
template <int M>
__device__ __forceinline__ void project(double* v, const P4& from, const P4& to) {
  const double b2 = -(to.v[3] - from.v[3]);  // 2b
  const bool ds = to.v[3] != from.v[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (!ds && to.v[d] == from.v[d]) continue;
    const double a = -(to.v[d] - from.v[d]);
    double c[M + 1];
    c[0] = 1.0;
    c[1] = a;
#pragma unroll
    for (int n = 2; n <= M; ++n) c[n] = fma(a, c[n - 1], b2 * c[n - 2]) * rcp(n);
    if (d == 0) Gen<M>::template pass0<VS>(v, c);
    if (d == 1) Gen<M>::template pass1<VS>(v, c);
    if (d == 2) Gen<M>::template pass2<VS>(v, c);
  }
}

// grad_normalize (projection.hpp:96-121) in place; prm updated.  Returns
// W_NONE or the failure kind.
template <int M>
__device__ __forceinline__ int grad_normalize(double* v, P4& prm, double* bad) {
  const double rel_tol = 1e-12;
  for (int iter = 0; iter < 30; ++iter) {
    const double rho = v[0];
    if (!isfinite(rho) || !(rho > 0.0)) {
      *bad = rho;
      return W_GRAD_RHO;
    }
    if (grad_defect(v) <= rel_tol) return W_NONE;
    P4 to;
    to.v[0] = rep_u(v, prm, 0);
    to.v[1] = rep_u(v, prm, 1);
    to.v[2] = rep_u(v, prm, 2);
    to.v[3] = rep_theta(v, prm);
    if (!isfinite(to.v[3]) || !(to.v[3] > 0.0)) {
      *bad = to.v[3];
      return W_GRAD_THETA;
    }
    if (!isfinite(to.v[0]) || !isfinite(to.v[1]) || !isfinite(to.v[2])) return W_GRAD_U;
    project<M>(v, prm, to);
    prm = to;
  }
  if (grad_defect(v) > rel_tol) return W_GRAD_CAP;
  return W_NONE;
}

// ------------------------------------------------------ half-range kernels
// Folded half-flux kernels (flux.cpp:58-73 hoisted, halfspace.hpp:18-57):
//   Ku[m][p] = rs^(p-m)/p! (u_n P+(m,p) + rs P+(m+1,p) + rs m P+(m-1,p)),
//   Kl[m][p] = same with P- = m! delta - P+.
// The pairing table follows the reference recurrence column by column.
// The transcendental part of the base row (one erfc, one exp per face):
// a = -u_n / rs, g = e^{-a^2/2}/sqrt(2 pi), e0 = erfc(a/sqrt 2)/2.
struct HalfBase {
  double a, g, e0, irs;
};
__device__ __forceinline__ HalfBase half_base(double un, double rs) {
  HalfBase h;
  h.irs = 1.0 / rs;
  h.a = -un * h.irs;
  h.g = exp(-h.a * h.a * 0.5) * 0.3989422804014327;
  h.e0 = 0.5 * erfc(h.a * 0.7071067811865476);
  return h;
}
template <int M>
__device__ __forceinline__ void half_kernels_b(double un, double rs, const HalfBase& hb,
                                               double (&Ku)[M + 1][M + 1], double (&Kl)[M + 1][M + 1]);
template <int M>
__device__ __forceinline__ void half_kernels(double un, double rs, double (&Ku)[M + 1][M + 1],
                                             double (&Kl)[M + 1][M + 1]) {
  half_kernels_b<M>(un, rs, half_base(un, rs), Ku, Kl);
}
template <int M>
__device__ __forceinline__ void half_kernels_b(double un, double rs, const HalfBase& hb,
                                               double (&Ku)[M + 1][M + 1], double (&Kl)[M + 1][M + 1]) {
  constexpr int P = M + 1;
  const double a = hb.a;
  const double g = hb.g;
  double he[P + 1];
  he[0] = 1.0;
  he[1] = a;
#pragma unroll
  for (int k = 1; k + 1 <= P; ++k) he[k + 1] = a * he[k] - (double)k * he[k - 1];
  const double irs = hb.irs;
  double prev[P + 1];  // column p-1 of the pairing table
  double fp = 1.0, rsp = 1.0;  // p!, rs^p
  // 1/p! as compile-time constants (a multiplication instead of a division
  // on the flux path; differs from rsp / p! by at most one rounding)
  constexpr double kInvFact[9] = {1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0, 1.0 / 720.0, 1.0 / 5040.0,
                                  1.0 / 40320.0};
  static_assert(M <= 8, "kInvFact covers M <= 8");
#pragma unroll
  for (int p = 0; p <= M; ++p) {
    double col[P + 1];
    col[0] = p == 0 ? hb.e0 : he[p - 1] * g;
#pragma unroll
    for (int m = 0; m + 1 <= P; ++m) {
      const double t = he[m] * he[p] * g;
      col[m + 1] = p > 0 ? fma((double)p, prev[m], t) : t;
    }
    if (p > 0) {
      fp *= (double)p;
      rsp *= rs;
    }
    double scale = rsp * kInvFact[p];
#pragma unroll
    for (int m = 0; m <= M; ++m) {
      const double lo_m = (m == p ? fp : 0.0) - col[m];
      const double lo_p1 = (m + 1 == p ? fp : 0.0) - col[m + 1];
      double ku = fma(un, col[m], rs * col[m + 1]);
      double kl = fma(un, lo_m, rs * lo_p1);
      if (m > 0) {
        const double lo_m1 = (m - 1 == p ? fp : 0.0) - col[m - 1];
        ku = fma(rs * (double)m, col[m - 1], ku);
        kl = fma(rs * (double)m, lo_m1, kl);
      }
      Ku[m][p] = scale * ku;
      Kl[m][p] = scale * kl;
      scale *= irs;
    }
#pragma unroll
    for (int m = 0; m <= P; ++m) prev[m] = col[m];
  }
}

template <int M, int AXIS>
__device__ __forceinline__ void half_sum(double* L, const double* R, const double (&Ku)[M + 1][M + 1],
                                         const double (&Kl)[M + 1][M + 1]) {
  if (AXIS == 0) Gen<M>::template half_sum0<VS>(L, R, Ku, Kl);
  else Gen<M>::template half_sum1<VS>(L, R, Ku, Kl);
}
template <int M, int AXIS>
__device__ __forceinline__ void half_one(double* L, const double (&K)[M + 1][M + 1]) {
  if (AXIS == 0) Gen<M>::template half_one0<VS>(L, K);
  else Gen<M>::template half_one1<VS>(L, K);
}
template <int M, int AXIS>
__device__ __forceinline__ void full_flux(const double* s, double* o, double un, double th) {
  if (AXIS == 0) Gen<M>::template full_flux0<VS>(s, o, un, th);
  else Gen<M>::template full_flux1<VS>(s, o, un, th);
}

// --------------------------------------------------------------- faces
// Reconstructed face state (face_state + safe_face_state, spatial.cpp:34-80)
// of the cell at global record `c` (position m along the axis, last index
// `last`) on its side `off` (+-dx/2), slope from records lo/hi over distance
// h; written into thread vector v, params returned.
template <int M, int ORDER, bool CG>
__device__ __forceinline__ P4 face_state(const DevField& f, size_t cell, size_t lo, size_t hi,
                                         int m, int last, double h, double off, double* v) {
  constexpr int NP = (Gen<M>::N + 3) & ~3;
  const P4 cp = ldp<CG>(f.p + cell * 4);
  if (ORDER == 1 || m == 0 || m == last) {
    load_vec<M, CG>(f.c + cell * NP, v);
    return cp;
  }
  const P4 pl = ldp<CG>(f.p + lo * 4), ph = ldp<CG>(f.p + hi * 4);
  P4 w;
#pragma unroll
  for (int q = 0; q < 4; ++q) w.v[q] = cp.v[q] + off * ((ph.v[q] - pl.v[q]) / h);
  if (!(w.v[3] > 0.0)) {  // NonphysicalReconstruction -> first order
    load_vec<M, CG>(f.c + cell * NP, v);
    return cp;
  }
  const double rh = 1.0 / h;
  const double* sc = f.c + cell * NP;
  const double* sl = f.c + lo * NP;
  const double* sh = f.c + hi * NP;
#pragma unroll
  for (int k = 0; k < Gen<M>::N; ++k) v[k * VS] = fma(off, (ld<CG>(sh + k) - ld<CG>(sl + k)) * rh, ld<CG>(sc + k));
  return w;
}

// Flux through face (AXIS, high) of cell (i, j), projected into the cell
// basis cp, left in thread vector L (U is scratch).  The `face` lambda of
// cell_residual (spatial.cpp:106-124): wall_flux (flux.cpp:105-130) on
// boundary faces, face_flux (flux.cpp:77-97) with the lo/hi roles of
// spatial.cpp:114-121 inside.
template <int M, int ORDER, int AXIS, bool CG>
__device__ __forceinline__ int face(const DevField& f, const DevCtx& ctx, int i, int j, bool high,
                                    double* L, double* U) {
  constexpr int NP = (Gen<M>::N + 3) & ~3;
  const int n = AXIS == 0 ? f.nx : f.ny;
  const int pos = AXIS == 0 ? i : j;
  const size_t cell = (size_t)j * f.nx + i;
  const size_t stride = AXIS == 0 ? 1 : (size_t)f.nx;
  const P4 cp = ldp<CG>(f.p + cell * 4);
  const bool at_wall = high ? pos == n - 1 : pos == 0;
  if (at_wall) {
    const int w = AXIS == 0 ? (high ? 1 : 0) : (high ? 3 : 2);
    P4 wb;
    wb.v[0] = wb.v[1] = wb.v[2] = 0.0;
    wb.v[AXIS == 0 ? 1 : 0] = ctx.wall_speed[w];
    wb.v[3] = ctx.wall_theta[w];
    if (!(wb.v[3] > 0.0)) return W_PROJ_SPREAD;
    load_vec<M, CG>(f.c + cell * NP, L);
    project<M>(L, cp, wb);
    const double rs = sqrt(wb.v[3]);
    double Ku[M + 1][M + 1], Kl[M + 1][M + 1];
    half_kernels<M>(0.0, rs, Ku, Kl);
    if (high) half_one<M, AXIS>(L, Ku);
    else half_one<M, AXIS>(L, Kl);
    const double in0 = high ? Kl[0][0] : Ku[0][0];
    if (in0 == 0.0) return W_WALL_DEGEN;
    const double wall_rho = -L[0] / in0;
    if (!(wall_rho > 0.0)) return W_WALL_RHO;
    // incoming unit-wall half flux rs^p/p! K(0,p) at beta = p e_axis
#pragma unroll
    for (int p = 1; p <= M; ++p) {
      const int k = AXIS == 0 ? flat3(p, 0, 0) : flat3(0, p, 0);
      L[k * VS] = fma(wall_rho, high ? Kl[0][p] : Ku[0][p], L[k * VS]);
    }
    L[0] = 0.0;
    project<M>(L, wb, cp);
    return W_NONE;
  }
  const double* xc = AXIS == 0 ? f.xc : f.yc;
  const double* dd = AXIS == 0 ? f.dx : f.dy;
  // lower cell (position pl) on its high side, upper cell (pu) on its low side
  const int pl = high ? pos : pos - 1;
  const int pu = pl + 1;
  const size_t cl = high ? cell : cell - stride;
  const size_t cu = cl + stride;
  const double hl = (ORDER == 2 && pl > 0 && pl < n - 1) ? xc[pl + 1] - xc[pl - 1] : 1.0;
  const double hu = (ORDER == 2 && pu > 0 && pu < n - 1) ? xc[pu + 1] - xc[pu - 1] : 1.0;
  const P4 lp = face_state<M, ORDER, CG>(f, cl, pl > 0 ? cl - stride : cl, cu, pl, n - 1, hl, 0.5 * dd[pl], L);
  const P4 rp = face_state<M, ORDER, CG>(f, cu, cl, pu < n - 1 ? cu + stride : cu, pu, n - 1, hu, -0.5 * dd[pu], U);
  const double ul = rep_u(L, lp, AXIS), ur = rep_u(U, rp, AXIS);
  const double cl_ = ctx.c_bound * sqrt(rep_theta(L, lp));
  const double cr_ = ctx.c_bound * sqrt(rep_theta(U, rp));
  const double lminus = smin(ul - cl_, ur - cr_);
  const double lplus = smax(ul + cl_, ur + cr_);
  P4 fp;
#pragma unroll
  for (int q = 0; q < 4; ++q) fp.v[q] = 0.5 * (lp.v[q] + rp.v[q]);
  if (!(fp.v[3] > 0.0)) return W_PROJ_SPREAD;
  if (lminus >= 0.0) {
    project<M>(L, lp, fp);
    full_flux<M, AXIS>(L, U, fp.v[AXIS], fp.v[3]);
    project<M>(U, fp, cp);
#pragma unroll
    for (int k = 0; k < Gen<M>::N; ++k) L[k * VS] = U[k * VS];
    return W_NONE;
  }
  if (lplus <= 0.0) {
    project<M>(U, rp, fp);
    full_flux<M, AXIS>(U, L, fp.v[AXIS], fp.v[3]);
    project<M>(L, fp, cp);
    return W_NONE;
  }
  project<M>(L, lp, fp);
  project<M>(U, rp, fp);
  double Ku[M + 1][M + 1], Kl[M + 1][M + 1];
  half_kernels<M>(fp.v[AXIS], sqrt(fp.v[3]), Ku, Kl);
  half_sum<M, AXIS>(L, U, Ku, Kl);
  project<M>(L, fp, cp);
  return W_NONE;
}

// collision_coeffs scalars (collision.hpp:120-127, extract_macro
// moment_rep.hpp:116-146): nu and the Shakhov heat flux q.
template <int M>
__device__ __forceinline__ int collision_scalars(const double* S, const P4& cp, const DevCtx& ctx,
                                                 double* nu, double* q) {
  const double rho = S[0];
  if (!(rho > 0.0)) return W_MACRO_RHO;
  if (!(cp.v[3] > 0.0)) return W_MACRO_RHO;
  q[0] = q[1] = q[2] = 0.0;
  if (ctx.collision == 1) {  // ES-BGK: SPD check here, the Gaussian in assemble (min eig -> q[0])
    const int w = es::check<VS>(S, cp.v[3], ctx.prandtl, &q[0]);
    if (w) return w;
  }
  *nu = ctx.nu_coef * rho * pow(cp.v[3], ctx.nu_exp);
  if (ctx.collision == 2) {
    q[0] = 2.0 * S[flat3(3, 0, 0) * VS] + S[flat3(3, 0, 0) * VS] + S[flat3(1, 2, 0) * VS] + S[flat3(1, 0, 2) * VS];
    q[1] = 2.0 * S[flat3(0, 3, 0) * VS] + S[flat3(2, 1, 0) * VS] + S[flat3(0, 3, 0) * VS] + S[flat3(0, 1, 2) * VS];
    q[2] = 2.0 * S[flat3(0, 0, 3) * VS] + S[flat3(2, 0, 1) * VS] + S[flat3(0, 2, 1) * VS] + S[flat3(0, 0, 3) * VS];
  }
  return W_NONE;
}

// Writes into D (thread vector): D_k = Q_k - (Fxp-Fxm)/dx - (Fyp-Fym)/dy
// (cell_residual assembly, spatial.cpp:127-132) [- rhs_k], Q = nu (eq - S).
// ES-BGK (es, basis temperature theta): the Gaussian equilibrium is first
// written into D (es::fill) and read back element by element.
template <int M>
__device__ __forceinline__ void assemble(const double* S, double nu, const double* q, int shakhov,
                                         double shw, const double* Fxm, const double* Fxp,
                                         const double* Fym, const double* Fyp, double dx, double dy,
                                         const double* rhs, double* D, int es = 0, double theta = 1.0,
                                         double prandtl = 1.0) {
  if (es) es::fill<M, VS>(S, theta, prandtl, D);
  double eq[Gen<M>::N];
#pragma unroll
  for (int k = 0; k < Gen<M>::N; ++k) eq[k] = 0.0;
  eq[0] = S[0];
  if (shakhov) {
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int dd = 0; dd < 3; ++dd)
        eq[flat3((dd == 0 ? 2 : 0) + (d == 0), (dd == 1 ? 2 : 0) + (d == 1), (dd == 2 ? 2 : 0) + (d == 2))] =
            shw * q[d];
  }
#pragma unroll
  for (int k = 0; k < Gen<M>::N; ++k) {
    double r = nu * ((es ? D[k * VS] : eq[k]) - S[k * VS]);
    r -= (Fxp[k * VS] - Fxm[k * VS]) / dx;
    r -= (Fyp[k * VS] - Fym[k * VS]) / dy;
    if (rhs) r -= rhs[k * VS];
    D[k * VS] = r;
  }
}

}  // namespace tc
}  // namespace momg_gpu
