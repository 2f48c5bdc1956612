// Transfer operators of the FAS V-cycle with warp-cooperative record staging
// (moment orders M <= 5: N <= 56 coefficients, one record <= 448 B):
//
//   xf_restrict_sol  restrict_solution  multigrid.cpp:67-112   thread per coarse cell
//   xf_restrict_res  restrict_residual  multigrid.cpp:114-142  thread per coarse cell
//   xf_fas           fas_correct        multigrid.cpp:144-164  thread per fine cell
//
// These kernels are HBM-bound (a few thousand flops per 448-byte record), and
// the shared-memory vectors of the thread-per-face kernels (kernels_v3.cuh)
// cap them at ~30% of the HBM roofline (occupancy and LDS/STS traffic).  Here
// a thread keeps its cell's whole record in REGISTERS: it loads it with 16-byte
// streaming loads (all of them in flight together), the projections are the
// generated straight-line Toeplitz passes with stride 1 on a register array
// (compile-time offsets), the 2x2 averages and the FAS difference accumulate in
// registers, and grad_normalize runs in registers; no shared memory at all.
// Operation order and branches are the reference's (see each kernel).
#pragma once

#include "gen/simplex_gen.cuh"
#include "thread_cell.cuh"
#include "types.h"

namespace momg_gpu {
namespace xf {

constexpr int XT = 128;  // threads per block (4 warps)

using tc::P4;

template <int M>
struct Dim {
  static constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
};

// a record (N doubles, 16-byte aligned) into / out of a register array
template <int M, bool STREAM = true>
__device__ __forceinline__ void load_rec(const double* __restrict__ p, double (&v)[Gen<M>::N]) {
  constexpr int N = Gen<M>::N;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    const double2 x = STREAM ? __ldcs(reinterpret_cast<const double2*>(p + k))
                             : __ldcg(reinterpret_cast<const double2*>(p + k));
    v[k] = x.x;
    v[k + 1] = x.y;
  }
  if (N & 1) v[N - 1] = STREAM ? __ldcs(p + N - 1) : __ldcg(p + N - 1);
}
template <int M>
__device__ __forceinline__ void store_rec(double* __restrict__ p, const double (&v)[Gen<M>::N]) {
  constexpr int N = Gen<M>::N;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) __stcs(reinterpret_cast<double2*>(p + k), make_double2(v[k], v[k + 1]));
  if (N & 1) __stcs(p + N - 1, v[N - 1]);
}

// project (projection.hpp:64-89) of a stride-1 row in place.  SKIP = false
// runs every axis pass (an identity pass when the axis' shift is zero: the
// same values), which keeps the code straight-line for the large orders.
template <int M, bool SKIP = true>
__device__ __forceinline__ void project_row(double* v, const P4& from, const P4& to) {
  const double b2 = -(to.v[3] - from.v[3]);
  const bool ds = to.v[3] != from.v[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (SKIP && !ds && to.v[d] == from.v[d]) continue;
    const double a = -(to.v[d] - from.v[d]);
    double c[M + 1];
    c[0] = 1.0;
    c[1] = a;
#pragma unroll
    for (int n = 2; n <= M; ++n) c[n] = fma(a, c[n - 1], b2 * c[n - 2]) * tc::rcp(n);
    if (d == 0) Gen<M>::template pass0<1>(v, c);
    if (d == 1) Gen<M>::template pass1<1>(v, c);
    if (d == 2) Gen<M>::template pass2<1>(v, c);
  }
}

// grad_normalize (projection.hpp:96-121) of a stride-1 row; rep_velocity /
// rep_temperature / grad_defect (moment_rep.hpp:69-110), 2e_d at 4, 7, 9
template <int M, bool SKIP = true>
__device__ __forceinline__ int normalize_row(double* v, P4& prm, double* bad) {
  for (int iter = 0; iter < 30; ++iter) {
    const double rho = v[0];
    if (!isfinite(rho) || !(rho > 0.0)) {
      *bad = rho;
      return W_GRAD_RHO;
    }
    double defect = 0.0, trace = 0.0;
    defect = tc::smax(defect, fabs(v[1]));
    trace += v[4];
    defect = tc::smax(defect, fabs(v[2]));
    trace += v[7];
    defect = tc::smax(defect, fabs(v[3]));
    trace += v[9];
    defect = tc::smax(defect, fabs(trace));
    if (defect / fabs(v[0]) <= 1e-12) return W_NONE;
    P4 to;
#pragma unroll
    for (int d = 0; d < 3; ++d) to.v[d] = prm.v[d] + v[1 + d] / rho;
    double tr = 0.0, fe2 = 0.0;
    tr += v[4];
    fe2 += v[1] * v[1];
    tr += v[7];
    fe2 += v[2] * v[2];
    tr += v[9];
    fe2 += v[3] * v[3];
    to.v[3] = prm.v[3] + (2.0 * tr - fe2 / rho) / (3.0 * rho);
    if (!isfinite(to.v[3]) || !(to.v[3] > 0.0)) {
      *bad = to.v[3];
      return W_GRAD_THETA;
    }
    if (!isfinite(to.v[0]) || !isfinite(to.v[1]) || !isfinite(to.v[2])) return W_GRAD_U;
    project_row<M, SKIP>(v, prm, to);
    prm = to;
  }
  double defect = 0.0, trace = 0.0;
  defect = tc::smax(defect, fabs(v[1]));
  trace += v[4];
  defect = tc::smax(defect, fabs(v[2]));
  trace += v[7];
  defect = tc::smax(defect, fabs(v[3]));
  trace += v[9];
  defect = tc::smax(defect, fabs(trace));
  return defect / fabs(v[0]) > 1e-12 ? W_GRAD_CAP : W_NONE;
}

__device__ __forceinline__ void store_params(double* p, const P4& v) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(v.v[0], v.v[1]));
  __stcs(reinterpret_cast<double2*>(p) + 1, make_double2(v.v[2], v.v[3]));
}

// restrict_solution (multigrid.cpp:67-112): the children's mass, momentum and
// energy fix the coarse basis; the children are projected into it,
// area-averaged and Grad-normalized.  Thread per coarse cell.
template <int M>
__global__ void __launch_bounds__(XT) xf_restrict_sol(DevField fine, DevField coarse, DevErr* err) {
  using D = Dim<M>;
  const int cells = coarse.nx * coarse.ny;
  for (int K = blockIdx.x * XT + threadIdx.x; K < cells; K += gridDim.x * XT) {
    if (tc::err_on(err)) return;
    const int I = K % coarse.nx, J = K / coarse.nx;
    size_t child[4];
    double area[4];
    P4 cpar[4];
    double S = 0.0, mass = 0.0, energy = 0.0, mom[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      child[c] = (size_t)j * fine.nx + i;
      area[c] = fine.dx[i] * fine.dy[j];
      cpar[c] = tc::ldp<true>(fine.p + child[c] * 4);
      const double rho = __ldcg(fine.c + child[c] * D::NP);
      const double* u = cpar[c].v;
      S += area[c];
      mass += rho * area[c];
#pragma unroll
      for (int q = 0; q < 3; ++q) mom[q] += rho * u[q] * area[c];
      const double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
      energy += rho * (3.0 * u[3] + usq) * area[c];
    }
    P4 basis;
    const double rho_H = mass / S;
#pragma unroll
    for (int q = 0; q < 3; ++q) basis.v[q] = mom[q] / mass;
    const double msq = basis.v[0] * basis.v[0] + basis.v[1] * basis.v[1] + basis.v[2] * basis.v[2];
    basis.v[3] = (energy / S - rho_H * msq) / (3.0 * rho_H);
    if (!(rho_H > 0.0) || !(basis.v[3] > 0.0)) {
      tc::raise(err, E_NONPHYSICAL, W_RESTRICT, I, J, rho_H);
      return;
    }
    double acc[D::N], v[D::N];
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      load_rec<M>(fine.c + child[c] * D::NP, v);
      project_row<M>(v, cpar[c], basis);
      const double wgt = area[c] / S;
#pragma unroll
      for (int k = 0; k < D::N; ++k) acc[k] = c == 0 ? wgt * v[k] : fma(wgt, v[k], acc[k]);
    }
    P4 prm = basis;
    double bad = 0.0;
    const int w = normalize_row<M>(acc, prm, &bad);
    if (w) {
      tc::raise(err, tc::code_for(w), w, I, J, bad);
      return;
    }
    store_rec<M>(coarse.c + (size_t)K * D::NP, acc);
    store_params(coarse.p + (size_t)K * 4, prm);
  }
}

// restrict_residual (multigrid.cpp:114-142): each child's array carries its
// own basis and is projected into the coarse cell's basis, area-averaged.
template <int M>
__global__ void __launch_bounds__(XT) xf_restrict_res(DevField arrays, DevField coarse, DevField out, DevErr* err) {
  using D = Dim<M>;
  const int cells = coarse.nx * coarse.ny;
  for (int K = blockIdx.x * XT + threadIdx.x; K < cells; K += gridDim.x * XT) {
    if (tc::err_on(err)) return;
    const int I = K % coarse.nx, J = K / coarse.nx;
    const P4 basis = tc::ldp<true>(coarse.p + (size_t)K * 4);
    if (!(basis.v[3] > 0.0)) {
      tc::raise(err, E_NONPHYSICAL, W_PROJ_SPREAD, I, J, basis.v[3]);
      return;
    }
    double S = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) S += arrays.dx[2 * I + c % 2] * arrays.dy[2 * J + c / 2];
    double acc[D::N], v[D::N];
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      const size_t ch = (size_t)j * arrays.nx + i;
      load_rec<M>(arrays.c + ch * D::NP, v);
      project_row<M>(v, tc::ldp<true>(arrays.p + ch * 4), basis);
      const double wgt = (arrays.dx[i] * arrays.dy[j]) / S;
#pragma unroll
      for (int k = 0; k < D::N; ++k) acc[k] = c == 0 ? wgt * v[k] : fma(wgt, v[k], acc[k]);
    }
    store_rec<M>(out.c + (size_t)K * D::NP, acc);
    store_params(out.p + (size_t)K * 4, basis);
  }
}

// fas_correct (multigrid.cpp:144-164): f += project(after -> f basis) -
// project(before -> f basis), then grad_normalize; nonphysical -> SolverError.
// Thread per fine cell.
template <int M>
__global__ void __launch_bounds__(XT) xf_fas(DevField fine, DevField before, DevField after, DevErr* err) {
  using D = Dim<M>;
  const int cells = fine.nx * fine.ny;
  for (int k = blockIdx.x * XT + threadIdx.x; k < cells; k += gridDim.x * XT) {
    if (tc::err_on(err)) return;
    const int i = k % fine.nx, j = k / fine.nx;
    const size_t Kc = (size_t)(j / 2) * before.nx + (i / 2);
    const P4 cp = tc::ldp<true>(fine.p + (size_t)k * 4);
    if (!(cp.v[3] > 0.0)) {
      tc::raise(err, E_NONPHYSICAL, W_PROJ_SPREAD, i, j, cp.v[3]);
      return;
    }
    double a[D::N], v[D::N];
    // each coarse record serves 4 fine cells: keep it in L2
    load_rec<M, false>(after.c + Kc * D::NP, a);
    project_row<M>(a, tc::ldp<true>(after.p + Kc * 4), cp);
    load_rec<M, false>(before.c + Kc * D::NP, v);
    project_row<M>(v, tc::ldp<true>(before.p + Kc * 4), cp);
#pragma unroll
    for (int q = 0; q < D::N; ++q) a[q] = a[q] - v[q];
    load_rec<M>(fine.c + (size_t)k * D::NP, v);
#pragma unroll
    for (int q = 0; q < D::N; ++q) v[q] = v[q] + a[q];
    P4 prm = cp;
    double bad = 0.0;
    int w = normalize_row<M>(v, prm, &bad);
    if (w) {
      if (tc::code_for(w) == E_NONPHYSICAL) w = W_FAS;
      tc::raise(err, tc::code_for(w), w, i, j, bad);
      return;
    }
    store_rec<M>(fine.c + (size_t)k * D::NP, v);
    store_params(fine.p + (size_t)k * 4, prm);
  }
}

}  // namespace xf
}  // namespace momg_gpu
