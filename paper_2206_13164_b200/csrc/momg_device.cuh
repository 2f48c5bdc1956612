// Warp-cooperative FP64 device primitives of the moment method (sm_100a).
//
// One warp owns one cell (or one face) at a time.  Every N-vector of Hermite
// coefficients lives in a per-warp shared-memory buffer; lane l owns the
// coefficients k = l, l+32, ... (T = ceil(N/32) "items").  Cross-coefficient
// reads (mean-shift chains, the spread Laplacian, the half-range pairing
// along the normal) are shared-memory loads; one __syncwarp separates
// consecutive passes.  Multi-index arithmetic is closed-form: the graded-lex
// position of (a1,a2,a3) is tet(D) + tri(a2+a3) + a3 with D = a1+a2+a3
// (multi_index.hpp:31-40); each block keeps the packed multi-index of every
// position in shared memory (`alpha`).
//
// Primitives take and return shared-memory vectors (no register arrays
// cross a call), so they can stay out of line: this bounds code size and
// register pressure for M up to 8 (N = 165).
//
// Numerics follow the reference's formulas and summation order; FMA
// contraction and reciprocal multiplications make results differ from the
// CPU reference by a few ulp per operation (parity bar: 1e-10 per sweep,
// north_star).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "types.h"

namespace momg_gpu {

constexpr unsigned FULL = 0xffffffffu;

template <int M>
struct Cfg {
  static constexpr int N = tet(M + 1);          // IndexSet::count
  static constexpr int NP = (N + 3) & ~3;       // row pitch in doubles (32 B sectors)
  static constexpr int T = (N + 31) / 32;       // items per lane
  static constexpr int KT = (M + 1) * (M + 1);  // half-flux kernel table size
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ constexpr double rcp_int(int n) { return 1.0 / (double)n; }

// std::min / std::max semantics (NaN handling as the reference).
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// Packed multi-index table of one block: alpha[k] = a1 | a2 << 8 | a3 << 16.
template <int M>
__device__ __forceinline__ void build_alpha(uint32_t* alpha) {
  for (int k = threadIdx.x; k < Cfg<M>::N; k += blockDim.x) {
    int D = 0;
    while (tet(D + 1) <= k) ++D;
    const int rem = k - tet(D);
    int r = 0;
    while (tri(r + 1) <= rem) ++r;
    const int a3 = rem - tri(r), a2 = r - a3, a1 = D - r;
    alpha[k] = (uint32_t)a1 | ((uint32_t)a2 << 8) | ((uint32_t)a3 << 16);
  }
}

template <int M>
struct Items {
  static constexpr int N = Cfg<M>::N, T = Cfg<M>::T;
  uint32_t pk[T];
  __device__ __forceinline__ explicit Items(const uint32_t* alpha) {
    const int lane = lane_id();
#pragma unroll
    for (int t = 0; t < T; ++t) pk[t] = (lane + 32 * t < N) ? alpha[lane + 32 * t] : 0u;
  }
  __device__ __forceinline__ bool v(int t) const { return lane_id() + 32 * t < N; }
  __device__ __forceinline__ int a1(int t) const { return pk[t] & 0xff; }
  __device__ __forceinline__ int a2(int t) const { return (pk[t] >> 8) & 0xff; }
  __device__ __forceinline__ int a3(int t) const { return pk[t] >> 16; }
  __device__ __forceinline__ int ax(int t, int d) const { return (pk[t] >> (8 * d)) & 0xff; }
  __device__ __forceinline__ int deg(int t) const { return a1(t) + a2(t) + a3(t); }
};

struct P4 {
  double v[4];
};

// ------------------------------------------------------------- projection
// Moment-preserving change of basis (projection.hpp:16-73): mean shifts along
// x, y, z (skipped when delta == 0, projection.hpp:18), then the spread shift
// (skipped when delta == 0, :36; floor(M/2) passes of the sum_d down^2
// operator).  Input in smem `x` (basis `from`, clobbered), `y` scratch; the
// result is written to `dst` (may alias x or y) and the warp is synced on
// return.  Returns false when the target spread is not positive
// (NonphysicalState, projection.hpp:68-69); dst is then not written.
template <int M>
__device__ __noinline__ bool project_smem(const uint32_t* alpha, double* x, double* y, P4 from,
                                          P4 to, double* dst) {
  constexpr int T = Cfg<M>::T;
  if (!(to.v[3] > 0.0)) return false;
  const Items<M> it(alpha);
  const int lane = lane_id();
  double out[T];
#pragma unroll
  for (int t = 0; t < T; ++t) out[t] = it.v(t) ? x[lane + 32 * t] : 0.0;
  double* cur = x;
  double* nxt = y;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double delta = to.v[d] - from.v[d];
    if (delta == 0.0) continue;
    const double nd = -delta;
    double w[M + 1];
    w[0] = 1.0;
#pragma unroll
    for (int n = 1; n <= M; ++n) w[n] = w[n - 1] * (nd * rcp_int(n));
#pragma unroll
    for (int t = 0; t < T; ++t) {
      if (!it.v(t)) continue;
      const int ad = it.ax(t, d);
      const int a1 = it.a1(t), a2 = it.a2(t), a3 = it.a3(t);
      double acc = out[t];
#pragma unroll
      for (int n = 1; n <= M; ++n)
        if (n <= ad)
          acc = fma(w[n], cur[flat3(a1 - (d == 0 ? n : 0), a2 - (d == 1 ? n : 0),
                                    a3 - (d == 2 ? n : 0))],
                    acc);
      out[t] = acc;
    }
#pragma unroll
    for (int t = 0; t < T; ++t)
      if (it.v(t)) nxt[lane + 32 * t] = out[t];
    __syncwarp();
    double* s = cur;
    cur = nxt;
    nxt = s;
  }
  const double ds = to.v[3] - from.v[3];
  if (ds != 0.0) {
    const double nd = -ds;
    double w = 1.0;
#pragma unroll
    for (int kk = 1; 2 * kk <= M; ++kk) {
      w = w * (nd * rcp_int(2 * kk));
      double lap[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        double s = 0.0;
        if (it.v(t)) {
          const int a1 = it.a1(t), a2 = it.a2(t), a3 = it.a3(t);
          if (a1 >= 2) s += cur[flat3(a1 - 2, a2, a3)];
          if (a2 >= 2) s += cur[flat3(a1, a2 - 2, a3)];
          if (a3 >= 2) s += cur[flat3(a1, a2, a3 - 2)];
        }
        lap[t] = s;
        out[t] = fma(w, s, out[t]);
      }
      if (2 * (kk + 1) <= M) {
#pragma unroll
        for (int t = 0; t < T; ++t)
          if (it.v(t)) nxt[lane + 32 * t] = lap[t];
        __syncwarp();
        double* s = cur;
        cur = nxt;
        nxt = s;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < T; ++t)
    if (it.v(t)) dst[lane + 32 * t] = out[t];
  __syncwarp();
  return true;
}

// ------------------------------------------------------- rep scalars (uniform)
// rep_velocity (moment_rep.hpp:69-76) along one axis.
__device__ __forceinline__ double rep_u(const double* c, const double* p, int axis) {
  return p[axis] + c[1 + axis] / c[0];
}
// rep_temperature (moment_rep.hpp:80-93); 2e_d sit at positions 4, 7, 9.
__device__ __forceinline__ double rep_theta(const double* c, const double* p) {
  const double rho = c[0];
  double trace = 0.0, fe2 = 0.0;
  trace += c[4];
  fe2 += c[1] * c[1];
  trace += c[7];
  fe2 += c[2] * c[2];
  trace += c[9];
  fe2 += c[3] * c[3];
  return p[3] + (2.0 * trace - fe2 / rho) / (3.0 * rho);
}
// grad_defect (moment_rep.hpp:97-110)
__device__ __forceinline__ double grad_defect(const double* c) {
  double defect = 0.0, trace = 0.0;
  defect = smax(defect, fabs(c[1]));
  trace += c[4];
  defect = smax(defect, fabs(c[2]));
  trace += c[7];
  defect = smax(defect, fabs(c[3]));
  trace += c[9];
  defect = smax(defect, fabs(trace));
  return defect / fabs(c[0]);
}

// ------------------------------------------------------- half-range kernels
// Combined half-flux kernels for a basis with normal mean u_n and spread
// theta = rs^2 (flux.cpp:58-73 with the m-loop kernel hoisted):
//   Kup(m,p) = u_n P+(m,p) + rs P+(m+1,p) + rs m P+(m-1,p),   P+ = upper
//   Klo(m,p) = same with P- = lower = m! delta - upper  (halfspace.hpp:46-49)
// for m, p = 0..M.  Lane p computes column p of the pairing table by the
// reference recurrence (halfspace.hpp:38-41), the (m, p-1) entry arriving
// from lane p-1 by shuffle.  Tables are row-major [m*(M+1)+p]; synced on return.
template <int M>
__device__ __noinline__ void half_kernels(double un, double rs, double* Kup, double* Klo) {
  constexpr int P = M + 1;  // pmax
  const int lane = lane_id();
  const double a = -un / rs;
  const double g = exp(-a * a * 0.5) * 0.3989422804014327;  // e^{-a^2/2}/sqrt(2 pi)
  double he[P + 1];
  he[0] = 1.0;
  he[1] = a;
#pragma unroll
  for (int k = 1; k + 1 <= P; ++k) he[k + 1] = a * he[k] - (double)k * he[k - 1];
  double mine = 0.0, prevhe = 0.0;
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    if (k == lane) mine = he[k];
    if (k == lane - 1) prevhe = he[k];
  }
  double col[P + 1];
  col[0] = lane == 0 ? 0.5 * erfc(a * 0.7071067811865476) : prevhe * g;
  const double pl = (double)lane;
#pragma unroll
  for (int m = 0; m + 1 <= P; ++m) {
    const double left = __shfl_up_sync(FULL, col[m], 1);
    const double t = he[m] * mine * g;
    col[m + 1] = lane > 0 ? fma(pl, left, t) : t;
  }
  if (lane <= M) {
    double fp = 1.0;
#pragma unroll
    for (int k = 2; k <= M; ++k)
      if (k <= lane) fp *= (double)k;
    double lo[P + 1];
#pragma unroll
    for (int m = 0; m <= P; ++m) lo[m] = (m == lane ? fp : 0.0) - col[m];
#pragma unroll
    for (int m = 0; m <= M; ++m) {
      double ku = fma(un, col[m], rs * col[m + 1]);
      double kl = fma(un, lo[m], rs * lo[m + 1]);
      if (m > 0) {
        ku = fma(rs * (double)m, col[m - 1], ku);
        kl = fma(rs * (double)m, lo[m - 1], kl);
      }
      Kup[m * (M + 1) + lane] = ku;
      Klo[m * (M + 1) + lane] = kl;
    }
  }
  __syncwarp();
}

// Half-space flux sum (flux.cpp:58-73) in the basis of the inputs:
//   dst_k = (1/p!) sum_m rs^(p-m) (fa[beta|m] Ka(m,p) + fb[beta|m] Kb(m,p))
// with p = beta_axis.  fb may be null (single half).  dst must not alias the
// inputs; synced on return.
template <int M>
__device__ __noinline__ void half_sum(const uint32_t* alpha, const double* fa, const double* Ka,
                                      const double* fb, const double* Kb, int axis, double rs,
                                      double* dst) {
  constexpr int T = Cfg<M>::T;
  const Items<M> it(alpha);
  const int lane = lane_id();
  const double irs = 1.0 / rs;
  double rpow[M + 1];
  rpow[0] = 1.0;
#pragma unroll
  for (int e = 1; e <= M; ++e) rpow[e] = rpow[e - 1] * rs;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    if (!it.v(t)) continue;
    const int a1 = it.a1(t), a2 = it.a2(t), a3 = it.a3(t);
    const int p = it.ax(t, axis);
    const int tan = a1 + a2 + a3 - p;
    double fac = 1.0, ifact = 1.0;
#pragma unroll
    for (int e = 1; e <= M; ++e)
      if (e <= p) {
        fac = rpow[e];
        ifact *= rcp_int(e);
      }
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m <= M; ++m) {
      if (m + tan <= M) {
        const int idx = flat3(axis == 0 ? m : a1, axis == 1 ? m : a2, axis == 2 ? m : a3);
        double v = fa[idx] * Ka[m * (M + 1) + p];
        if (fb) v = fma(fb[idx], Kb[m * (M + 1) + p], v);
        acc = fma(fac, v, acc);
      }
      fac *= irs;
    }
    dst[lane + 32 * t] = acc * ifact;
  }
  __syncwarp();
}

// full_flux_coeffs (flux.cpp:10-27) of src (basis normal mean un, spread
// theta) into dst (must not alias src); synced on return.
template <int M>
__device__ __noinline__ void full_flux(const uint32_t* alpha, const double* src, double un,
                                       double theta, int axis, double* dst) {
  const Items<M> it(alpha);
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    if (!it.v(t)) continue;
    const int a1 = it.a1(t), a2 = it.a2(t), a3 = it.a3(t);
    const int an = it.ax(t, axis);
    const int k = lane + 32 * t;
    double g = un * src[k];
    if (an >= 1) g = fma(theta, src[flat3(a1 - (axis == 0), a2 - (axis == 1), a3 - (axis == 2))], g);
    if (a1 + a2 + a3 < M)
      g = fma((double)(an + 1), src[flat3(a1 + (axis == 0), a2 + (axis == 1), a3 + (axis == 2))], g);
    dst[k] = g;
  }
  __syncwarp();
}

// Element-wise helpers over a warp's vectors (synced on return).
template <int M>
__device__ __forceinline__ void vcopy(double* dst, const double* src) {
  for (int k = lane_id(); k < Cfg<M>::N; k += 32) dst[k] = src[k];
  __syncwarp();
}

}  // namespace momg_gpu
