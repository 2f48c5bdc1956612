// Warp-cooperative FP64 device primitives of the moment method (sm_100a).
//
// One warp owns one cell at a time.  Every N-vector of Hermite coefficients
// lives in a per-warp shared-memory buffer of NB doubles whose slot N holds a
// constant 0.0 (the "zero slot"); lane l owns coefficients k = l, l+32, ...
// (T = ceil(N/32) items) and keeps their running values in registers.
//
// Index structure.  All cross-coefficient access patterns of the path are
// chains along one velocity axis of the graded-lex multi-index set
// (multi_index.hpp:31-52): mean/spread shifts (projection.hpp:16-57) walk
// alpha - n e_d, the half-space flux (flux.cpp:58-73) walks the pencil
// beta|_{beta_n = m}.  A per-block table (built once per launch, laid out
// [word][lane] so every lane's lookups are bank-conflict free) stores, per
// lane item, the source positions of those chains as bytes, with out-of-set
// positions pointing at the zero slot.  A chain term is then
// byte-extract + shared load + FMA, with no integer graded-lex arithmetic.
//
// Projection.  The reference applies three mean shifts (Taylor sums along
// each axis) and one spread shift exp(-dtheta/2 L), L = sum_d down_d^2
// (projection.hpp:16-73).  All these operators commute and L splits by axis,
// so the projection is the product over axes of the lower-triangular
// Toeplitz operators  T_d = sum_n c^d_n down_d^n  with
//   c^d_n = sum_{j+2k=n} (-delta_d)^j/j! (-dtheta/2)^k/k!,
// i.e. three axis passes of M chain terms each.  Identical in exact
// arithmetic; rounding differs from the reference at the ulp level (the
// parity bar is 1e-10 relative).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "types.h"

namespace momg_gpu {

constexpr unsigned FULL = 0xffffffffu;

template <int M>
struct Cfg {
  static constexpr int N = tet(M + 1);          // IndexSet::count
  static constexpr int NP = (N + 3) & ~3;       // global row pitch in doubles (32 B sectors)
  static constexpr int NB = (N + 2) & ~1;       // smem buffer stride: N coefficients + zero slot
  static constexpr int T = (N + 31) / 32;       // items per lane
  static constexpr int K1 = M + 1;              // half-flux kernel table side
  static constexpr int KT = K1 * K1;
  static constexpr int CW = (M + 3) / 4;        // 32-bit words per chain (M bytes)
  static constexpr int PW = (M + 4) / 4;        // 32-bit words per pencil (M+1 bytes)
  // per-lane table layout (words); entry w of lane l at tab[w * 32 + l]
  static constexpr int W_CH = 0;                        // [t][d][CW]   chain alpha - n e_d, n=1..M
  static constexpr int W_PEN = T * 3 * CW;              // [t][a][PW]   pencil beta|_{beta_a=m}, m=0..M
  static constexpr int W_MISC = W_PEN + T * 2 * PW;     // [t]          a1 | a2<<8 | a3<<16
  static constexpr int WORDS = W_MISC + T;
  static constexpr int PC = 3 * M;                      // coefficients per projection (c^d_n, n>=1)
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ constexpr double rcp_int(int n) { return 1.0 / (double)n; }

// std::min / std::max semantics (NaN handling as the reference).
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// ----------------------------------------------------------- index tables
__device__ __forceinline__ void decode(int k, int& a1, int& a2, int& a3) {
  int D = 0;
  while (tet(D + 1) <= k) ++D;
  const int rem = k - tet(D);
  int r = 0;
  while (tri(r + 1) <= rem) ++r;
  a3 = rem - tri(r);
  a2 = r - a3;
  a1 = D - r;
}

// Builds the per-lane chain/pencil tables of one block (all threads).
template <int M>
__device__ __forceinline__ void build_tables(uint32_t* tab) {
  using C = Cfg<M>;
  constexpr int N = C::N;
  for (int e = threadIdx.x; e < 32 * C::T; e += blockDim.x) {
    const int l = e & 31, t = e >> 5;
    const int k = l + 32 * t;
    int a[3] = {0, 0, 0};
    const bool valid = k < N;
    if (valid) decode(k, a[0], a[1], a[2]);
    const int D = a[0] + a[1] + a[2];
    for (int d = 0; d < 3; ++d) {
      for (int w = 0; w < C::CW; ++w) {
        uint32_t word = 0;
        for (int b = 0; b < 4; ++b) {
          const int n = 4 * w + b + 1;
          int src = N;
          if (valid && n <= M && n <= a[d]) {
            int s[3] = {a[0], a[1], a[2]};
            s[d] -= n;
            src = flat3(s[0], s[1], s[2]);
          }
          word |= (uint32_t)(src & 0xff) << (8 * b);
        }
        tab[(C::W_CH + (t * 3 + d) * C::CW + w) * 32 + l] = word;
      }
    }
    for (int ax = 0; ax < 2; ++ax) {
      const int tan = D - a[ax];
      for (int w = 0; w < C::PW; ++w) {
        uint32_t word = 0;
        for (int b = 0; b < 4; ++b) {
          const int m = 4 * w + b;
          int src = N;
          if (valid && m <= M && m + tan <= M) {
            int s[3] = {a[0], a[1], a[2]};
            s[ax] = m;
            src = flat3(s[0], s[1], s[2]);
          }
          word |= (uint32_t)(src & 0xff) << (8 * b);
        }
        tab[(C::W_PEN + (t * 2 + ax) * C::PW + w) * 32 + l] = word;
      }
    }
    tab[(C::W_MISC + t) * 32 + l] = (uint32_t)a[0] | ((uint32_t)a[1] << 8) | ((uint32_t)a[2] << 16);
  }
}

__device__ __forceinline__ int byte_of(uint32_t w, int b) { return (w >> (8 * b)) & 0xff; }

// Position of lane item t, or the zero slot for the padding items of the
// last slot.
template <int M>
__device__ __forceinline__ int item_pos(int t) {
  const int k = lane_id() + 32 * t;
  return (t < Cfg<M>::T - 1 || k < Cfg<M>::N) ? k : Cfg<M>::N;
}

template <int M>
__device__ __forceinline__ uint32_t misc(const uint32_t* tab, int t) {
  return tab[(Cfg<M>::W_MISC + t) * 32 + lane_id()];
}

struct P4 {
  double v[4];
};

// --------------------------------------------------------- projection
// Lane-parallel setup: c[d*M + n-1] = c^d_n for the projection from -> to.
// Executed by the whole warp (tasks strided over lanes); caller syncs.
template <int M>
__device__ __forceinline__ void proj_coeffs(P4 from, P4 to, double* c) {
  const double ds = to.v[3] - from.v[3];
  for (int task = lane_id(); task < 3 * M; task += 32) {
    const int d = task / M, n = task % M + 1;
    const double dd = to.v[d] - from.v[d];
    double aj[M + 1], bk[M / 2 + 1];
    aj[0] = 1.0;
#pragma unroll
    for (int j = 1; j <= M; ++j) aj[j] = aj[j - 1] * (-dd * rcp_int(j));
    bk[0] = 1.0;
#pragma unroll
    for (int k = 1; 2 * k <= M; ++k) bk[k] = bk[k - 1] * (-0.5 * ds * rcp_int(k));
    double s = 0.0;
#pragma unroll
    for (int k = 0; 2 * k <= M; ++k)
#pragma unroll
      for (int j = 0; j <= M; ++j)
        if (j + 2 * k == n) s = fma(aj[j], bk[k], s);
    c[task] = s;
  }
}

// Which axis passes a projection needs (identity when both deltas vanish,
// the reference's `delta == 0` early returns, projection.hpp:18, 36).
__device__ __forceinline__ int pass_mask(P4 from, P4 to) {
  const bool ds = to.v[3] != from.v[3];
  return ((ds || to.v[0] != from.v[0]) ? 1 : 0) | ((ds || to.v[1] != from.v[1]) ? 2 : 0) |
         ((ds || to.v[2] != from.v[2]) ? 4 : 0);
}

// One axis pass: dst[k] = v[k] + sum_{n=1..M} c^d_n src[alpha - n e_d].
// v holds src[k] on entry and dst[k] on exit.  dst != src; synced on return.
template <int M>
__device__ __forceinline__ void axis_pass(const uint32_t* tab, const double* src, double* dst,
                                          const double* c, int d, double* v) {
  using C = Cfg<M>;
  const int lane = lane_id();
  double cc[M];
#pragma unroll
  for (int n = 0; n < M; ++n) cc[n] = c[d * M + n];
#pragma unroll
  for (int t = 0; t < C::T; ++t) {
    double acc = v[t];
#pragma unroll
    for (int w = 0; w < C::CW; ++w) {
      const uint32_t word = tab[(C::W_CH + (t * 3 + d) * C::CW + w) * 32 + lane];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int n = 4 * w + b + 1;
        if (n <= M) acc = fma(cc[n - 1], src[byte_of(word, b)], acc);
      }
    }
    v[t] = acc;
  }
#pragma unroll
  for (int t = 0; t < C::T; ++t)
    if (t < C::T - 1 || lane + 32 * t < C::N) dst[lane + 32 * t] = v[t];
  __syncwarp();
}

// Projects src (read-only) with precomputed coefficients c and pass mask;
// uses scratch buffers x, y.  Returns the buffer holding the result (src
// itself when no pass runs); v holds the result items.
template <int M>
__device__ __forceinline__ const double* project_apply(const uint32_t* tab, const double* src,
                                                       double* x, double* y, const double* c,
                                                       int mask, double* v) {
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) v[t] = src[item_pos<M>(t)];
  (void)lane;
  const double* cur = src;
  double* nxt = x;
  double* other = y;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (!(mask & (1 << d))) continue;
    axis_pass<M>(tab, cur, nxt, c, d, v);
    cur = nxt;
    double* s = nxt;
    nxt = other;
    other = s;
  }
  return cur;
}

// Two projections sharing their sync points (the two face states).
template <int M>
__device__ __forceinline__ void project_apply2(const uint32_t* tab, const double* srcA, double* xA,
                                               double* yA, const double* cA, int maskA,
                                               double* vA, const double* srcB, double* xB,
                                               double* yB, const double* cB, int maskB,
                                               double* vB, const double** outA,
                                               const double** outB) {
  using C = Cfg<M>;
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < C::T; ++t) {
    vA[t] = srcA[item_pos<M>(t)];
    vB[t] = srcB[item_pos<M>(t)];
  }
  const double* curA = srcA;
  double* nA = xA;
  double* oA = yA;
  const double* curB = srcB;
  double* nB = xB;
  double* oB = yB;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const bool ra = maskA & (1 << d), rb = maskB & (1 << d);
    if (!ra && !rb) continue;
    double ccA[M], ccB[M];
#pragma unroll
    for (int n = 0; n < M; ++n) {
      ccA[n] = cA[d * M + n];
      ccB[n] = cB[d * M + n];
    }
#pragma unroll
    for (int t = 0; t < C::T; ++t) {
      double accA = vA[t], accB = vB[t];
#pragma unroll
      for (int w = 0; w < C::CW; ++w) {
        const uint32_t word = tab[(C::W_CH + (t * 3 + d) * C::CW + w) * 32 + lane];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int n = 4 * w + b + 1;
          if (n <= M) {
            const int s = byte_of(word, b);
            if (ra) accA = fma(ccA[n - 1], curA[s], accA);
            if (rb) accB = fma(ccB[n - 1], curB[s], accB);
          }
        }
      }
      vA[t] = accA;
      vB[t] = accB;
    }
#pragma unroll
    for (int t = 0; t < C::T; ++t)
      if (t < C::T - 1 || lane + 32 * t < C::N) {
        if (ra) nA[lane + 32 * t] = vA[t];
        if (rb) nB[lane + 32 * t] = vB[t];
      }
    __syncwarp();
    if (ra) {
      curA = nA;
      double* s = nA;
      nA = oA;
      oA = s;
    }
    if (rb) {
      curB = nB;
      double* s = nB;
      nB = oB;
      oB = s;
    }
  }
  *outA = curA;
  *outB = curB;
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
// Folded half-flux kernels for a basis with normal mean u_n and spread
// theta = rs^2 (flux.cpp:58-73 with the kernel and the rs powers hoisted):
//   Kup[m][p] = rs^(p-m)/p! (u_n P+(m,p) + rs P+(m+1,p) + rs m P+(m-1,p)),
//   Klo[m][p] = same with P- = lower = m! delta - upper  (halfspace.hpp:46-49)
// for m, p = 0..M.  Lane p computes column p of the pairing table by the
// reference recurrence (halfspace.hpp:38-41), the (m, p-1) entry arriving
// from lane p-1 by shuffle.  All lanes must call; caller syncs.
template <int M>
__device__ __forceinline__ void half_kernels(double un, double rs, double* Kup, double* Klo) {
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
    double fp = 1.0, rsp = 1.0;  // lane!, rs^lane
#pragma unroll
    for (int k = 1; k <= M; ++k)
      if (k <= lane) {
        fp *= (double)k;
        rsp *= rs;
      }
    const double irs = 1.0 / rs;
    double scale = rsp / fp;  // rs^(p-m)/p! at m = 0
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
      Kup[m * (M + 1) + lane] = scale * ku;
      Klo[m * (M + 1) + lane] = scale * kl;
      scale *= irs;
    }
  }
}

// Half-space flux sum in the inputs' basis (flux.cpp:58-73, folded kernels):
//   out_k = sum_m fa[beta|m] Ka[m][p] + fb[beta|m] Kb[m][p],  p = beta_axis.
// fb may be null (single half).  Result in registers.
template <int M>
__device__ __forceinline__ void half_sum(const uint32_t* tab, const double* fa, const double* Ka,
                                         const double* fb, const double* Kb, int axis,
                                         double* out) {
  using C = Cfg<M>;
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < C::T; ++t) {
    const uint32_t ms = misc<M>(tab, t);
    const int p = byte_of(ms, axis);
    const double* ka = Ka + p;
    const double* kb = fb ? Kb + p : nullptr;
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < C::PW; ++w) {
      const uint32_t word = tab[(C::W_PEN + (t * 2 + axis) * C::PW + w) * 32 + lane];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int m = 4 * w + b;
        if (m <= M) {
          const int s = byte_of(word, b);
          acc = fma(fa[s], ka[m * (M + 1)], acc);
          if (fb) acc = fma(fb[s], kb[m * (M + 1)], acc);
        }
      }
    }
    out[t] = acc;
  }
}

// full_flux_coeffs (flux.cpp:10-27) of src (basis normal mean un, spread
// theta), result in registers.
template <int M>
__device__ __forceinline__ void full_flux(const uint32_t* tab, const double* src, double un,
                                          double theta, int axis, double* out) {
  using C = Cfg<M>;
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < C::T; ++t) {
    const int k = lane + 32 * t;
    const uint32_t ms = misc<M>(tab, t);
    const int a[3] = {byte_of(ms, 0), byte_of(ms, 1), byte_of(ms, 2)};
    const int an = a[axis];
    double g = un * src[k < C::N ? k : C::N];
    // alpha - e_axis: first chain entry; alpha + e_axis: pencil entry m = an+1
    const uint32_t ch = tab[(C::W_CH + (t * 3 + axis) * C::CW) * 32 + lane];
    if (an >= 1) g = fma(theta, src[byte_of(ch, 0)], g);
    if (a[0] + a[1] + a[2] < M && k < C::N) {
      const int up = flat3(a[0] + (axis == 0), a[1] + (axis == 1), a[2] + (axis == 2));
      g = fma((double)(an + 1), src[up], g);
    }
    out[t] = g;
  }
}

template <int M>
__device__ __forceinline__ void store_items(double* dst, const double* v) {
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t)
    if (t < Cfg<M>::T - 1 || lane + 32 * t < Cfg<M>::N) dst[lane + 32 * t] = v[t];
}

}  // namespace momg_gpu
