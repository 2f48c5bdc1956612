// Split design of the exact-order fast-sweeping update (moment orders 3..5).
//
// The sweep is latency-bound: its dependency DAG has ~2.5-4 (nx+ny) levels
// per iteration, so the time of ONE cell update is what matters.  A block
// updates a segment of 32 independent cells of one anti-diagonal (lane =
// cell).  The four face fluxes of every cell are evaluated concurrently by
// four face groups of 4 warps each, and each face's work (the two
// projections into the face basis, the half-space flux, the projection back)
// is cut into 4 compile-time partitions of balanced cost (gen/split_gen.cuh),
// one per warp.  Axis passes are split by pencils (disjoint element sets) and
// run in place; a named barrier of the face group separates consecutive
// passes.  Group 0 then assembles the residual, applies the local update and
// re-normalises, again split 4 ways.  Control flow around barriers is uniform
// per group (per-cell decisions only select the work done between barriers).
#pragma once

#include <cuda_runtime.h>

#include "gen/split_gen.cuh"
#include "thread_cell.cuh"
#include "types.h"

namespace momg_gpu {
namespace sp {

constexpr int P = 4;                 // warps (partitions) per face group
constexpr int G = 4;                 // face groups: x-low, x-high, y-low, y-high
constexpr int THREADS = 32 * P * G;  // 512

using tc::P4;

template <int M>
struct Layout {
  static constexpr int N = Gen<M>::N;
  static constexpr int VEC = N * SPV;  // doubles of one vector for the 32 cells (stride SPV)
  // per group L, U, F; then SB (cell state) and RB (rhs) of the update
  static constexpr size_t bytes = ((size_t)G * 3 + 2) * VEC * sizeof(double) + 64;
};

// Non-.aligned named barriers: lanes of one warp may reach them from
// divergent paths (bar.sync is the .aligned form and would not allow it).
__device__ __forceinline__ void gbar(int g) {
  asm volatile("barrier.cta.sync %0, %1;" ::"r"(g + 1), "r"(32 * P) : "memory");
}
// barrier of face group g returning whether any thread passed a nonzero flag
__device__ __forceinline__ int gbar_or(int g, int flag) {
  int out;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.s32 p, %1, 0;\n barrier.cta.red.or.pred q, %2, %3, p;\n"
      " selp.s32 %0, 1, 0, q;\n}"
      : "=r"(out)
      : "r"(flag), "r"(g + 1), "r"(32 * P)
      : "memory");
  return out;
}

#define SP_DISPATCH(q, call) \
  switch (q) {               \
    case 0: call(0); break;  \
    case 1: call(1); break;  \
    case 2: call(2); break;  \
    default: call(3); break; \
  }

// projection coefficients of exp(a t + b t^2) (see tc::project)
template <int M>
__device__ __forceinline__ void coeffs(const P4& from, const P4& to, int d, double* c) {
  const double b2 = -(to.v[3] - from.v[3]);
  const double a = -(to.v[d] - from.v[d]);
  c[0] = 1.0;
  c[1] = a;
#pragma unroll
  for (int n = 2; n <= M; ++n) c[n] = fma(a, c[n - 1], b2 * c[n - 2]) * tc::rcp(n);
}

// one in-place axis pass of partition q on vector v (base of this cell)
template <int M>
__device__ __forceinline__ void pass(int q, int d, double* v, const double* c) {
#define SP_PASS(Q)                                            \
  {                                                           \
    if (d == 0) Split<M, P>::pass0_##Q(v, c);                 \
    else if (d == 1) Split<M, P>::pass1_##Q(v, c);            \
    else Split<M, P>::pass2_##Q(v, c);                        \
  }
  SP_DISPATCH(q, SP_PASS)
#undef SP_PASS
}

// both vectors' passes of partition q with every load issued first
template <int M>
__device__ __forceinline__ void pass_two(int q, int d, double* a, const double* ca, bool acta, double* b,
                                         const double* cb, bool actb) {
#define SP_PASS2(Q)                                                    \
  {                                                                    \
    if (d == 0) Split<M, P>::pass20_##Q(a, ca, acta, b, cb, actb);     \
    else if (d == 1) Split<M, P>::pass21_##Q(a, ca, acta, b, cb, actb); \
    else Split<M, P>::pass22_##Q(a, ca, acta, b, cb, actb);            \
  }
  SP_DISPATCH(q, SP_PASS2)
#undef SP_PASS2
}

// Projection (projection.hpp:64-89) of the vectors of this cell, split over
// the group's partitions: every thread of the group runs the three passes
// and barriers; `active` selects whether this cell's vector is touched.
template <int M>
__device__ __forceinline__ void project2(int g, int q, double* a, const P4& af, const P4& at, bool act_a,
                                         double* b, const P4& bf, const P4& bt, bool act_b) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double ca[M + 1], cb[M + 1];
    coeffs<M>(af, at, d, ca);
    coeffs<M>(bf, bt, d, cb);
    if (act_a || act_b) pass_two<M>(q, d, a, ca, act_a, b, cb, act_b);
    gbar(g);
  }
}

// single-vector projection (one pass body per call site)
template <int M>
__device__ __forceinline__ void project1(int g, int q, double* a, const P4& af, const P4& at, bool act_a) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double ca[M + 1];
    coeffs<M>(af, at, d, ca);
    if (act_a) pass<M>(q, d, a, ca);
    gbar(g);
  }
}

template <int M, int AXIS>
__device__ __forceinline__ void half_sum(int q, const double* L, const double* U, const double (&Ku)[M + 1][M + 1],
                                         const double (&Kl)[M + 1][M + 1], double* o) {
#define SP_HALF(Q)                                                      \
  {                                                                     \
    if (AXIS == 0) Split<M, P>::half_sum0_##Q(L, U, Ku, Kl, o);         \
    else Split<M, P>::half_sum1_##Q(L, U, Ku, Kl, o);                   \
  }
  SP_DISPATCH(q, SP_HALF)
#undef SP_HALF
}
template <int M, int AXIS>
__device__ __forceinline__ void half_one(int q, const double* L, const double (&K)[M + 1][M + 1], double* o) {
#define SP_ONE(Q)                                            \
  {                                                          \
    if (AXIS == 0) Split<M, P>::half_one0_##Q(L, K, o);      \
    else Split<M, P>::half_one1_##Q(L, K, o);                \
  }
  SP_DISPATCH(q, SP_ONE)
#undef SP_ONE
}
template <int M, int AXIS>
__device__ __forceinline__ void full_flux(int q, const double* s, double* o, double un, double th) {
#define SP_FULL(Q)                                                 \
  {                                                                \
    if (AXIS == 0) Split<M, P>::full_flux0_##Q(s, o, un, th);      \
    else Split<M, P>::full_flux1_##Q(s, o, un, th);                \
  }
  SP_DISPATCH(q, SP_FULL)
#undef SP_FULL
}

// (one reciprocal of the density, shared by the callers after CSE: no
// divisions on the face / update critical path; differences from the
// reference's divisions are single roundings)
__device__ __forceinline__ double rep_u32(const double* v, const P4& p, int axis) {
  return p.v[axis] + v[(1 + axis) * SPV] * (1.0 / v[0]);
}
__device__ __forceinline__ double rep_theta32(const double* v, const P4& p) {
  const double rho = v[0];
  double trace = 0.0, fe2 = 0.0;
  const double c1 = v[1 * SPV], c2 = v[2 * SPV], c3 = v[3 * SPV];
  trace += v[4 * SPV];
  fe2 += c1 * c1;
  trace += v[7 * SPV];
  fe2 += c2 * c2;
  trace += v[9 * SPV];
  fe2 += c3 * c3;
  const double ir = 1.0 / rho;
  return p.v[3] + (2.0 * trace - fe2 * ir) * (ir * (1.0 / 3.0));
}
__device__ __forceinline__ double grad_defect32(const double* v) {
  double defect = 0.0, trace = 0.0;
  defect = tc::smax(defect, fabs(v[1 * SPV]));
  trace += v[4 * SPV];
  defect = tc::smax(defect, fabs(v[2 * SPV]));
  trace += v[7 * SPV];
  defect = tc::smax(defect, fabs(v[3 * SPV]));
  trace += v[9 * SPV];
  defect = tc::smax(defect, fabs(trace));
  return defect * fabs(1.0 / v[0]);
}

template <int M>
__device__ __forceinline__ void krange(int q, int* lo, int* hi) {
  *lo = (q * Gen<M>::N) / P;
  *hi = ((q + 1) * Gen<M>::N) / P;
}

enum : int { B_NONE = 0, B_HALF = 1, B_FULL_L = 2, B_FULL_R = 3, B_WALL = 4 };

// Element-wise copies of partition Q with compile-time bounds: every load is
// issued before the first dependent store, so one L2 round trip covers the
// whole partition (a runtime-bounded loop serialises them).
template <int M, int Q>
struct Part {
  static constexpr int LO = (Q * Gen<M>::N) / P, HI = ((Q + 1) * Gen<M>::N) / P, CNT = HI - LO;
  static __device__ __forceinline__ void load(const double* __restrict__ src, double* __restrict__ dst) {
    double r[CNT];
#pragma unroll
    for (int k = 0; k < CNT; ++k) r[k] = __ldcg(src + LO + k);
#pragma unroll
    for (int k = 0; k < CNT; ++k) dst[(LO + k) * SPV] = r[k];
  }
  static __device__ __forceinline__ void load2(const double* __restrict__ s0, double* __restrict__ d0,
                                               const double* __restrict__ s1, double* __restrict__ d1) {
    double r0[CNT], r1[CNT];
#pragma unroll
    for (int k = 0; k < CNT; ++k) {
      r0[k] = __ldcg(s0 + LO + k);
      r1[k] = __ldcg(s1 + LO + k);
    }
#pragma unroll
    for (int k = 0; k < CNT; ++k) {
      d0[(LO + k) * SPV] = r0[k];
      d1[(LO + k) * SPV] = r1[k];
    }
  }
  static __device__ __forceinline__ void copy(const double* __restrict__ s, double* __restrict__ d) {
#pragma unroll
    for (int k = 0; k < CNT; ++k) d[(LO + k) * SPV] = s[(LO + k) * SPV];
  }
  // second-order face states in place from raw L (lower) and U (upper):
  //   L += offL (U - LL) rhL,  U += offU (UU - L) rhU  (spatial.cpp:34-80)
  static __device__ __forceinline__ void recon2(double* L, double* U, const double* gLL, const double* gUU,
                                                bool rl, bool ru, double offL, double rhL, double offU,
                                                double rhU) {
    double ll[CNT], uu[CNT];
#pragma unroll
    for (int k = 0; k < CNT; ++k) {
      ll[k] = rl ? __ldcg(gLL + LO + k) : 0.0;
      uu[k] = ru ? __ldcg(gUU + LO + k) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < CNT; ++k) {
      const double lk = L[(LO + k) * SPV], uk = U[(LO + k) * SPV];
      if (rl) L[(LO + k) * SPV] = fma(offL, (uk - ll[k]) * rhL, lk);
      if (ru) U[(LO + k) * SPV] = fma(offU, (uu[k] - lk) * rhU, uk);
    }
  }
  // dst = c + off * (h - l) * rh  (second-order face state, spatial.cpp:64-80)
  static __device__ __forceinline__ void recon(const double* __restrict__ c, const double* __restrict__ l,
                                               const double* __restrict__ h, double off, double rh,
                                               double* __restrict__ dst) {
    double rc[CNT], rl[CNT], rhh[CNT];
#pragma unroll
    for (int k = 0; k < CNT; ++k) {
      rc[k] = __ldcg(c + LO + k);
      rl[k] = __ldcg(l + LO + k);
      rhh[k] = __ldcg(h + LO + k);
    }
#pragma unroll
    for (int k = 0; k < CNT; ++k) dst[(LO + k) * SPV] = fma(off, (rhh[k] - rl[k]) * rh, rc[k]);
  }
  // residual assembly (spatial.cpp:127-132, collision.hpp:120-127), update_delta
  // (single_level.cpp:64-70) and f + dt delta (apply_update :47)
  // elements [LO + KB, LO + KE) of the partition (default: all of them)
  template <int KB = 0, int KE = CNT>
  static __device__ __forceinline__ void assemble(const double* S, const double* RH, const double* Fxm,
                                                  const double* Fxp, const double* Fym, const double* Fyp,
                                                  double nu, int shakhov, double shw, const double* qv,
                                                  double idx, double idy, double dt, bool rhs, double* D,
                                                  double* V) {
#pragma unroll
    for (int kk = KB; kk < KE; ++kk) {
      constexpr int dummy = 0;
      (void)dummy;
      const int k = LO + kk;
      double eq = k == 0 ? S[0] : 0.0;
      if (shakhov) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int e = 0; e < 3; ++e)
            if (k == flat3((e == 0 ? 2 : 0) + (d == 0), (e == 1 ? 2 : 0) + (d == 1), (e == 2 ? 2 : 0) + (d == 2)))
              eq = shw * qv[d];
      }
      const double sk = S[k * SPV];
      double r = nu * (eq - sk);
      r -= (Fxp[k * SPV] - Fxm[k * SPV]) * idx;
      r -= (Fyp[k * SPV] - Fym[k * SPV]) * idy;
      if (rhs) r -= RH[k * SPV];
      D[k * SPV] = r;
      V[k * SPV] = fma(dt, r, sk);
    }
  }
  static __device__ __forceinline__ void restep(const double* S, const double* D, double step, double* V) {
#pragma unroll
    for (int kk = 0; kk < CNT; ++kk) V[(LO + kk) * SPV] = fma(step, D[(LO + kk) * SPV], S[(LO + kk) * SPV]);
  }
  static __device__ __forceinline__ void store(const double* __restrict__ v, double* __restrict__ dst) {
    double r[CNT];
#pragma unroll
    for (int k = 0; k < CNT; ++k) r[k] = v[(LO + k) * SPV];
#pragma unroll
    for (int k = 0; k < CNT; ++k) __stcg(dst + LO + k, r[k]);
  }
};

template <int M>
__device__ __forceinline__ void part_load(int q, const double* src, double* dst) {
#define SP_LD(Q) Part<M, Q>::load(src, dst)
  SP_DISPATCH(q, SP_LD)
#undef SP_LD
}
template <int M>
__device__ __forceinline__ void part_recon(int q, const double* c, const double* l, const double* h, double off,
                                           double rh, double* dst) {
#define SP_RC(Q) Part<M, Q>::recon(c, l, h, off, rh, dst)
  SP_DISPATCH(q, SP_RC)
#undef SP_RC
}
template <int M>
__device__ __forceinline__ void part_load2(int q, const double* s0, double* d0, const double* s1, double* d1) {
#define SP_L2(Q) Part<M, Q>::load2(s0, d0, s1, d1)
  SP_DISPATCH(q, SP_L2)
#undef SP_L2
}
template <int M>
__device__ __forceinline__ void part_copy(int q, const double* src, double* dst) {
#define SP_CP(Q) Part<M, Q>::copy(src, dst)
  SP_DISPATCH(q, SP_CP)
#undef SP_CP
}
template <int M>
__device__ __forceinline__ void part_recon2(int q, double* L, double* U, const double* gLL, const double* gUU,
                                            bool rl, bool ru, double offL, double rhL, double offU, double rhU) {
#define SP_R2(Q) Part<M, Q>::recon2(L, U, gLL, gUU, rl, ru, offL, rhL, offU, rhU)
  SP_DISPATCH(q, SP_R2)
#undef SP_R2
}
template <int M>
__device__ __forceinline__ void part_store(int q, const double* v, double* dst) {
#define SP_ST(Q) Part<M, Q>::store(v, dst)
  SP_DISPATCH(q, SP_ST)
#undef SP_ST
}

// --------------------------------------------------------------- face phase
// Face flux of face group g (AXIS = g/2, high = g%2) for cell (i, j) (lane),
// partition q; result (cell basis) left in F.  `valid` false: barriers only.
// Returns W_NONE or the failure kind (same in all partitions of the cell).
// Phase 3 of one partition: kernels of its own half-flux columns only (so
// the other partitions' columns are dead code), then its share of the
// half / full flux.  Partition 0 also returns row 0 of the incoming-side
// wall kernel for the wall closure.
template <int M, int AXIS, int Q>
__device__ __forceinline__ void flux_q(int branch, bool high, double un, double rs, const tc::HalfBase& hb,
                                       const P4& fp, const double* L, const double* U, double* F,
                                       double (&kin0)[M + 1]) {
  if (branch == B_HALF || branch == B_WALL) {
    double Ku[M + 1][M + 1], Kl[M + 1][M + 1];
    tc::half_kernels_b<M>(un, rs, hb, Ku, Kl);
    if (branch == B_HALF) {
      if constexpr (AXIS == 0) {
        if constexpr (Q == 0) Split<M, P>::half_sum0_0(L, U, Ku, Kl, F);
        else if constexpr (Q == 1) Split<M, P>::half_sum0_1(L, U, Ku, Kl, F);
        else if constexpr (Q == 2) Split<M, P>::half_sum0_2(L, U, Ku, Kl, F);
        else Split<M, P>::half_sum0_3(L, U, Ku, Kl, F);
      } else {
        if constexpr (Q == 0) Split<M, P>::half_sum1_0(L, U, Ku, Kl, F);
        else if constexpr (Q == 1) Split<M, P>::half_sum1_1(L, U, Ku, Kl, F);
        else if constexpr (Q == 2) Split<M, P>::half_sum1_2(L, U, Ku, Kl, F);
        else Split<M, P>::half_sum1_3(L, U, Ku, Kl, F);
      }
    } else {
      double Kw[M + 1][M + 1];
#pragma unroll
      for (int m = 0; m <= M; ++m)
#pragma unroll
        for (int p = 0; p <= M; ++p) Kw[m][p] = high ? Ku[m][p] : Kl[m][p];
      if constexpr (AXIS == 0) {
        if constexpr (Q == 0) Split<M, P>::half_one0_0(L, Kw, F);
        else if constexpr (Q == 1) Split<M, P>::half_one0_1(L, Kw, F);
        else if constexpr (Q == 2) Split<M, P>::half_one0_2(L, Kw, F);
        else Split<M, P>::half_one0_3(L, Kw, F);
      } else {
        if constexpr (Q == 0) Split<M, P>::half_one1_0(L, Kw, F);
        else if constexpr (Q == 1) Split<M, P>::half_one1_1(L, Kw, F);
        else if constexpr (Q == 2) Split<M, P>::half_one1_2(L, Kw, F);
        else Split<M, P>::half_one1_3(L, Kw, F);
      }
      if constexpr (Q == 0) {
#pragma unroll
        for (int p = 0; p <= M; ++p) kin0[p] = high ? Kl[0][p] : Ku[0][p];
      }
    }
  } else if (branch == B_FULL_L || branch == B_FULL_R) {
    const double* src = branch == B_FULL_L ? L : U;
    if constexpr (AXIS == 0) {
      if constexpr (Q == 0) Split<M, P>::full_flux0_0(src, F, fp.v[0], fp.v[3]);
      else if constexpr (Q == 1) Split<M, P>::full_flux0_1(src, F, fp.v[0], fp.v[3]);
      else if constexpr (Q == 2) Split<M, P>::full_flux0_2(src, F, fp.v[0], fp.v[3]);
      else Split<M, P>::full_flux0_3(src, F, fp.v[0], fp.v[3]);
    } else {
      if constexpr (Q == 0) Split<M, P>::full_flux1_0(src, F, fp.v[1], fp.v[3]);
      else if constexpr (Q == 1) Split<M, P>::full_flux1_1(src, F, fp.v[1], fp.v[3]);
      else if constexpr (Q == 2) Split<M, P>::full_flux1_2(src, F, fp.v[1], fp.v[3]);
      else Split<M, P>::full_flux1_3(src, F, fp.v[1], fp.v[3]);
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer0() {
#ifdef TRACE_CLOCK
  return (unsigned long long)clock64() * 1000ull / 1965ull;
#else
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
#endif
}

// Phases 1-4 of one face group on states already staged in L / U
// (face_flux, flux.cpp:77-132, and the back projection of spatial.cpp:118-125).
// branch: B_HALF (interior face, lp / rp the face states' bases) or B_WALL
// (L = the cell state in basis cp); invalid lanes pass B_NONE.
template <int M>
__device__ __forceinline__ int face_core(const DevCtx& ctx, int g, int q, int axis, bool high, int branch, int fail,
                                         const P4& lp, const P4& rp, const P4& cp, double* L, double* U,
                                         double* F, unsigned long long* stamp) {
  P4 fp{};
  // ---- phase 1: wave-speed bounds and branch (flux.cpp:77-97)
  P4 wb{};
  double rs = 1.0;
  if (branch == B_WALL) {
    // selects only: a runtime index would copy ctx / wb to local memory
    const double ws = axis == 0 ? (high ? ctx.wall_speed[1] : ctx.wall_speed[0])
                                : (high ? ctx.wall_speed[3] : ctx.wall_speed[2]);
    wb.v[0] = axis == 0 ? 0.0 : ws;
    wb.v[1] = axis == 0 ? ws : 0.0;
    wb.v[3] = axis == 0 ? (high ? ctx.wall_theta[1] : ctx.wall_theta[0])
                        : (high ? ctx.wall_theta[3] : ctx.wall_theta[2]);
    if (!(wb.v[3] > 0.0)) {
      fail = W_PROJ_SPREAD;
      branch = B_NONE;
    } else {
      rs = sqrt(wb.v[3]);
    }
  } else if (branch == B_HALF) {
    const double ul = (axis == 0 ? lp.v[0] : lp.v[1]) + L[(1 + axis) * SPV] * (1.0 / L[0]);
    const double ur = (axis == 0 ? rp.v[0] : rp.v[1]) + U[(1 + axis) * SPV] * (1.0 / U[0]);
    const double cl = ctx.c_bound * sqrt(rep_theta32(L, lp));
    const double cr = ctx.c_bound * sqrt(rep_theta32(U, rp));
    const double lminus = tc::smin(ul - cl, ur - cr);
    const double lplus = tc::smax(ul + cl, ur + cr);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) fp.v[qq] = 0.5 * (lp.v[qq] + rp.v[qq]);
    if (!(fp.v[3] > 0.0)) {
      fail = W_PROJ_SPREAD;
      branch = B_NONE;
    } else if (lminus >= 0.0) {
      branch = B_FULL_L;
    } else if (lplus <= 0.0) {
      branch = B_FULL_R;
    }
    rs = fp.v[3] > 0.0 ? sqrt(fp.v[3]) : 1.0;
  }
  // ---- phase 2: project the state(s) into the face (or wall) basis
  {
    const bool wall = branch == B_WALL;
    project2<M>(g, q, L, wall ? cp : lp, wall ? wb : fp, wall || branch == B_HALF || branch == B_FULL_L,
                U, rp, fp, branch == B_HALF || branch == B_FULL_R);
  }
  if (stamp) stamp[1] = gtimer0();
  // ---- phase 3: flux in the face basis into F (per-partition K columns)
  double kin0[M + 1];
  {
    const double un = branch == B_WALL ? 0.0 : (axis == 0 ? fp.v[0] : fp.v[1]);
    // one erfc / exp per face, shared by the 8 partition x axis flux bodies
    const tc::HalfBase hb = tc::half_base(un, rs);
    if (axis == 0) {
#define SP_FQ(Q) flux_q<M, 0, Q>(branch, high, un, rs, hb, fp, L, U, F, kin0)
      SP_DISPATCH(q, SP_FQ)
#undef SP_FQ
    } else {
#define SP_FQ(Q) flux_q<M, 1, Q>(branch, high, un, rs, hb, fp, L, U, F, kin0)
      SP_DISPATCH(q, SP_FQ)
#undef SP_FQ
    }
  }
  gbar(g);
  if (stamp) stamp[2] = gtimer0();
  // wall closure: density of the incoming wall Maxwellian (flux.cpp:119-129)
  if (branch == B_WALL && q == 0) {
    const double in0 = kin0[0];
    const double wall_rho = in0 == 0.0 ? 0.0 : -F[0] / in0;
    if (in0 == 0.0) {
      fail = W_WALL_DEGEN;
    } else if (!(wall_rho > 0.0)) {
      fail = W_WALL_RHO;
    } else {
#pragma unroll
      for (int p = 1; p <= M; ++p) {
        const int k = axis == 0 ? flat3(p, 0, 0) : flat3(0, p, 0);
        F[k * SPV] = fma(wall_rho, kin0[p], F[k * SPV]);
      }
      F[0] = 0.0;
    }
  }
  gbar(g);
  // ---- phase 4: flux back into the cell basis (in F)
  const P4 from = branch == B_WALL ? wb : fp;
  project1<M>(g, q, F, from, cp, branch != B_NONE);
  return fail;
}


// ------------------------------------------------------------- cell update
// sweep_cell (single_level.cpp:103-111): local dt, residual assembly
// (spatial.cpp:127-132), rhs projection (update_delta :64-70), the update and
// grad_normalize with the dt/2 retry (apply_update :44-62); face group 0.
// Per-cell scalars of the update from the cell's current state S (lane's
// column, stride SPV) and basis cp: local_dt (single_level.cpp:18-29), the
// collision frequency (collision.hpp:36-44) and, for Shakhov, the heat flux
// of extract_macro (moment_rep.hpp:134-144).  Returns the failure kind.
__device__ __forceinline__ int cell_scalars(const DevCtx& ctx, const double* S, const P4& cp, double dxi,
                                            double dyj, double* dt, double* nu, double* qv) {
  if (!(cp.v[3] > 0.0)) return W_DT_THETA;
  const double cc = ctx.cfl_c_bound * sqrt(cp.v[3]);
  *dt = ctx.cfl / ((fabs(cp.v[0]) + cc) / dxi + (fabs(cp.v[1]) + cc) / dyj);
  const double rho = S[0];
  if (!(rho > 0.0)) return W_MACRO_RHO;
  if (ctx.collision == 1) return W_ES_UNSUPPORTED;
  *nu = ctx.nu_coef * rho * pow(cp.v[3], ctx.nu_exp);
  if (ctx.collision == 2) {
    qv[0] = 2.0 * S[flat3(3, 0, 0) * SPV] + S[flat3(3, 0, 0) * SPV] + S[flat3(1, 2, 0) * SPV] + S[flat3(1, 0, 2) * SPV];
    qv[1] = 2.0 * S[flat3(0, 3, 0) * SPV] + S[flat3(2, 1, 0) * SPV] + S[flat3(0, 3, 0) * SPV] + S[flat3(0, 1, 2) * SPV];
    qv[2] = 2.0 * S[flat3(0, 0, 3) * SPV] + S[flat3(2, 0, 1) * SPV] + S[flat3(0, 2, 1) * SPV] + S[flat3(0, 0, 3) * SPV];
  }
  return W_NONE;
}
// layout of a precomputed scalar block: value t of lane c at pre[t * 32 + c]
enum : int { PRE_DT = 0, PRE_NU = 1, PRE_Q0 = 2, PRE_FAIL = 5, PRE_IDX = 6, PRE_IDY = 7, PRE_N = 8 };

template <int M>
__device__ __forceinline__ int update_split(const DevField& f, const DevField* rhs, const DevCtx& ctx,
                                            int q, bool valid, int i, int j, double* base, double* bad,
                                            P4 cp, double dxi, double dyj, P4* new_p = nullptr,
                                            unsigned long long* dbg = nullptr, const double* pre = nullptr,
                                            int* ok_out = nullptr, bool assembled = false) {
  // dbg (one thread, debug): [0] step start; accumulators [8] scalars,
  // [9] assembled, [10] normalize iterations, [11] normalized, [12] written
#define US_STAMP(slot) \
  if (dbg) dbg[slot] += gtimer0() - dbg[0]
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3, VEC = Layout<M>::VEC;
  const int c = threadIdx.x & 31;
  double* S = base + 12 * VEC + c;      // SB (staged in the face phase)
  double* RH = base + 13 * VEC + c;     // RB
  double* V = base + 3 * VEC + c;       // L_1
  double* D = base + 4 * VEC + c;       // U_1
  const double* Fxm = base + 2 * VEC + c;
  const double* Fxp = base + 5 * VEC + c;
  const double* Fym = base + 8 * VEC + c;
  const double* Fyp = base + 11 * VEC + c;
  int klo, khi;
  krange<M>(q, &klo, &khi);
  const size_t cell = (size_t)j * f.nx + i;
  P4 rp{};
  if (valid && rhs) rp = tc::ldp<true>(rhs->p + cell * 4);
  int fail = W_NONE;
  double dt = 0.0, nu = 0.0, qv[3] = {0.0, 0.0, 0.0};
  if (valid) {
    if (pre) {  // computed ahead from the same cell state (band sweep)
      dt = pre[PRE_DT * 32];
      nu = pre[PRE_NU * 32];
      qv[0] = pre[PRE_Q0 * 32];
      qv[1] = pre[PRE_Q0 * 32 + 32];
      qv[2] = pre[PRE_Q0 * 32 + 64];
      fail = (int)pre[PRE_FAIL * 32];
    } else {
      fail = cell_scalars(ctx, S, cp, dxi, dyj, &dt, &nu, qv);
    }
  }
  US_STAMP(8);
  if (rhs) project1<M>(0, q, RH, rp, cp, valid && fail == W_NONE);
  const bool ok0 = valid && fail == W_NONE;
  if (!assembled) {  // (the band sweep assembles on 8 warps before calling)
    if (ok0) {
      const double idx = pre ? pre[PRE_IDX * 32] : 1.0 / dxi, idy = pre ? pre[PRE_IDY * 32] : 1.0 / dyj;
      const int shk = ctx.collision == 2;
      const double shw = ctx.shakhov_w;
      const bool hr = rhs != nullptr;
#define SP_AS(Q) Part<M, Q>::assemble(S, RH, Fxm, Fxp, Fym, Fyp, nu, shk, shw, qv, idx, idy, dt, hr, D, V)
      SP_DISPATCH(q, SP_AS)
#undef SP_AS
    }
    gbar(0);
  }
  US_STAMP(9);
  // apply_update with the dt/2 retry; grad_normalize loop uniform per group
  bool done = !ok0;
  bool good = false;
  P4 prm = cp;
  for (int attempt = 0; attempt < 2; ++attempt) {
    bool active = !done;
    int status = W_NONE;
    prm = cp;
    if (attempt == 1 && active) {
      const double half = 0.5 * dt;
#define SP_RS(Q) Part<M, Q>::restep(S, D, half, V)
      SP_DISPATCH(q, SP_RS)
#undef SP_RS
    }
    // at attempt 0 the barrier after the assembly already ordered V
    if (attempt == 1) gbar(0);
    for (int iter = 0; iter <= 30; ++iter) {
      bool need = false;
      P4 to = prm;
      if (active) {
        const double rho = V[0];
        if (!isfinite(rho) || !(rho > 0.0)) {
          status = W_GRAD_RHO;
          *bad = rho;
          active = false;
        } else if (grad_defect32(V) <= 1e-12) {
          active = false;
        } else if (iter == 30) {
          status = W_GRAD_CAP;
          active = false;
        } else {
          to.v[0] = rep_u32(V, prm, 0);
          to.v[1] = rep_u32(V, prm, 1);
          to.v[2] = rep_u32(V, prm, 2);
          to.v[3] = rep_theta32(V, prm);
          if (!isfinite(to.v[3]) || !(to.v[3] > 0.0)) {
            status = W_GRAD_THETA;
            *bad = to.v[3];
            active = false;
          } else if (!isfinite(to.v[0]) || !isfinite(to.v[1]) || !isfinite(to.v[2])) {
            status = W_GRAD_U;
            active = false;
          } else {
            need = true;
          }
        }
      }
      if (!gbar_or(0, need)) break;
      if (dbg) dbg[10] += 1;
      project1<M>(0, q, V, prm, to, need);
      if (need) prm = to;
    }
    if (!done) {
      const bool nonphys = status == W_GRAD_RHO || status == W_GRAD_THETA || status == W_GRAD_U;
      if (status == W_NONE) {
        good = true;
        done = true;
      } else if (nonphys) {
        if (attempt == 1) {  // SolverError after the dt/2 retry
          fail = W_DT_HALVING;
          done = true;
        }
      } else {  // plain Error (iteration cap) propagates
        fail = status;
        done = true;
      }
    }
    if (!gbar_or(0, !done)) break;
  }
  US_STAMP(11);
  // coalesced write-back: warp q stores cells 8q..8q+7, lane = coefficient
  // (ok_out: the caller stores V later; only the per-cell flag is returned)
  if (ok_out) {
    if (q == 0) ok_out[threadIdx.x & 31] = valid && fail == W_NONE && good;
  } else {
    const int lane = threadIdx.x & 31;
    const bool ok = valid && fail == W_NONE && good;
    if (ok && q == 0) {
      __stcg(reinterpret_cast<double2*>(f.p + cell * 4), make_double2(prm.v[0], prm.v[1]));
      __stcg(reinterpret_cast<double2*>(f.p + cell * 4) + 1, make_double2(prm.v[2], prm.v[3]));
    }
    const double* Vb = V - lane;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int cc = 8 * q + t;
      const int okc = __shfl_sync(0xffffffffu, ok ? 1 : 0, cc);
      const long long bc = __shfl_sync(0xffffffffu, (long long)cell, cc);
      if (!okc) continue;
      double* dst = f.c + (size_t)bc * NP;
#pragma unroll
      for (int h = 0; h < (N + 31) / 32; ++h) {
        const int k = lane + 32 * h;
        if (k < N) __stcg(dst + k, Vb[k * SPV + cc]);
      }
    }
    // no fence here: the caller publishes the cells with st.release after a
    // CTA barrier, which orders every thread's write-back (cumulativity)
  }
  if (new_p) *new_p = prm;
  US_STAMP(12);
#undef US_STAMP
  return (valid && !good && fail == W_NONE) ? W_DT_HALVING : fail;
}


__device__ __forceinline__ unsigned long long gtimer() {
#ifdef TRACE_CLOCK  // SM cycle counter scaled to ns at 1965 MHz (per-SM, not global)
  return (unsigned long long)clock64() * 1000ull / 1965ull;
#else
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
#endif
}

}  // namespace sp
}  // namespace momg_gpu
