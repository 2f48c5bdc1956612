// Band-persistent exact fast sweep for second order and/or an FAS
// right-hand side (k6_band; M <= 5).  Same schedule and dependency rule as
// k5_band (band_sweep.cuh): one CTA walks a band of B2W = 16 rotated columns
// of one sweep diagonal by diagonal, tasks in (sweep, band) order.  What
// changes is the stencil: the second-order face states (spatial.cpp:34-80)
// reach two cells along each axis, and coarse levels subtract the projected
// right-hand side (single_level.cpp:64-70).  So every state the step needs
// is kept on chip in rings indexed by diagonal:
//   OLD ring (4): old states of diagonals d .. d+3 (d+3 prefetched at step d)
//   NEW ring (3): new states of d-2, d-1 and d (written by the update)
//   RHS ring (2): rhs of d and d+1 (prefetched)
// A ring vector has 20 slots, slot s+2 for rotated column 16k+s: old
// vectors hold s = 0..17 (the two columns of band k+1 for the downstream
// faces), new vectors s = -2..15 (the two columns of band k-1, polled on
// their per-cell counters: the band-to-band halo).
//
// This header is compiled with SPV = 21 (element stride of every vector, odd:
// bank-conflict free both lane = cell and lane = coefficient), in its own
// translation units (band2_m<M>.cu), so the vectors of 16 cells are 40%
// smaller than k5_band's 33-slot ones.
#pragma once

#include "kernels_v3.cuh"
#include "band_sweep.cuh"
#include "band2.h"

namespace momg_gpu {
namespace sp {

constexpr int B2W = 16;  // columns per band task
static_assert(SPV >= 20, "band2 vectors need 20 slots (compile with SPV=21)");


template <int M>
struct Band2Layout {
  static constexpr int N = Gen<M>::N;
  static constexpr int VEC = N * SPV;
  // vectors: 0..11 face groups (L, U, F), 12..15 OLD ring, 16..18 NEW ring,
  // 19..20 RHS ring, 21 D (update delta for the dt/2 retry)
  static constexpr int V_OLD = 12, V_NEW = 16, V_RHS = 19, V_D = 21, NV = 22;
  static constexpr int PO = NV * VEC;      // OLD ring params [4][20][4]
  static constexpr int PN = PO + 4 * 80;   // NEW ring params [3][20][4]
  static constexpr int PR = PN + 3 * 80;   // RHS ring params [2][16][4]
  static constexpr int PRE = PR + 2 * 64;  // 2 blocks [PRE_N][32] of update scalars
  static constexpr size_t bytes = (size_t)(PRE + 2 * PRE_N * 32) * sizeof(double);
};

// ring slots of diagonal dd
template <int M>
__device__ __forceinline__ double* b2_old(double* smem, int dd) {
  return smem + (Band2Layout<M>::V_OLD + (dd & 3)) * Band2Layout<M>::VEC;
}
template <int M>
__device__ __forceinline__ double* b2_new(double* smem, int dd) {
  return smem + (Band2Layout<M>::V_NEW + (dd + 3) % 3) * Band2Layout<M>::VEC;  // dd >= -2
}
template <int M>
__device__ __forceinline__ double* b2_oldp(double* smem, int dd) {
  return smem + Band2Layout<M>::PO + (dd & 3) * 80;
}
template <int M>
__device__ __forceinline__ double* b2_newp(double* smem, int dd) {
  return smem + Band2Layout<M>::PN + ((dd + 3) % 3) * 80;
}

// Cell update of face group 0 (update_split, single_level.cpp:44-70 and
// projection.hpp:96-121) on explicit vectors: S the cell state, RH the rhs
// (projected in place into the cell basis), V the new state, D the delta.
template <int M>
__device__ __forceinline__ int b2_update(const DevCtx& ctx, int q, bool valid, bool has_rhs, double* S, double* RH,
                                         const P4& rp, double* V, double* D, const double* Fxm, const double* Fxp,
                                         const double* Fym, const double* Fyp, const P4& cp, const double* pre,
                                         double* bad, P4* new_p) {
  int fail = valid ? (int)pre[PRE_FAIL * 32] : W_NONE;
  const double dt = pre[PRE_DT * 32], nu = pre[PRE_NU * 32];
  const double qv[3] = {pre[PRE_Q0 * 32], pre[PRE_Q0 * 32 + 32], pre[PRE_Q0 * 32 + 64]};
  if (has_rhs) project1<M>(0, q, RH, rp, cp, valid && fail == W_NONE);
  const bool ok0 = valid && fail == W_NONE;
  if (ok0) {
    const double idx = pre[PRE_IDX * 32], idy = pre[PRE_IDY * 32];
    const int shk = ctx.collision == 2;
    const double shw = ctx.shakhov_w;
#define B2_AS(Q) Part<M, Q>::assemble(S, RH, Fxm, Fxp, Fym, Fyp, nu, shk, shw, qv, idx, idy, dt, has_rhs, D, V)
    SP_DISPATCH(q, B2_AS)
#undef B2_AS
  }
  gbar(0);
  bool done = !ok0, good = false;
  P4 prm = cp;
  for (int attempt = 0; attempt < 2; ++attempt) {
    bool active = !done;
    int status = W_NONE;
    prm = cp;
    if (attempt == 1 && active) {
      const double half = 0.5 * dt;
#define B2_RS(Q) Part<M, Q>::restep(S, D, half, V)
      SP_DISPATCH(q, B2_RS)
#undef B2_RS
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
      project1<M>(0, q, V, prm, to, need);
      if (need) prm = to;
    }
    if (!done) {
      const bool nonphys = status == W_GRAD_RHO || status == W_GRAD_THETA || status == W_GRAD_U;
      if (status == W_NONE) {
        good = true;
        done = true;
      } else if (nonphys) {
        if (attempt == 1) {
          fail = W_DT_HALVING;
          done = true;
        }
      } else {
        fail = status;
        done = true;
      }
    }
    if (!gbar_or(0, !done)) break;
  }
  *new_p = prm;
  return (valid && !good && fail == W_NONE) ? W_DT_HALVING : fail;
}

template <int M, bool ST = false>
__global__ void __launch_bounds__(THREADS, 1) k6_band(DevField f, DevField rhsf, DevCtx ctx, DevErr* err,
                                                      Band2Plan plan) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int s_task, s_stop;
  __shared__ int s_ok[32];
  using LY = Band2Layout<M>;
  constexpr int VEC = LY::VEC;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, g = warp / P, q = warp % P, c = tid & 31;
  const int ntasks = plan.nsweeps * plan.nk;
  const CellAddr<ST> fa{plan.strips, f.c, f.p, plan.ver};
  const CellAddr<> ra{nullptr, rhsf.c, rhsf.p, plan.ver};
  const unsigned ep = plan.epoch;  // counters count from here (0: zeroed per launch)
  const bool sys = ST && plan.sys != 0;
  const bool has_rhs = !ST && plan.has_rhs != 0;
  const bool o2 = plan.order == 2;
  for (;;) {
    if (tid == 0) {
      sched_jitter(plan.jitter, 1u);
      s_task = (int)atomicAdd(plan.next, 1u);
      s_stop = band_stop(err);
    }
    __syncthreads();
    const int task = s_task;
    if (task >= ntasks || s_stop) return;
    const int s = task / plan.nk;
    const int dir = (int)((plan.dirbits >> (2 * s)) & 3u);
    const int frame = dir == 0 || dir == 3 ? 0 : 1;
    const int k = plan.korder ? (int)plan.korder[frame * plan.nbands + task % plan.nk]
                              : (frame == 0 ? plan.kb_up : plan.kb_dn) + task % plan.nk;
    // blocked mode: a block-start band's 2-column halo is OLD, a block-end
    // band's next two columns (slots B2W, B2W + 1) are NEW
    const int bfl = plan.bflags ? (int)plan.bflags[frame * plan.nbands + k] : 0;
    const unsigned hneed = (bfl & 1) ? 0u : 1u;
    const int hi_slot = (bfl & 2) ? B2W + 2 : 1 << 30;  // (old-ring slot index: +2 for the halo slots)
    BandGeo<ST> b;
    b.nx = f.nx;
    b.ny = f.ny;
    b.k = k;
    b.bw = B2W;
    b.i_up = dir == 0 || dir == 3;  // kSweepDirs (single_level.cpp:116-117)
    b.j_up = dir == 0 || dir == 1;
    b.st = plan.strips;
    b.strips_init();
    const int ir = B2W * k + c;
    const int dfirst = B2W * k, dlast = min(B2W * k + B2W - 1, f.nx - 1) + f.ny - 1;
    // ---- prologue: old states of dfirst .. dfirst+2, band k-1's new states
    // of dfirst-1 and dfirst-2, the rhs of dfirst; then the update scalars
#pragma unroll 1
    for (int t = 0; t < 3; ++t)
      band_load<M, 2>(fa, b, dfirst + t, 0, 18, ep + (unsigned)s, b2_old<M>(smem, dfirst + t) + 2, SPV,
                      b2_oldp<M>(smem, dfirst + t) + 8, warp, 16, err, kPrologueSleepNs, 0u, sys, hi_slot - 2,
                      ep + (unsigned)s + 1u);
    if (k > 0 && warp >= 14)
      band_load<M, 2>(fa, b, dfirst - 1 - (warp - 14), -2, 2, ep + (unsigned)s + hneed,
                      b2_new<M>(smem, dfirst - 1 - (warp - 14)), SPV, b2_newp<M>(smem, dfirst - 1 - (warp - 14)),
                      0, 1, err, kPrologueSleepNs, 0u, sys);
    if (has_rhs)
      band_load<M, 1>(ra, b, dfirst, 0, B2W, 0u, smem + (LY::V_RHS + (dfirst & 1)) * VEC, SPV,
                      smem + LY::PR + (dfirst & 1) * 64, warp, 16, err, 0);
    __syncthreads();
    if (warp == 4)
      band_pre<M, B2W>(f, ctx, b, dfirst, b2_old<M>(smem, dfirst) + 2, b2_oldp<M>(smem, dfirst) + 8,
                       smem + LY::PRE + (dfirst & 1) * PRE_N * 32);
    __syncthreads();
    for (int d = dfirst; d <= dlast; ++d) {
      // ---- (A) write-back of step d-1, then the face states of group g
      if (d > dfirst)
        band_writeback<M>(fa, b, d - 1, b2_new<M>(smem, d - 1) + 2, b2_newp<M>(smem, d - 1) + 8, s_ok, warp);
      const int jr = d - ir;
      const bool valid = c < B2W && ir < f.nx && jr >= 0 && jr < f.ny;
      const int i = valid ? (b.i_up ? ir : f.nx - 1 - ir) : 0;
      const int j = valid ? (b.j_up ? jr : f.ny - 1 - jr) : 0;
      P4 cp, lp, rp;
      int branch = B_NONE;
      {
        const int axis = g >> 1;
        const bool high = g & 1;
        const bool up = axis == 0 ? b.i_up : b.j_up;  // original +1 = rotated +1
        const int n = axis == 0 ? f.nx : f.ny, pos = axis == 0 ? i : j;
        // original offsets of the face's cells: ll, l (lower), u (upper), uu
        const int oL = high ? 0 : -1;
        // (vector, params) of the cell at original offset o along the axis
        auto at = [&](int o, const double** v, const double** pp) {
          const int dl = up ? o : -o;  // rotated offset
          const int dd = d + dl, slot = (axis == 0 ? c + dl : c) + 2;
          const double* base = dl < 0 ? b2_new<M>(smem, dd) : b2_old<M>(smem, dd);
          const double* pb = dl < 0 ? b2_newp<M>(smem, dd) : b2_oldp<M>(smem, dd);
          *v = base + slot;
          *pp = pb + slot * 4;
        };
        const double *vs, *ps;
        at(0, &vs, &ps);
#pragma unroll
        for (int t = 0; t < 4; ++t) cp.v[t] = ps[t];
        const bool at_wall = high ? pos == n - 1 : pos == 0;
        double* L = smem + (g * 3) * VEC + c;
        double* U = L + VEC;
        if (valid && at_wall) {
          branch = B_WALL;
          lp = cp;
          rp = cp;
#define B2_CP(Q) Part<M, Q>::copy(vs, L)
          SP_DISPATCH(q, B2_CP)
#undef B2_CP
        } else if (valid) {
          branch = B_HALF;
          const int pl = pos + oL, pu = pl + 1;
          const bool rl = o2 && pl > 0 && pl < n - 1;
          const bool ru = o2 && pu > 0 && pu < n - 1;
          const double *vl, *pl4, *vu, *pu4, *vll = nullptr, *pll4 = nullptr, *vuu = nullptr, *puu4 = nullptr;
          at(oL, &vl, &pl4);
          at(oL + 1, &vu, &pu4);
          if (rl) at(oL - 1, &vll, &pll4);
          if (ru) at(oL + 2, &vuu, &puu4);
          P4 pL, pU;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            pL.v[t] = pl4[t];
            pU.v[t] = pu4[t];
          }
          lp = pL;
          rp = pU;
          // safe_face_state (spatial.cpp:64-80): reconstruct unless the face
          // temperature would be nonpositive (same arithmetic as face_split)
          const double* xc = axis == 0 ? f.xc : f.yc;
          const double* ddx = axis == 0 ? f.dx : f.dy;
          double aL = 0.0, aU = 0.0;
          bool recl = false, recu = false;
          // one reciprocal per slope denominator (no divisions on the
          // staging path; single-rounding differences from face_split)
          if (rl) {
            const double ihl = 1.0 / (xc[pl + 1] - xc[pl - 1]), offL = 0.5 * ddx[pl];
            P4 w;
#pragma unroll
            for (int t = 0; t < 4; ++t) w.v[t] = pL.v[t] + offL * ((pU.v[t] - pll4[t]) * ihl);
            if (w.v[3] > 0.0) {
              recl = true;
              lp = w;
              aL = offL * ihl;
            }
          }
          if (ru) {
            const double ihu = 1.0 / (xc[pu + 1] - xc[pu - 1]), offU = -0.5 * ddx[pu];
            P4 w;
#pragma unroll
            for (int t = 0; t < 4; ++t) w.v[t] = pU.v[t] + offU * ((puu4[t] - pL.v[t]) * ihu);
            if (w.v[3] > 0.0) {
              recu = true;
              rp = w;
              aU = offU * ihu;
            }
          }
          const int klo = (q * Gen<M>::N) / P, khi = ((q + 1) * Gen<M>::N) / P;
          for (int kk = klo; kk < khi; ++kk) {
            const double l = vl[kk * SPV], u = vu[kk * SPV];
            L[kk * SPV] = recl ? fma(aL, u - vll[kk * SPV], l) : l;
            U[kk * SPV] = recu ? fma(aU, vuu[kk * SPV] - l, u) : u;
          }
        }
      }
      __syncthreads();
      // ---- (B) face fluxes
      {
        double* L = smem + (g * 3) * VEC + c;
        const int w = face_core<M>(ctx, g, q, g >> 1, g & 1, branch, W_NONE, lp, rp, cp, L, L + VEC, L + 2 * VEC,
                                   nullptr);
        if (w && valid && q == 0) tc::raise(err, tc::code_for(w), w, i, j, 0.0);
      }
      __syncthreads();
      // ---- (C) group 0: the cell update into NEW(d); groups 1-3: publish
      // d-1, prefetch old(d+3), rhs(d+1), band k-1's new(d), scalars of d+1
      if (g == 0) {
        double bad = 0.0;
        P4 np = cp, rpp{};
        if (has_rhs && valid) {
#pragma unroll
          for (int t = 0; t < 4; ++t) rpp.v[t] = smem[LY::PR + (d & 1) * 64 + c * 4 + t];
        }
        double* S = b2_old<M>(smem, d) + 2 + c;
        const int w = b2_update<M>(ctx, q, valid, has_rhs, S, smem + (LY::V_RHS + (d & 1)) * VEC + c, rpp,
                                   b2_new<M>(smem, d) + 2 + c, smem + LY::V_D * VEC + c, smem + 2 * VEC + c,
                                   smem + 5 * VEC + c, smem + 8 * VEC + c, smem + 11 * VEC + c, cp,
                                   smem + LY::PRE + (d & 1) * PRE_N * 32 + c, &bad, &np);
        if (w && valid && q == 0) tc::raise(err, tc::code_for(w), w, i, j, bad);
        if (q == 0) {
          s_ok[c] = valid && w == W_NONE;
          if (c < B2W) {
            double* pn = b2_newp<M>(smem, d) + (c + 2) * 4;
#pragma unroll
            for (int t = 0; t < 4; ++t) pn[t] = np.v[t];
          }
        }
      } else {
        const int wi = warp - 4;
        const int stop_now = tid == 128 ? band_stop(err) : 0;
        if (wi == 0 && d > dfirst && c < B2W) {
          sched_jitter(plan.jitter, (unsigned)d);
          const int cl = b.cell(c, d - 1);
          if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, sys);
        }
        if (wi < 6 && d + 1 <= dlast)
          band_load<M, 3>(fa, b, d + 3, 0, 18, ep + (unsigned)s, b2_old<M>(smem, d + 3) + 2, SPV,
                          b2_oldp<M>(smem, d + 3) + 8, wi, 6, err, plan.poll_ns, plan.jitter, sys, hi_slot - 2,
                          ep + (unsigned)s + 1u);
        if (has_rhs && wi >= 6 && wi < 10 && d + 1 <= dlast)
          band_load<M, 4>(ra, b, d + 1, 0, B2W, 0u, smem + (LY::V_RHS + ((d + 1) & 1)) * VEC, SPV,
                          smem + LY::PR + ((d + 1) & 1) * 64, wi - 6, 4, err, 0);
        if (wi == 10 && d + 1 <= dlast)
          band_pre<M, B2W>(f, ctx, b, d + 1, b2_old<M>(smem, d + 1) + 2, b2_oldp<M>(smem, d + 1) + 8,
                           smem + LY::PRE + ((d + 1) & 1) * PRE_N * 32);
        if (k > 0 && wi == 11 && d + 1 <= dlast)
          band_load<M, 2>(fa, b, d, -2, 2, ep + (unsigned)s + hneed, b2_new<M>(smem, d), SPV, b2_newp<M>(smem, d),
                          0, 1, err, plan.poll_ns, plan.jitter, sys);
        if (tid == 128) s_stop = stop_now;
      }
      __syncthreads();
      if (s_stop) return;
    }
    band_writeback<M>(fa, b, dlast, b2_new<M>(smem, dlast) + 2, b2_newp<M>(smem, dlast) + 8, s_ok, warp);
    __syncthreads();
    if (warp == 4 && c < B2W) {
      const int cl = b.cell(c, dlast);
      if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, sys);
    }
  }
}

}  // namespace sp

// host launcher, one per moment order (band2_m<M>.cu)
template <int M>
void band2_launch_impl(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err,
                       const sp::Band2Plan& plan, cudaStream_t st) {
  static int nsm = 0;
  if (!nsm) {
    cudaFuncSetAttribute(sp::k6_band<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sp::Band2Layout<M>::bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int nb = nsm;  // one CTA per SM (smem-bound); tasks are claimed dynamically
  if (nb > plan.nsweeps * plan.nk) nb = plan.nsweeps * plan.nk;
  sp::k6_band<M><<<nb, sp::THREADS, sp::Band2Layout<M>::bytes, st>>>(f, rhs, ctx, err, plan);
}
template <int M>
void band2_strips_launch_impl(const DevField& geo, const DevCtx& ctx, DevErr* err, const sp::Band2Plan& plan,
                              cudaStream_t st) {
  static int nsm = 0;
  if (!nsm) {
    cudaFuncSetAttribute(sp::k6_band<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sp::Band2Layout<M>::bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int nb = nsm;
  if (nb > plan.nsweeps * plan.nk) nb = plan.nsweeps * plan.nk;
  sp::k6_band<M, true><<<nb, sp::THREADS, sp::Band2Layout<M>::bytes, st>>>(geo, geo, ctx, err, plan);
}

}  // namespace momg_gpu
