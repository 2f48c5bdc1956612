// Register-resident band sweep: first order, M <= 5, BGK / Shakhov, no rhs,
// one flat field, exact order (threads = 1).  Same schedule as k5_band
// (band_sweep.cuh: a task = one sweep x one band of 32 rotated columns walked
// diagonal by diagonal, tasks claimed in (sweep, band) order, per-cell
// counters, band k-1's halo cell polled), different cell math.
//
// k5_band splits each face 4 ways across warps and moves every axis pass
// through shared memory (~55 vector round trips and ~24 named barriers per
// step at 128 registers per thread), which keeps the SM's FP64 pipe ~12% busy
// (DESIGN.md sec. 5).  Here one THREAD evaluates one side of one face with
// the whole moment vector in registers (the transfer kernels' stride-1
// generated passes, transfer.cuh): 8 warps = 4 faces x {cell side,
// neighbour side}, lane = cell of the diagonal.  A side projects its state
// into the face (or wall) basis, applies its half of the half-range flux
// (flux.cpp:29-75: left side the upper kernel, right side the lower; one
// side alone on the supersonic full-flux branches, flux.cpp:91-92; the wall
// closure flux.cpp:105-130 on the cell side), projects the result back into
// the cell basis and stores it once.  The residual assembly (spatial.cpp:
// 127-132) is split by coefficient over the 8 warps; the update (local dt,
// f + dt delta, grad_normalize with the dt/2 retry, single_level.cpp:44-62,
// 103-111) runs on warp 0 in registers while the other warps publish, load
// diagonal d+2 and compute the next update's scalars.  Per step: three CTA
// barriers and ~20 shared-memory vector passes (k5_band: ~24 named + 3 CTA
// barriers, ~55 passes).
//
// numerics: project(F_left + F_right) = project(F_left) + project(F_right)
// (projection is linear); the two halves are summed after the back
// projection instead of before it (one rounding apart, well inside the
// 1e-10 parity tolerance).
#pragma once

#include "band_sweep.cuh"
#include "transfer.cuh"

#include <utility>

namespace momg_gpu {
namespace rb {

using sp::BandGeo;
using sp::BandPlan;
using tc::P4;

constexpr int RT = 256;  // threads: 8 warps

template <int M>
struct RLayout {
  static constexpr int N = Gen<M>::N;
  static constexpr int VEC = N * SPV;
  // vectors: O[4] old-state ring (O[d & 3] = old(d), 33 slots: the band's 32
  // columns + band k+1's first; old(d), old(d+1) in use, old(d+2) landed,
  // old(d+3) in flight as cp.async), V[2] new states (V[d & 1]), F[8] face
  // sides (F[0] doubles as the assembled residual D).  Band k-1's halo cell
  // of a diagonal lives in slot 32 of that diagonal's upstream vector (V of
  // the sweep, O of the residual), which is free once the diagonal is upstream.
  static constexpr int V_O = 0, V_V = 4, V_F = 6, NV = 14;
  static constexpr int PO = NV * VEC;      // [4][33][4]
  static constexpr int PV = PO + 4 * 132;  // [2][33][4]
  static constexpr int PRE = PV + 2 * 132;  // [2][PRE_N][32]
  static constexpr size_t bytes = (size_t)(PRE + 2 * sp::PRE_N * 32) * sizeof(double);
};

// One side of the half-range flux kernel (tc::half_kernels_b restricted to
// one side; the pairing-table recurrence of halfspace.hpp:18-57 is shared):
// K[m][p] = rs^(p-m)/p! (u_n P(m,p) + rs P(m+1,p) + rs m P(m-1,p)) with P the
// upper (P+) or lower (P- = m! delta - P+) table.  kin0: row m = 0 of the
// OTHER side (the incoming unit-wall flux of wall_flux).
template <int M>
__device__ __forceinline__ void half_kernel_side(double un, double rs, const tc::HalfBase& hb, bool upper,
                                                 double (&K)[M + 1][M + 1], double (&kin0)[M + 1]) {
  constexpr int P = M + 1;
  const double a = hb.a;
  const double g = hb.g;
  double he[P + 1];
  he[0] = 1.0;
  he[1] = a;
#pragma unroll
  for (int k = 1; k + 1 <= P; ++k) he[k + 1] = a * he[k] - (double)k * he[k - 1];
  const double irs = hb.irs;
  double prev[P + 1];
  double fp = 1.0, rsp = 1.0;
  constexpr double kInvFact[9] = {1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0, 1.0 / 720.0, 1.0 / 5040.0,
                                  1.0 / 40320.0};
#pragma unroll
  for (int p = 0; p <= M; ++p) {
    double col[P + 1];
    col[0] = p == 0 ? hb.e0 : he[p - 1] * g;
    const double hpg = he[p] * g;
#pragma unroll
    for (int m = 0; m + 1 <= P; ++m) {
      const double t = he[m] * hpg;
      col[m + 1] = p > 0 ? fma((double)p, prev[m], t) : t;
    }
    if (p > 0) {
      fp *= (double)p;
      rsp *= rs;
    }
    double scale = rsp * kInvFact[p];
#pragma unroll
    for (int m = 0; m <= M; ++m) {
      // upper table: ku; the lower one is the full-space (tridiagonal) kernel minus ku
      double ku = fma(un, col[m], rs * col[m + 1]);
      if (m > 0) ku = fma(rs * (double)m, col[m - 1], ku);
      double kl = -ku;
      if (m == p) kl = fma(un, fp, -ku);
      else if (m + 1 == p) kl = fma(rs, fp, -ku);
      else if (m - 1 == p) kl = fma(rs * (double)m, fp, -ku);
      K[m][p] = scale * (upper ? ku : kl);
      if (m == 0) kin0[p] = scale * (upper ? kl : ku);
      scale *= irs;
    }
#pragma unroll
    for (int m = 0; m <= P; ++m) prev[m] = col[m];
  }
}

template <int M>
__device__ __forceinline__ void vload(const double* s, double (&v)[Gen<M>::N]) {
#pragma unroll
  for (int k = 0; k < Gen<M>::N; ++k) v[k] = s[k * SPV];
}
template <int M>
__device__ __forceinline__ void vstore(double* s, const double (&v)[Gen<M>::N]) {
#pragma unroll
  for (int k = 0; k < Gen<M>::N; ++k) s[k * SPV] = v[k];
}
__device__ __forceinline__ P4 pload(const double* p) {
  P4 r;
#pragma unroll
  for (int t = 0; t < 4; ++t) r.v[t] = p[t];
  return r;
}

// One side of one face of the lane's cell into F (stride SPV), in the cell
// basis cp; zeros when this side contributes nothing.  `high`: the face is
// the cell's high face along `axis`; side 0 = the cell, 1 = the neighbour.
// Returns the failure kind (reported by side 0).
template <int M>
__device__ __forceinline__ int face_side(const DevCtx& ctx, int axis, bool high, int side, bool valid, bool has_nb,
                                         const double* Sc, const P4& cp, const double* Nb, const P4& np,
                                         double* F) {
  constexpr int N = Gen<M>::N;
  int fail = W_NONE;
  int branch = sp::B_NONE;
  P4 to{};
  double rs = 1.0;
  const bool my_left = side == 0 ? high : !high;  // left = lower-index cell of the face
  if (valid) {
    if (!has_nb) {
      if (side == 0) {
        const double ws = axis == 0 ? (high ? ctx.wall_speed[1] : ctx.wall_speed[0])
                                    : (high ? ctx.wall_speed[3] : ctx.wall_speed[2]);
        to.v[0] = axis == 0 ? 0.0 : ws;
        to.v[1] = axis == 0 ? ws : 0.0;
        to.v[2] = 0.0;
        to.v[3] = axis == 0 ? (high ? ctx.wall_theta[1] : ctx.wall_theta[0])
                            : (high ? ctx.wall_theta[3] : ctx.wall_theta[2]);
        if (!(to.v[3] > 0.0)) fail = W_PROJ_SPREAD;
        else {
          branch = sp::B_WALL;
          rs = sqrt(to.v[3]);
        }
      }
    } else {
      // wave-speed bounds (flux.cpp:79-84) from both states
      const double* L = high ? Sc : Nb;
      const double* R = high ? Nb : Sc;
      const P4& lp = high ? cp : np;
      const P4& rp = high ? np : cp;
      const double ul = (axis == 0 ? lp.v[0] : lp.v[1]) + L[(1 + axis) * SPV] * (1.0 / L[0]);
      const double ur = (axis == 0 ? rp.v[0] : rp.v[1]) + R[(1 + axis) * SPV] * (1.0 / R[0]);
      const double cl = ctx.c_bound * sqrt(sp::rep_theta32(L, lp));
      const double cr = ctx.c_bound * sqrt(sp::rep_theta32(R, rp));
      const double lminus = tc::smin(ul - cl, ur - cr);
      const double lplus = tc::smax(ul + cl, ur + cr);
#pragma unroll
      for (int q = 0; q < 4; ++q) to.v[q] = 0.5 * (lp.v[q] + rp.v[q]);
      if (!(to.v[3] > 0.0)) {
        fail = W_PROJ_SPREAD;
      } else {
        branch = lminus >= 0.0 ? sp::B_FULL_L : (lplus <= 0.0 ? sp::B_FULL_R : sp::B_HALF);
        rs = sqrt(to.v[3]);
        if ((branch == sp::B_FULL_L && !my_left) || (branch == sp::B_FULL_R && my_left)) branch = sp::B_NONE;
      }
    }
  }
  double v[N];
  if (branch == sp::B_NONE) {
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = 0.0;
  } else {
    const bool full = branch == sp::B_FULL_L || branch == sp::B_FULL_R;
    const bool wall = branch == sp::B_WALL;
    const P4 from = side == 0 ? cp : np;
    vload<M>(side == 0 ? Sc : Nb, v);
    xf::project_row<M>(v, from, to);
    // the projected state goes through F (its own slot) once: the flux
    // reads it back pencil by pencil, so the moment vector and the 6x6
    // half-range kernel are never both fully live in registers
    vstore<M>(F, v);
    asm volatile("" ::: "memory");
    if (full) {  // full-space flux xi_n f (flux.cpp:10-27)
      if (axis == 0) Gen<M>::template full_flux0<SPV, 1>(F, v, to.v[0], to.v[3]);
      else Gen<M>::template full_flux1<SPV, 1>(F, v, to.v[1], to.v[3]);
    } else {
      const double un = wall ? 0.0 : (axis == 0 ? to.v[0] : to.v[1]);
      double K[M + 1][M + 1];
      double kin0[M + 1];
      half_kernel_side<M>(un, rs, tc::half_base(un, rs), wall ? high : my_left, K, kin0);
      if (axis == 0) Gen<M>::template half_sr0<SPV, 1>(F, v, K);
      else Gen<M>::template half_sr1<SPV, 1>(F, v, K);
      if (wall) {  // density of the incoming wall Maxwellian (flux.cpp:119-129)
        const double in0 = kin0[0];
        const double wall_rho = in0 == 0.0 ? 0.0 : -v[0] / in0;
        if (in0 == 0.0) fail = W_WALL_DEGEN;
        else if (!(wall_rho > 0.0)) fail = W_WALL_RHO;
#pragma unroll
        for (int p = 1; p <= M; ++p) {
          if (axis == 0) v[flat3(p, 0, 0)] = fma(wall_rho, kin0[p], v[flat3(p, 0, 0)]);
          else v[flat3(0, p, 0)] = fma(wall_rho, kin0[p], v[flat3(0, p, 0)]);
        }
        v[0] = 0.0;
      }
    }
    xf::project_row<M>(v, to, cp);
  }
  vstore<M>(F, v);
  return fail;
}

// Residual assembly of coefficients [K0, K1) of the 32 cells (lane = cell):
// D_k = nu (eq_k - S_k) - (F_xhigh - F_xlow)_k / dx - (F_yhigh - F_ylow)_k / dy
// (spatial.cpp:127-132; collision_coeffs collision.hpp:120-127 with the BGK /
// Shakhov equilibrium in the cell's own basis).  F_*: the two sides' sums.
// Shakhov equilibrium positions 2 e_dd + e_d (collision.hpp:95-111): the q
// component d at position k, or -1
__host__ __device__ constexpr int shakhov_d(int k) {
  for (int d = 0; d < 3; ++d)
    for (int dd = 0; dd < 3; ++dd)
      if (flat3((dd == 0 ? 2 : 0) + (d == 0), (dd == 1 ? 2 : 0) + (d == 1), (dd == 2 ? 2 : 0) + (d == 2)) == k)
        return d;
  return -1;
}

struct AsmArgs {
  const double *S, *Fxh0, *Fxh1, *Fxl0, *Fxl1, *Fyh0, *Fyh1, *Fyl0, *Fyl1;
  double nu, shw, idx, idy, s0;
  bool shk;
  const double* qv;
  double* D;
};
template <int K>
__device__ __forceinline__ void assemble_one(const AsmArgs& a) {
  double eq = K == 0 ? a.s0 : 0.0;
  constexpr int sd = shakhov_d(K);
  if constexpr (sd >= 0) {
    if (a.shk) eq = a.shw * a.qv[sd];
  }
  constexpr int o = K * SPV;
  const double fx = (a.Fxh0[o] + a.Fxh1[o]) - (a.Fxl0[o] + a.Fxl1[o]);
  const double fy = (a.Fyh0[o] + a.Fyh1[o]) - (a.Fyl0[o] + a.Fyl1[o]);
  double r = a.nu * (eq - a.S[o]);
  r -= fx * a.idx;
  r -= fy * a.idy;
  a.D[o] = r;
}
template <int K0, int... I>
__device__ __forceinline__ void assemble_seq(const AsmArgs& a, std::integer_sequence<int, I...>) {
  (assemble_one<K0 + I>(a), ...);
}
template <int M, int K0, int K1>
__device__ __forceinline__ void assemble_range(const double* S, const double* Fxh0, const double* Fxh1,
                                               const double* Fxl0, const double* Fxl1, const double* Fyh0,
                                               const double* Fyh1, const double* Fyl0, const double* Fyl1,
                                               double nu, bool shk, double shw, const double* qv, double idx,
                                               double idy, double* D) {
  const AsmArgs a{S, Fxh0, Fxh1, Fxl0, Fxl1, Fyh0, Fyh1, Fyl0, Fyl1, nu, shw, idx, idy, S[0], shk, qv, D};
  assemble_seq<K0>(a, std::make_integer_sequence<int, K1 - K0>{});
}

template <int M>
__device__ __forceinline__ void assemble_part(int w, const double* S, const double* const* Fp, double nu, bool shk,
                                              double shw, const double* qv, double idx, double idy, double* D) {
  constexpr int N = Gen<M>::N, CH = (N + 7) / 8;
#define RB_AS(W)                                                                                                \
  case W:                                                                                                       \
    assemble_range<M, (W * CH < N ? W * CH : N), ((W + 1) * CH < N ? (W + 1) * CH : N)>(                      \
        S, Fp[0], Fp[1], Fp[2], Fp[3], Fp[4], Fp[5], Fp[6], Fp[7], nu, shk, shw, qv, idx, idy, D);            \
    break;
  switch (w) {
    RB_AS(0)
    RB_AS(1)
    RB_AS(2)
    RB_AS(3)
    RB_AS(4)
    RB_AS(5)
    RB_AS(6)
    RB_AS(7)
  }
#undef RB_AS
}

// Asynchronous variant of sp::band_load: warp wi of nw polls the counters of
// its slots of diagonal dd (one lane per slot), then issues 8-byte cp.async
// copies (lane = coefficient: coalesced in HBM, transposed into
// vec[k * SPV + slot] on the way) and returns without waiting; the caller
// waits (cp_async_wait) before a CTA barrier one step later.  Slots outside
// the grid are zero-filled with plain stores.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Wait until the cell's counter reaches `need`: one acquire load when it
// already has (the common case: one round trip), else relaxed polling with
// back-off and a final acquire.
__device__ __forceinline__ void poll_acquire(const unsigned* a, unsigned need, int cell, int nx, DevErr* err,
                                             int poll_ns) {
  if (ld_acquire_s(a, false) >= need) return;
  long long polls = 0;
  while (ld_relaxed_s(a, false) < need) {
    if (sp::band_stop(err)) break;
    if (++polls > (1LL << 26)) {
      tc::raise(err, E_ERROR, W_DEADLOCK, cell % nx, cell / nx, (double)need);
      break;
    }
    if (poll_ns) __nanosleep(poll_ns);
  }
  (void)ld_acquire_s(a, false);
}

template <int M, int MAXS, class Addr, class Geo>
__device__ __forceinline__ void band_load_async(const Addr& fld, const Geo& b, int dd, int ns, unsigned need,
                                                double* vec, double* prm, int wi, int nw, DevErr* err, int poll_ns,
                                                unsigned jit, unsigned ahead) {
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3, H = (N + 31) / 32;
  const int lane = threadIdx.x & 31;
  int my_cell = -1;
  if (lane < MAXS) {
    const int slot = wi + lane * nw;
    if (slot < ns) my_cell = b.cell(slot, dd);
  }
  if (jit && need) sp::sched_jitter(jit, (unsigned)dd);
  // `ahead`: this lane's counter of diagonal dd as the previous step's acquire load saw it
  if (need && my_cell >= 0 && ahead < need) poll_acquire(fld.vptr(my_cell), need, my_cell, b.nx, err, poll_ns);
  __syncwarp();
#pragma unroll
  for (int t = 0; t < MAXS; ++t) {
    const int slot = wi + t * nw;
    if (slot >= ns) continue;
    const int cl = __shfl_sync(0xffffffffu, my_cell, t);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int kk = lane + 32 * h;
      if (kk < N) {
        if (cl >= 0) cp_async8(vec + kk * SPV + slot, fld.cptr(cl, NP) + kk);
        else vec[kk * SPV + slot] = 0.0;
      }
    }
  }
  // the slots' parameters, eight slots per instruction (4 lanes each)
#pragma unroll
  for (int r = 0; r < (MAXS + 7) / 8; ++r) {
    const int t = 8 * r + (lane >> 2);
    const int slot = wi + t * nw;
    const int cl = __shfl_sync(0xffffffffu, my_cell, t < MAXS ? t : 0);
    if (t < MAXS && slot < ns) {
      if (cl >= 0) cp_async8(prm + slot * 4 + (lane & 3), fld.pptr(cl) + (lane & 3));
      else prm[slot * 4 + (lane & 3)] = 0.0;
    }
  }
}
// the acquire load of a diagonal's counters (the lane -> slot map of
// band_load_async), one step ahead of their use
template <int MAXS, class Addr, class Geo>
__device__ __forceinline__ unsigned band_counters_ahead(const Addr& fld, const Geo& b, int dd, int ns, unsigned need,
                                                        int wi, int nw) {
  const int lane = threadIdx.x & 31;
  unsigned ahead = 0u;
  if (need && lane < MAXS) {
    const int slot = wi + lane * nw;
    const int nc = slot < ns ? b.cell(slot, dd) : -1;
    if (nc >= 0) ahead = ld_acquire_s(fld.vptr(nc), false);
  }
  return ahead;
}

// apply_update (single_level.cpp:44-62) of one cell in registers: f + dt
// delta, grad_normalize, the dt/2 retry; the new state into Vout / PVout.
// Returns the failure kind (W_NONE: ok).  For the large orders this is an
// out-of-line function, so that its 2 N-register vector is allocated apart
// from the kernel's loop-carried state.
template <int M>
__device__ __forceinline__ int cell_update_body(const double* S, const double* D, const double* cpp, double dt,
                                                double* Vout, double* PVout, double* bad, int& tries) {
  constexpr int N = Gen<M>::N;
  double v[N];
  const P4 cp = pload(cpp);
  P4 prm = cp;
  int fail = W_NONE;
  bool good = false;
#pragma unroll 1
  for (int attempt = 0; attempt < 2; ++attempt) {
    const double h = attempt ? 0.5 * dt : dt;
    tries = attempt + 1;
    asm volatile("" ::: "memory");
#pragma unroll
    for (int kk = 0; kk < N; ++kk) v[kk] = S[kk * SPV] + h * D[kk * SPV];
    prm = cp;
    const int st = xf::normalize_row<M, (M <= 5)>(v, prm, bad);
    if (st == W_NONE) {
      good = true;
      break;
    }
    if (st != W_GRAD_RHO && st != W_GRAD_THETA && st != W_GRAD_U) {  // plain Error (cap)
      fail = st;
      break;
    }
    if (attempt == 1) fail = W_DT_HALVING;  // SolverError after the dt/2 retry
  }
  if (fail == W_NONE && good) {
    vstore<M>(Vout, v);
#pragma unroll
    for (int t = 0; t < 4; ++t) PVout[t] = prm.v[t];
  }
  return fail;
}
template <int M>
__device__ __forceinline__ int cell_update_body(const double* S, const double* D, const double* cpp, double dt,
                                                double* Vout, double* PVout, double* bad) {
  int tries = 0;
  return cell_update_body<M>(S, D, cpp, dt, Vout, PVout, bad, tries);
}
template <int M>
__device__ __noinline__ int cell_update_call(const double* S, const double* D, const double* cpp, double dt,
                                             double* Vout, double* PVout, double* bad) {
  return cell_update_body<M>(S, D, cpp, dt, Vout, PVout, bad);
}

// Coalesced write-back of nc cells starting at c0 of diagonal dd (new states
// V[dd & 1], bases PV, only cells whose update succeeded); lane = coefficient.
template <int M, class Geo>
__device__ __forceinline__ void rb_writeback(const DevField& f, const Geo& b, int dd, const double* V,
                                             const double* PV, const int* ok, int c0, int nc) {
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3, H = (N + 31) / 32;
  const int lane = threadIdx.x & 31;
  // the cells' indices by the lanes up front (no dependent chain per cell)
  int mine = -1;
  if (lane < nc && ok[c0 + lane]) mine = b.cell(c0 + lane, dd);
#pragma unroll 2
  for (int t = 0; t < nc; ++t) {
    const int cc = c0 + t;
    const int cl = __shfl_sync(0xffffffffu, mine, t);
    if (cl < 0) continue;
    double* dst = f.c + (size_t)cl * NP;
    double r[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int k = lane + 32 * h;
      r[h] = k < N ? V[k * SPV + cc] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int k = lane + 32 * h;
      if (k < N) __stcg(dst + k, r[h]);
    }
    if (lane < 4) __stcg(f.p + (size_t)cl * 4 + lane, PV[cc * 4 + lane]);
  }
}

// RES = true: the standalone residual (spatial.cpp:135-159): (band, chunk)
// tasks over old states only.  A sweep launch with plan.nchunks > 0 appends
// the residual of its result as (chunk, band) tasks polling the final version.
template <int M, bool RES>
__global__ void __launch_bounds__(RT, 1) k8_band(DevField f, DevCtx ctx, DevErr* err, BandPlan plan, DevField out) {
  constexpr int BW = 32, NS = BW + 1;
  using LY = RLayout<M>;
  constexpr int N = LY::N, VEC = LY::VEC, NP = (N + 3) & ~3;
  extern __shared__ __align__(128) double smem[];
  __shared__ int s_task, s_stop;
  __shared__ int s_ok[2][32];
  // debug trace accumulators: [0] step start, [1] write-back, [2] faces, [3] assembled, [4] updated, [5] end;
  // s_wA: histogram of the step durations; s_wC: per-warp arrival at the end-of-step barrier;
  // s_retry: steps with a dt/2 retry | steps with an update > 3 us << 32; s_b: barrier (B) of the step
  __shared__ unsigned long long s_tr[6], s_wA[8], s_wC[8], s_wM[8], s_retry, s_b;
  const int tid = threadIdx.x, warp = tid >> 5, c = tid & 31;
  const int sweep_tasks = RES ? 0 : plan.nsweeps * plan.nk;
  const int ntasks = sweep_tasks + plan.nchunks * plan.nk;
  const unsigned ep = plan.epoch;
  const unsigned rneed = RES ? 0u : ep + (unsigned)plan.nsweeps;
  const sp::CellAddr<false> fa{nullptr, f.c, f.p, plan.ver};
  double* const O = smem + LY::V_O * VEC;
  double* const PO = smem + LY::PO;
  for (;;) {
    if (tid == 0) {
      sp::sched_jitter(plan.jitter, 1u);
      s_task = (int)atomicAdd(plan.next, 1u);
      s_stop = sp::band_stop(err);
    }
    __syncthreads();
    const int task = s_task;
    if (task >= ntasks || s_stop) return;
    const bool res = task >= sweep_tasks;
    const int rtask = task - sweep_tasks;
    const int s = res ? plan.nsweeps - 1 : task / plan.nk;
    const int dir = (int)((plan.dirbits >> (2 * s)) & 3u);
    const int frame = dir == 0 || dir == 3 ? 0 : 1;
    const int k = (frame == 0 ? plan.kb_up : plan.kb_dn) + (res ? rtask : task) % plan.nk;
    BandGeo<false> b;
    b.nx = f.nx;
    b.ny = f.ny;
    b.k = k;
    b.bw = BW;
    b.i_up = dir == 0 || dir == 3;
    b.j_up = dir == 0 || dir == 1;
    const int ir = BW * k + c;
    int dfirst = BW * k, dlast = min(BW * k + BW - 1, f.nx - 1) + f.ny - 1;
    if (res) {
      dfirst += (rtask / plan.nk) * plan.clen;
      dlast = min(dlast, dfirst + plan.clen - 1);
      if (dfirst > dlast) {
        __syncthreads();
        continue;
      }
    }
    const bool trw = plan.trace && 4 * task + 3 < plan.trace_cap && c == 0;
    const bool tr = trw && tid == 0;
    unsigned long long t0 = 0;
    long long c0 = 0;
    if (trw) {
      s_wA[warp] = s_wC[warp] = s_wM[warp] = 0;
      if (tid == 0)
        for (int q = 0; q < 6; ++q) s_tr[q] = 0;
      if (tid == 0) s_retry = s_b = 0;
    }
    // ---- prologue: warp 0 waits (with back-off) for the first two diagonals
    // and band k-1's halo cell; then O <- old(dfirst), old(dfirst+1), halo
    if (!res && warp == 0) {
      for (int e = c; e < 2 * NS + 1; e += 32) {
        const int cl = e < 2 * NS ? b.cell(e % NS, dfirst + e / NS) : (k > 0 ? b.cell(-1, dfirst - 1) : -1);
        const unsigned need = ep + (unsigned)s + (e < 2 * NS ? 0u : 1u);
        if (cl >= 0 && need) {
          long long polls = 0;
          const unsigned* a = fa.vptr(cl);
          while (ld_relaxed_s(a, false) < need) {
            if (sp::band_stop(err)) break;
            if (++polls > (1LL << 26)) {
              tc::raise(err, E_ERROR, W_DEADLOCK, cl % f.nx, cl / f.nx, (double)need);
              break;
            }
            __nanosleep(sp::kPrologueSleepNs);
          }
          (void)ld_acquire_s(a, false);
        }
      }
    }
    __syncthreads();
    const unsigned pn = res ? rneed : 0u;
    sp::band_load<M, 5>(fa, b, dfirst, 0, NS, pn, O + (dfirst & 3) * VEC, SPV, PO + (dfirst & 3) * 132, warp, 8,
                        err, sp::kPrologueSleepNs);
    sp::band_load<M, 5>(fa, b, dfirst + 1, 0, NS, pn, O + ((dfirst + 1) & 3) * VEC, SPV,
                        PO + ((dfirst + 1) & 3) * 132, warp, 8, err, sp::kPrologueSleepNs);
    sp::band_load<M, 5>(fa, b, dfirst + 2, 0, NS, res ? rneed : ep + (unsigned)s, O + ((dfirst + 2) & 3) * VEC, SPV,
                        PO + ((dfirst + 2) & 3) * 132, warp, 8, err, sp::kPrologueSleepNs);
    if (res)  // a chunk may start mid-band: its upstream states are old(dfirst-1)
      sp::band_load<M, 4>(fa, b, dfirst - 1, 0, BW, pn, O + ((dfirst + 3) & 3) * VEC, SPV,
                          PO + ((dfirst + 3) & 3) * 132, warp, 8, err, sp::kPrologueSleepNs);
    if (k > 0 && warp == 7)
      sp::band_load<M, 1>(fa, b, dfirst - 1, -1, 1, pn,
                          (res ? O + ((dfirst + 3) & 3) * VEC : smem + (LY::V_V + ((dfirst - 1) & 1)) * VEC) + 32,
                          SPV, (res ? PO + ((dfirst + 3) & 3) * 132 : smem + LY::PV + ((dfirst - 1) & 1) * 132) + 128,
                          0, 1, err,
                          sp::kPrologueSleepNs);
    __syncthreads();
    if (warp == 1)
      sp::band_pre<M, BW>(f, ctx, b, dfirst, O + (dfirst & 3) * VEC, PO + (dfirst & 3) * 132,
                          smem + LY::PRE + (dfirst & 1) * sp::PRE_N * 32);
    __syncthreads();
    if (tr) {
      t0 = sp::gtimer();
      c0 = clock64();
    }
    // face of this warp: f = warp >> 1 (0 x-upstream, 1 x-downstream, 2 y-up,
    // 3 y-down in the sweep's rotated frame), side = warp & 1
    const int fw = warp >> 1, side = warp & 1, axis = fw >> 1;
    const bool upf = (fw & 1) == 0;
    const bool a_up = axis == 0 ? b.i_up : b.j_up;
    const bool high = upf ? !a_up : a_up;  // the rotated upstream face is the low face of an ascending axis
    // F pointers of the assembly: [x high side0, side1, x low ..., y high ..., y low ...]
    const bool xu_high = !b.i_up, yu_high = !b.j_up;
    const int fxh = xu_high ? 0 : 1, fyh = yu_high ? 2 : 3;
    unsigned ahead = 0u;  // warps 2, 5, 6: the counters of the next diagonal to copy, read one step ahead
    for (int d = dfirst; d <= dlast; ++d) {
      // old(d), old(d+1); om: old(d-1) (residual tasks) until phase (C) starts the copy of old(d+3) into it
      const int o0 = d & 3, o1 = (d + 1) & 3, om = (d + 3) & 3;
      if (tr) s_tr[0] = sp::gtimer();
      // ---- (A) faces: this warp's side of its face for the 32 cells
      const int jr = d - ir;
      const bool valid = ir < f.nx && jr >= 0 && jr < f.ny;
      {
        const double* Sc = O + o0 * VEC + c;
        const P4 cp = pload(PO + o0 * 132 + c * 4);
        const double* Nb;
        P4 np;
        bool has_nb;
        const double* Up = res ? O + om * VEC : smem + (LY::V_V + ((d - 1) & 1)) * VEC;  // upstream diagonal
        const double* UpP = res ? PO + om * 132 : smem + LY::PV + ((d - 1) & 1) * 132;
        if (fw == 0) {  // x-upstream: slot c-1 of d-1 (band k-1's halo for c = 0)
          has_nb = ir >= 1;
          Nb = Up + (c ? c - 1 : 32);
          np = pload(UpP + (c ? c - 1 : 32) * 4);
        } else if (fw == 1) {  // x-downstream: slot c+1 of d+1 (old)
          has_nb = ir + 1 < f.nx;
          Nb = O + o1 * VEC + c + 1;
          np = pload(PO + o1 * 132 + (c + 1) * 4);
        } else if (fw == 2) {  // y-upstream: slot c of d-1
          has_nb = jr >= 1;
          Nb = Up + c;
          np = pload(UpP + c * 4);
        } else {  // y-downstream: slot c of d+1 (old)
          has_nb = jr + 1 < f.ny;
          Nb = O + o1 * VEC + c;
          np = pload(PO + o1 * 132 + c * 4);
        }
        const int w = face_side<M>(ctx, axis, high, side, valid, has_nb, Sc, cp, Nb, np,
                                   smem + (LY::V_F + warp) * VEC + c);
        if (w && valid && side == 0) {
          const int i = b.i_up ? ir : f.nx - 1 - ir, j = b.j_up ? jr : f.ny - 1 - jr;
          tc::raise(err, tc::code_for(w), w, i, j, 0.0);
        }
      }
      __syncthreads();
      if (tr) s_tr[2] += sp::gtimer() - s_tr[0];
      // ---- (B) residual assembly, coefficients split over the 8 warps (D in F[0])
      const double* pre = smem + LY::PRE + (d & 1) * sp::PRE_N * 32 + c;
      const int pfail = valid ? (int)pre[sp::PRE_FAIL * 32] : W_NONE;
      {
        if (valid && pfail == W_NONE) {
          const double* Fb = smem + LY::V_F * VEC + c;
          const double* Fp[8] = {Fb + (2 * fxh) * VEC,       Fb + (2 * fxh + 1) * VEC,
                                 Fb + (2 * (1 - fxh)) * VEC, Fb + (2 * (1 - fxh) + 1) * VEC,
                                 Fb + (2 * fyh) * VEC,       Fb + (2 * fyh + 1) * VEC,
                                 Fb + (2 * (5 - fyh)) * VEC, Fb + (2 * (5 - fyh) + 1) * VEC};
          const double qv[3] = {pre[sp::PRE_Q0 * 32], pre[sp::PRE_Q0 * 32 + 32], pre[sp::PRE_Q0 * 32 + 64]};
          assemble_part<M>(warp, O + o0 * VEC + c, Fp, pre[sp::PRE_NU * 32], ctx.collision == 2, ctx.shakhov_w, qv,
                           pre[sp::PRE_IDX * 32], pre[sp::PRE_IDY * 32], smem + LY::V_F * VEC + c);
        }
      }
      __syncthreads();
      if (tr) {
        s_b = sp::gtimer() - s_tr[0];
        s_tr[3] += s_b;
      }
      // ---- (C) warp 0: the cell update (sweep) / the residual stores (res);
      // the others: publish d-1, scalars of d+1, old(d+2), band k-1's halo
      if (warp == 0 && !res) {
        int fail = pfail;
        double bad = 0.0;
        int tries = 0;
        if (valid && fail == W_NONE)
          fail = cell_update_body<M>(O + o0 * VEC + c, smem + LY::V_F * VEC + c, PO + o0 * 132 + c * 4,
                                     pre[sp::PRE_DT * 32], smem + (LY::V_V + (d & 1)) * VEC + c,
                                     smem + LY::PV + (d & 1) * 132 + c * 4, &bad, tries);
        if (plan.trace) {  // (debug trace) steps with a dt/2 retry, steps whose update took > 3 us
          const bool any2 = __any_sync(0xffffffffu, tries > 1);
          if (tr) {
            if (any2) s_retry += 1ull;
            if (sp::gtimer() - s_tr[0] - s_b > 3000) s_retry += 1ull << 32;
          }
        }
        if (valid && fail) {
          const int i = b.i_up ? ir : f.nx - 1 - ir, j = b.j_up ? jr : f.ny - 1 - jr;
          tc::raise(err, tc::code_for(fail), fail, i, j, bad);
        }
        const bool ok = valid && fail == W_NONE;
        s_ok[d & 1][c] = ok ? 1 : 0;
        if (tr) s_tr[4] += sp::gtimer() - s_tr[0];
      } else if (res && warp <= 1) {
        // residual: coalesced store of D (lane = coefficient), 16 cells per warp
        const double* Db = smem + LY::V_F * VEC;
        const double* pre0 = smem + LY::PRE + (d & 1) * sp::PRE_N * 32;
#pragma unroll 1
        for (int t = 0; t < 16; ++t) {
          const int cc = 16 * warp + t;
          const int irc = BW * k + cc, jrc = d - irc;
          if (irc >= f.nx || jrc < 0 || jrc >= f.ny) continue;
          if ((int)pre0[sp::PRE_FAIL * 32 + cc] != W_NONE) continue;
          const int cl = b.cell(cc, d);
          double* dst = out.c + (size_t)cl * NP;
#pragma unroll
          for (int h = 0; h < (N + 31) / 32; ++h) {
            const int kq = c + 32 * h;
            if (kq < N) __stcg(dst + kq, Db[kq * SPV + cc]);
          }
          if (c < 4) __stcg(out.p + (size_t)cl * 4 + c, PO[o0 * 132 + cc * 4 + c]);
        }
        if (warp == 0 && valid && pfail) {
          const int i = b.i_up ? ir : f.nx - 1 - ir, j = b.j_up ? jr : f.ny - 1 - jr;
          tc::raise(err, tc::code_for(pfail), pfail, i, j, 0.0);
        }
      } else if (warp == 1) {
        // the update scalars of d+1 (old(d+1) has been in O since step d-2)
        if (d + 1 <= dlast)
          sp::band_pre<M, BW>(f, ctx, b, d + 1, O + o1 * VEC, PO + o1 * 132,
                              smem + LY::PRE + ((d + 1) & 1) * sp::PRE_N * 32);
      } else {  // warps 2..7
        const int stop_now = warp == 2 && c == 0 ? sp::band_stop(err) : 0;
        // every role below is one or two dependent memory round trips, shorter than warp 0's update
        if (warp == 2) {
          // publication of step d-2: its stores were issued a step ago by
          // warps 3, 4 (ordered by that step's CTA barrier), so the one
          // release of the step has nothing to wait for
          if (!res && d - 2 >= dfirst) {
            sp::sched_jitter(plan.jitter, (unsigned)d);
            const int cl = b.cell(c, d - 2);
            if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, false);
          }
        } else if (warp <= 4) {
          // write-back of step d-1 (final since the last CTA barrier), 16 cells per warp
          if (!res && d > dfirst) {
            if (trw) s_wM[warp] += sp::gtimer() - s_tr[0];
            rb_writeback<M>(f, b, d - 1, smem + (LY::V_V + ((d - 1) & 1)) * VEC, smem + LY::PV + ((d - 1) & 1) * 132,
                            s_ok[(d - 1) & 1], 16 * (warp - 3), 16);
          }
        }
        if (warp == 2 || warp == 5 || warp == 6) {
          // old(d+2), issued one step ago, has landed; start the copy of
          // old(d+3), a third of the 33 slots per warp
          const int wi = warp == 2 ? 2 : warp - 5;
          cp_async_wait();
          if (d + 2 <= dlast) {
            const unsigned need = res ? rneed : ep + (unsigned)s;
            band_load_async<M, 11>(fa, b, d + 3, NS, need, O + om * VEC, PO + om * 132, wi, 3, err, plan.poll_ns,
                                   plan.jitter, ahead);
            if (trw) s_wM[warp] += sp::gtimer() - s_tr[0];
            ahead = band_counters_ahead<11>(fa, b, d + 4, NS, need, wi, 3);
          }
        } else if (warp == 7) {
          if (res && d + 1 <= dlast)
            sp::band_pre<M, BW>(f, ctx, b, d + 1, O + o1 * VEC, PO + o1 * 132,
                                smem + LY::PRE + ((d + 1) & 1) * sp::PRE_N * 32);
          // band k-1's new cell of diagonal d (the next step's x-upstream halo)
          if (k > 0 && d + 1 <= dlast) {
            double* hv = (res ? O + o0 * VEC : smem + (LY::V_V + (d & 1)) * VEC) + 32;
            double* hp = (res ? PO + o0 * 132 : smem + LY::PV + (d & 1) * 132) + 128;
            const int cl = b.cell(-1, d);
            if (cl >= 0) {
              const unsigned need = res ? rneed : ep + (unsigned)s + 1u;
              sp::sched_jitter(plan.jitter, (unsigned)d);
              if (c == 0 && need) poll_acquire(fa.vptr(cl), need, cl, b.nx, err, plan.poll_ns);
              if (trw) s_wM[warp] += sp::gtimer() - s_tr[0];
              __syncwarp();
              const double r0 = c < N ? __ldcg(fa.cptr(cl, NP) + c) : 0.0;
              const double r1 = c + 32 < N ? __ldcg(fa.cptr(cl, NP) + c + 32) : 0.0;
              const double pr = c < 4 ? __ldcg(fa.pptr(cl) + c) : 0.0;
              if (c < N) hv[c * SPV] = r0;
              if (c + 32 < N) hv[(c + 32) * SPV] = r1;
              if (c < 4) hp[c] = pr;
            } else {
              if (c < N) hv[c * SPV] = 0.0;
              if (c + 32 < N) hv[(c + 32) * SPV] = 0.0;
              if (c < 4) hp[c] = 0.0;
            }
          }
        }
        if (warp == 2 && c == 0) s_stop = stop_now;
      }
      if (trw) s_wC[warp] += sp::gtimer() - s_tr[0];
      __syncthreads();
      if (tr) {
        const unsigned long long dur = sp::gtimer() - s_tr[0];
        s_tr[5] += dur;
        // histogram of the step durations (bins end at 9, 10, 11, 12.5, 15, 20, 40 us, then the rest)
        const int bin = dur < 9000 ? 0 : dur < 10000 ? 1 : dur < 11000 ? 2 : dur < 12500 ? 3 : dur < 15000 ? 4
                        : dur < 20000 ? 5 : dur < 40000 ? 6 : 7;
        s_wA[bin] += 1;
      }
      if (s_stop) return;
    }
    if (!res) rb_writeback<M>(f, b, dlast, smem + (LY::V_V + (dlast & 1)) * VEC, smem + LY::PV + (dlast & 1) * 132,
                              s_ok[dlast & 1], 4 * warp, 4);
    __syncthreads();
    if (!res && warp == 1) {
      const int cp_ = dlast > dfirst ? b.cell(c, dlast - 1) : -1;  // (written back during step dlast)
      if (cp_ >= 0) st_release_s(fa.vptr(cp_), ep + (unsigned)s + 1u, false);
      const int cl = b.cell(c, dlast);
      if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, false);
    }
    if (tr) {
      unsigned long long* o = plan.trace + (size_t)task * 32;
      o[0] = t0;
      o[1] = sp::gtimer();
      o[2] = (unsigned long long)(dlast - dfirst + 1) | ((unsigned long long)s << 20) | ((unsigned long long)k << 28);
      for (int t = 3; t < 32; ++t) o[t] = 0;
      o[3] = s_tr[1];
      o[4] = s_tr[2];
      o[12] = s_tr[3];
      o[5] = s_tr[4];
      o[7] = s_tr[5];
      for (int w = 0; w < 8; ++w) {
        o[16 + w] = s_wA[w];
        o[24 + w] = s_wC[w];
        if (w >= 2 && w != 6) o[6 + w] = s_wM[w];  // [8..13]: mid-role stamps of warps 2..7 (warp 6 in [14])
      }
      o[10] = 0;  // (marks the k8 stamp set; warp 4's mid-role stamp is not kept)
      o[12] = s_tr[3];
      o[14] = s_wM[6];
      o[6] = s_retry;  // steps with a dt/2 retry | steps with an update > 3 us << 32
      o[15] = (unsigned long long)(clock64() - c0);  // SM cycles over the loop (effective clock)
    }
  }
}

}  // namespace rb
}  // namespace momg_gpu
