// Register-resident band sweep for second order and / or an FAS right-hand
// side (k9_band; M <= 5, BGK / Shakhov, one flat field, exact order): the
// NMG levels of BASELINE C2.  Same schedule as k8_band (reg_band.cuh: a task
// = one sweep x one band of 32 rotated columns walked diagonal by diagonal,
// 8 warps = 4 faces x {cell side, neighbour side}, one THREAD per face side
// with the whole moment vector in registers, assembly split over the warps,
// update in registers on warp 0, old states copied in with cp.async under the
// update, counters read one step ahead), what changes is the stencil:
//
//  * second-order face states (spatial.cpp:34-80) reach two cells along each
//    axis: a side's state is  w = c + (off / h) (hi - lo)  of three on-chip
//    vectors (its cell and that cell's two neighbours along the axis), with
//    the nonpositive-temperature fallback to the cell itself; the other
//    side's state is needed only through the seven coefficients of the
//    wave-speed bounds (flux.cpp:79-84), rebuilt from the same vectors;
//  * so the rings hold old(d) .. old(d+3) (34 slots: the band's 32 columns +
//    band k+1's first two) and new(d-2), new(d-1) (34 slots: band k-1's last
//    two columns, polled on their counters, + the 32 columns);
//  * coarse levels subtract the projected right-hand side
//    (single_level.cpp:64-70): an otherwise idle warp projects the rhs of
//    diagonal d+1 into its cells' bases one step ahead (vector R);
//  * 14 vectors of 34 slots fit shared memory: old ring 4, new ring 2, the
//    cell sides' F[4], R, and three vectors X[3] for the neighbour sides of
//    faces 0..2 -- face 3's neighbour side uses the old-ring slot that is
//    dead until phase (C) starts the next copy into it.
//
// Compiled in its own translation units (rb2_m<M>.cu) with SPV = 35.
#pragma once

#include "momg_cell.cuh"
#include "sweep_persistent.cuh"
#include "kernels_v3.cuh"
#include "reg_band.cuh"

namespace momg_gpu {
int rb_grid_cap(int nb, int nk);  // runtime.cu (declared with its rationale in kernels_impl.cuh)
namespace rb {


// BW: columns per band task (32; 16 for M = 6, whose 84-coefficient vectors
// would not fit shared memory at 32)
template <int M, int BW>
struct R2Layout {
  static_assert(SPV >= BW + 2, "k9 vectors need BW + 2 slots");
  static constexpr int N = Gen<M>::N;
  static constexpr int VEC = N * SPV;
  // vectors: O[4] old ring (slot = column), V[2] new ring (slot = column + 2),
  // F[4] cell sides of the faces (F[0] doubles as the assembled delta D), R
  // projected rhs, X[3] neighbour sides of faces 0..2
  static constexpr int V_O = 0, V_V = 4, V_F = 6, V_R = 10, V_X = 11, NV = 14;
  static constexpr int PS = (BW + 2) * 4;   // params of one vector
  static constexpr int PO = NV * VEC;       // [4][BW + 2][4]
  static constexpr int PV = PO + 4 * PS;    // [2][BW + 2][4]
  static constexpr int PRE = PV + 2 * PS;   // [2][PRE_N][32]
  static constexpr size_t bytes = (size_t)(PRE + 2 * sp::PRE_N * 32) * sizeof(double);
};

// the seven coefficients the wave-speed bounds read (rho, the three first
// moments, the three 2 e_d) of  c + a (hi - lo)
__device__ __forceinline__ void recon7(const double* cv, const double* hi, const double* lo, double a, bool rec,
                                       double (&o)[7]) {
  constexpr int K7[7] = {0, 1, 2, 3, 4, 7, 9};
#pragma unroll
  for (int t = 0; t < 7; ++t) {
    const double x = cv[K7[t] * SPV];
    o[t] = rec ? fma(a, hi[K7[t] * SPV] - lo[K7[t] * SPV], x) : x;
  }
}
// rep_temperature (moment_rep.hpp:77-90) of the seven coefficients
__device__ __forceinline__ double rep_theta7(const double (&s)[7], const P4& p) {
  const double rho = s[0];
  double trace = 0.0, fe2 = 0.0;
  trace += s[4];
  fe2 += s[1] * s[1];
  trace += s[5];
  fe2 += s[2] * s[2];
  trace += s[6];
  fe2 += s[3] * s[3];
  const double ir = 1.0 / rho;
  return p.v[3] + (2.0 * trace - fe2 * ir) * (ir * (1.0 / 3.0));
}

struct Asm2Args {
  const double *S, *Fxh0, *Fxh1, *Fxl0, *Fxl1, *Fyh0, *Fyh1, *Fyl0, *Fyl1, *R;
  double nu, shw, idx, idy, s0;
  bool shk, rhs;
  const double* qv;
  double* D;
};
template <int K>
__device__ __forceinline__ void assemble2_one(const Asm2Args& a) {
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
  if (a.rhs) r -= a.R[o];  // update_delta, single_level.cpp:64-70
  a.D[o] = r;
}
template <int K0, int... I>
__device__ __forceinline__ void assemble2_seq(const Asm2Args& a, std::integer_sequence<int, I...>) {
  (assemble2_one<K0 + I>(a), ...);
}
template <int M>
__device__ __forceinline__ void assemble2_part(int w, const Asm2Args& a) {
  constexpr int N = Gen<M>::N, CH = (N + 7) / 8;
#define RB_AS2(W)                                                                                          \
  case W:                                                                                                  \
    assemble2_seq<(W * CH < N ? W * CH : N)>(                                                              \
        a, std::make_integer_sequence<int, ((W + 1) * CH < N ? (W + 1) * CH : N) - (W * CH < N ? W * CH : N)>{}); \
    break;
  switch (w) {
    RB_AS2(0)
    RB_AS2(1)
    RB_AS2(2)
    RB_AS2(3)
    RB_AS2(4)
    RB_AS2(5)
    RB_AS2(6)
    RB_AS2(7)
  }
#undef RB_AS2
}

// Coalesced write-back of nc cells starting at column c0 of diagonal dd from
// a new-ring vector (slot = column + 2): the cells' indices are computed by
// the lanes up front, lane = coefficient in the stores.
template <int M, class Geo>
__device__ __forceinline__ void rb2_writeback(const DevField& f, const Geo& b, int dd, const double* V,
                                              const double* PV, const int* ok, int c0, int nc) {
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3, H = (N + 31) / 32;
  const int lane = threadIdx.x & 31;
  int mine = -1;
  if (lane < nc && ok[c0 + lane]) mine = b.cell(c0 + lane, dd);
#pragma unroll 2
  for (int t = 0; t < nc; ++t) {
    const int cl = __shfl_sync(0xffffffffu, mine, t);
    if (cl < 0) continue;
    const int sl = c0 + t + 2;
    double* dst = f.c + (size_t)cl * NP;
    double r[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int k = lane + 32 * h;
      r[h] = k < N ? V[k * SPV + sl] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int k = lane + 32 * h;
      if (k < N) __stcg(dst + k, r[h]);
    }
    if (lane < 4) __stcg(f.p + (size_t)cl * 4 + lane, PV[sl * 4 + lane]);
  }
}

// One cell record (coefficients, params) into slot `sl` of a vector, lane =
// coefficient; zeros for a cell outside the grid.
template <int M, class Addr>
__device__ __forceinline__ void load_slot(const Addr& fa, int cl, double* vec, double* prm, int sl) {
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  const int c = threadIdx.x & 31;
  constexpr int H = (N + 31) / 32;
  double r[H];
#pragma unroll
  for (int h = 0; h < H; ++h) r[h] = (cl >= 0 && c + 32 * h < N) ? __ldcg(fa.cptr(cl, NP) + c + 32 * h) : 0.0;
  const double pr = (cl >= 0 && c < 4) ? __ldcg(fa.pptr(cl) + c) : 0.0;
#pragma unroll
  for (int h = 0; h < H; ++h)
    if (c + 32 * h < N) vec[(c + 32 * h) * SPV + sl] = r[h];
  if (c < 4) prm[sl * 4 + c] = pr;
}

// The rhs of the cells of diagonal dd projected into their (old) bases, into
// R (slot = column); lane = cell, the record in registers (transfer.cuh).
template <int M, int BW, class Geo>
__device__ __forceinline__ void rhs_project(const DevField& rhs, const Geo& b, int dd, const double* PO, double* R) {
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  const int c = threadIdx.x & 31;
  const int cl = c < BW ? b.cell(c, dd) : -1;
  if (cl < 0) return;
  double v[N];
  xf::load_rec<M, false>(rhs.c + (size_t)cl * NP, v);
  const P4 from = tc::ldp<false>(rhs.p + (size_t)cl * 4);
  const P4 to = pload(PO + c * 4);
  if (to.v[3] > 0.0) xf::project_row<M, (M <= 5)>(v, from, to);
  vstore<M>(R + c, v);
}

template <int M, int BW>
__global__ void __launch_bounds__(RT, 1) k9_band(DevField f, DevField rhsf, DevCtx ctx, DevErr* err, BandPlan plan) {
  constexpr int NS = BW + 2;
  constexpr int AM = (NS + 1) / 2;  // slots per copying warp
  using LY = R2Layout<M, BW>;
  constexpr int N = LY::N, VEC = LY::VEC, PS = LY::PS;
  extern __shared__ __align__(128) double smem[];
  __shared__ int s_task, s_stop;
  __shared__ int s_ok[2][32];
  __shared__ unsigned long long s_tr[6];
  const int tid = threadIdx.x, warp = tid >> 5, c = tid & 31;
  const int ntasks = plan.nsweeps * plan.nk;
  const unsigned ep = plan.epoch;
  const bool o2 = plan.order == 2, has_rhs = plan.has_rhs != 0;
  const sp::CellAddr<false> fa{nullptr, f.c, f.p, plan.ver};
  double* const O = smem + LY::V_O * VEC;
  double* const V = smem + LY::V_V * VEC;
  double* const PO = smem + LY::PO;
  double* const PV = smem + LY::PV;
  double* const R = smem + LY::V_R * VEC;
  for (;;) {
    if (tid == 0) {
      sp::sched_jitter(plan.jitter, 1u);
      s_task = (int)atomicAdd(plan.next, 1u);
      s_stop = sp::band_stop(err);
    }
    __syncthreads();
    const int task = s_task;
    if (task >= ntasks || s_stop) return;
    const int s = task / plan.nk;
    const int dir = (int)((plan.dirbits >> (2 * s)) & 3u);
    const int k = task % plan.nk;
    BandGeo<false> b;
    b.nx = f.nx;
    b.ny = f.ny;
    b.k = k;
    b.bw = BW;
    b.i_up = dir == 0 || dir == 3;
    b.j_up = dir == 0 || dir == 1;
    const int ir = BW * k + c;
    const int dfirst = BW * k, dlast = min(BW * k + BW - 1, f.nx - 1) + f.ny - 1;
    const bool tr = plan.trace && 4 * task + 3 < plan.trace_cap && tid == 0;
    unsigned long long t0 = 0;
    if (tr)
      for (int q = 0; q < 6; ++q) s_tr[q] = 0;
    // ---- prologue: old(dfirst .. dfirst+2), band k-1's last two columns of
    // new(dfirst-1), new(dfirst-2), the update scalars and rhs of dfirst
    const unsigned nold = ep + (unsigned)s;
#pragma unroll 1
    for (int t = 0; t < 3; ++t)
      sp::band_load<M, 5>(fa, b, dfirst + t, 0, NS, nold, O + ((dfirst + t) & 3) * VEC, SPV,
                          PO + ((dfirst + t) & 3) * PS, warp, 8, err, sp::kPrologueSleepNs);
    if (k > 0 && warp >= 6) {
      const int dd = dfirst - 1 - (warp - 6);
      sp::band_load<M, 2>(fa, b, dd, -2, 2, nold + 1u, V + (dd & 1) * VEC, SPV, PV + (dd & 1) * PS, 0, 1, err,
                          sp::kPrologueSleepNs);
    }
    __syncthreads();
    if (warp == 1)
      sp::band_pre<M, BW>(f, ctx, b, dfirst, O + (dfirst & 3) * VEC, PO + (dfirst & 3) * PS,
                          smem + LY::PRE + (dfirst & 1) * sp::PRE_N * 32);
    if (warp == 2 && has_rhs) rhs_project<M, BW>(rhsf, b, dfirst, PO + (dfirst & 3) * PS, R);
    __syncthreads();
    if (tr) t0 = sp::gtimer();
    // face of this warp: fw (0 x-upstream, 1 x-downstream, 2 y-upstream, 3
    // y-downstream in the sweep's rotated frame) and side.  32-column bands:
    // fw = warp >> 1, side = warp & 1, lane = cell.  16-column bands (PAIR):
    // both sides of a face in ONE warp, lane = cell + 16 side, so warps 0..3
    // run the four faces with every lane busy (the sides differ by selects
    // only) instead of eight half-empty warps.
    constexpr bool PAIR = BW == 16;
    const int fw = PAIR ? (warp & 3) : warp >> 1, side = PAIR ? (c >> 4) : (warp & 1), axis = fw >> 1;
    const bool upf = (fw & 1) == 0;
    const bool a_up = axis == 0 ? b.i_up : b.j_up;
    const bool high = upf ? !a_up : a_up;  // the rotated upstream face is the low face of an ascending axis
    const int nax = axis == 0 ? f.nx : f.ny;
    const double* xcs = axis == 0 ? f.xc : f.yc;
    const double* dxs = axis == 0 ? f.dx : f.dy;
    // F vectors of the assembly: x high / low, y high / low
    const int fxh = !b.i_up ? 0 : 1, fyh = !b.j_up ? 2 : 3;
    unsigned ahead = 0u;
    for (int d = dfirst; d <= dlast; ++d) {
      if (tr) s_tr[0] = sp::gtimer();
      const int jr = d - ir;
      const bool valid = c < BW && ir < f.nx && jr >= 0 && jr < f.ny;
      // ---- (A) faces: this warp's side of its face for the 32 cells
      if (!PAIR || warp < 4) {
        // (inside this block c, ir, jr, valid are the face thread's cell: lane & 15 when PAIR)
        const int lane_ = c, ir_ = ir;
        const int c = PAIR ? (lane_ & 15) : lane_;
        const int ir = PAIR ? BW * k + c : ir_;
        const int jr = d - ir;
        const bool valid = c < BW && ir < f.nx && jr >= 0 && jr < f.ny;
        // the cell at rotated offset r along the axis: (c + r, d + r) for
        // x, (c, d + r) for y; new ring below the diagonal, old ring above
        auto at = [&](int r, const double** v, const double** pp) {
          const int dd = d + r;
          if (r < 0) {
            const int sl = (axis == 0 ? c + r : c) + 2;
            *v = V + (dd & 1) * VEC + sl;
            *pp = PV + (dd & 1) * PS + sl * 4;
          } else {
            const int sl = axis == 0 ? c + r : c;
            *v = O + (dd & 3) * VEC + sl;
            *pp = PO + (dd & 3) * PS + sl * 4;
          }
        };
        const int rn = upf ? -1 : 1;  // rotated offset of the face's neighbour
        const double *Sc, *Sp, *Nb, *Np;
        at(0, &Sc, &Sp);
        at(rn, &Nb, &Np);
        const P4 cp = pload(Sp);
        const int i = b.i_up ? ir : f.nx - 1 - ir, j = b.j_up ? jr : f.ny - 1 - jr;
        const int pos = axis == 0 ? i : j;
        const bool has_nb = valid && (high ? pos + 1 < nax : pos >= 1);
        // this side's vector: scratch for the projected state, then its flux in the cell basis
        double* F = (side == 0 ? smem + (LY::V_F + fw) * VEC
                               : (fw < 3 ? smem + (LY::V_X + fw) * VEC : O + ((d + 3) & 3) * VEC)) + c;
        int fail = W_NONE;
        int branch = sp::B_NONE;
        P4 to{}, from{};
        double rs = 1.0;
        // this side's state: Mv, or Mv + a_me (Mhi - Mlo) when reconstructed (rme_ok)
        const double *Mv = Sc, *Mhi = Sc, *Mlo = Sc;
        double a_me = 0.0;
        bool rme_ok = false;
        const bool my_left = side == 0 ? high : !high;  // left = lower-index cell of the face
        if (valid && !has_nb) {
          if (side == 0) {  // wall closure on the cell's own (unreconstructed) state, spatial.cpp:105-111
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
              from = cp;
            }
          }
        } else if (valid) {
          // the two cells of the face: me (this side's cell) and ot (the
          // other side's); each reconstructs with its own two neighbours
          // along the axis (safe_face_state, spatial.cpp:64-80), one of which
          // is the other cell.  Original offset +1 is rotated +1 on an
          // ascending axis.
          const int rme = side == 0 ? 0 : rn, rot = side == 0 ? rn : 0;
          const int pme = side == 0 ? pos : (high ? pos + 1 : pos - 1);
          const int pot = side == 0 ? (high ? pos + 1 : pos - 1) : pos;
          const double *Mp, *Ov, *Op;
          at(rme, &Mv, &Mp);
          at(rot, &Ov, &Op);
          const P4 mp0 = pload(Mp), op0 = pload(Op);
          P4 mp = mp0, opp = op0;
          // me is the face's lower cell iff my_left: its face is its high face (off = +dx/2)
          const bool rec_me = o2 && pme > 0 && pme < nax - 1;
          const bool rec_ot = o2 && pot > 0 && pot < nax - 1;
          double a_ot = 0.0;
          bool rot_ok = false;
          const double *Ohi = nullptr, *Olo = nullptr;
          const int up1 = a_up ? 1 : -1;  // rotated offset of original +1
          if (rec_me) {
            const double *hp, *lp_;
            at(rme + up1, &Mhi, &hp);
            at(rme - up1, &Mlo, &lp_);
            const double ih = 1.0 / (xcs[pme + 1] - xcs[pme - 1]);
            const double off = (my_left ? 0.5 : -0.5) * dxs[pme];
            P4 w;
#pragma unroll
            for (int t = 0; t < 4; ++t) w.v[t] = mp0.v[t] + off * ((hp[t] - lp_[t]) * ih);
            if (w.v[3] > 0.0) {
              rme_ok = true;
              mp = w;
              a_me = off * ih;
            }
          }
          if (rec_ot) {
            const double *hp, *lp_;
            at(rot + up1, &Ohi, &hp);
            at(rot - up1, &Olo, &lp_);
            const double ih = 1.0 / (xcs[pot + 1] - xcs[pot - 1]);
            const double off = (my_left ? -0.5 : 0.5) * dxs[pot];
            P4 w;
#pragma unroll
            for (int t = 0; t < 4; ++t) w.v[t] = op0.v[t] + off * ((hp[t] - lp_[t]) * ih);
            if (w.v[3] > 0.0) {
              rot_ok = true;
              opp = w;
              a_ot = off * ih;
            }
          }
          // wave-speed bounds (flux.cpp:79-84) from both face states, through
          // the seven coefficients they read (before this side's vector is
          // loaded: fewer live registers)
          {
            double m7[7], o7[7];
            recon7(Mv, rme_ok ? Mhi : Mv, rme_ok ? Mlo : Mv, a_me, rme_ok, m7);
            recon7(Ov, rot_ok ? Ohi : Ov, rot_ok ? Olo : Ov, a_ot, rot_ok, o7);
            const P4 lp = my_left ? mp : opp;
            const P4 rp = my_left ? opp : mp;
            double l7[7], r7[7];
#pragma unroll
            for (int t = 0; t < 7; ++t) {
              l7[t] = my_left ? m7[t] : o7[t];
              r7[t] = my_left ? o7[t] : m7[t];
            }
            const double ul = (axis == 0 ? lp.v[0] : lp.v[1]) + (axis == 0 ? l7[1] : l7[2]) * (1.0 / l7[0]);
            const double ur = (axis == 0 ? rp.v[0] : rp.v[1]) + (axis == 0 ? r7[1] : r7[2]) * (1.0 / r7[0]);
            const double cl = ctx.c_bound * sqrt(rep_theta7(l7, lp));
            const double cr = ctx.c_bound * sqrt(rep_theta7(r7, rp));
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
              from = mp;
            }
          }
        }
        double v[N];
        if (branch == sp::B_NONE) {
#pragma unroll
          for (int kk = 0; kk < N; ++kk) v[kk] = 0.0;
        } else {
          const bool full = branch == sp::B_FULL_L || branch == sp::B_FULL_R;
          const bool wall = branch == sp::B_WALL;
          // this side's state in registers
          if (rme_ok) {
#pragma unroll
            for (int kk = 0; kk < N; ++kk) v[kk] = fma(a_me, Mhi[kk * SPV] - Mlo[kk * SPV], Mv[kk * SPV]);
          } else {
            vload<M>(Mv, v);
          }
          xf::project_row<M, (M <= 5)>(v, from, to);
          // through F once: the flux reads it back pencil by pencil
          if (BW == 32 || c < BW) vstore<M>(F, v);
          asm volatile("" ::: "memory");
          if (full) {
            if (axis == 0) Gen<M>::template full_flux0<SPV, 1>(F, v, to.v[0], to.v[3]);
            else Gen<M>::template full_flux1<SPV, 1>(F, v, to.v[1], to.v[3]);
          } else {
            const double un = wall ? 0.0 : (axis == 0 ? to.v[0] : to.v[1]);
            double K[M + 1][M + 1];
            double kin0[M + 1];
            half_kernel_side<M>(un, rs, tc::half_base(un, rs), wall ? high : my_left, K, kin0);
            if constexpr (M <= 5) {
              if (axis == 0) Gen<M>::template half_sr0<SPV, 1>(F, v, K);
              else Gen<M>::template half_sr1<SPV, 1>(F, v, K);
            } else {
              // the (M+1)^2 table and the vector do not fit the registers
              // together: the flux runs in place in shared memory (a pencil's
              // inputs are read before its outputs are written)
              if (axis == 0) Gen<M>::template half_one0<SPV>(F, K);
              else Gen<M>::template half_one1<SPV>(F, K);
              asm volatile("" ::: "memory");
              vload<M>(F, v);
            }
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
          xf::project_row<M, (M <= 5)>(v, to, pload(Sp));
        }
        if (BW == 32 || c < BW) vstore<M>(F, v);
        if (fail && valid && side == 0) tc::raise(err, tc::code_for(fail), fail, i, j, 0.0);
      }
      __syncthreads();
      if (tr) s_tr[2] += sp::gtimer() - s_tr[0];
      // ---- (B) delta assembly, coefficients split over the 8 warps (D in F[0])
      const double* pre = smem + LY::PRE + (d & 1) * sp::PRE_N * 32 + c;
      const int pfail = valid ? (int)pre[sp::PRE_FAIL * 32] : W_NONE;
      if (valid && pfail == W_NONE) {
        const double* Fb = smem + LY::V_F * VEC + c;
        const double qv[3] = {pre[sp::PRE_Q0 * 32], pre[sp::PRE_Q0 * 32 + 32], pre[sp::PRE_Q0 * 32 + 64]};
        const double* S = O + (d & 3) * VEC + c;
        const double* Xb = smem + LY::V_X * VEC + c;
        const double* X3 = O + ((d + 3) & 3) * VEC + c;  // face 3's neighbour side
        const int fxl = 1 - fxh, fyl = 5 - fyh;
        const Asm2Args a{S,
                         Fb + fxh * VEC,
                         Xb + fxh * VEC,
                         Fb + fxl * VEC,
                         Xb + fxl * VEC,
                         Fb + fyh * VEC,
                         fyh < 3 ? Xb + fyh * VEC : X3,
                         Fb + fyl * VEC,
                         fyl < 3 ? Xb + fyl * VEC : X3,
                         R + c,
                         pre[sp::PRE_NU * 32],
                         ctx.shakhov_w,
                         pre[sp::PRE_IDX * 32],
                         pre[sp::PRE_IDY * 32],
                         S[0],
                         ctx.collision == 2,
                         has_rhs,
                         qv,
                         smem + LY::V_F * VEC + c};
        assemble2_part<M>(warp, a);
      }
      __syncthreads();
      if (tr) s_tr[3] += sp::gtimer() - s_tr[0];
      // ---- (C) warp 0: the cell update; the others: scalars and rhs of
      // d+1, publication of d-2 and write-back of d-1, the copy of old(d+3),
      // band k-1's new cells of diagonal d
      if (warp == 0) {
        int fail = pfail;
        double bad = 0.0;
        if (valid && fail == W_NONE) {
          const double* S = O + (d & 3) * VEC + c;
          const double* D = smem + LY::V_F * VEC + c;
          const double* cpp = PO + (d & 3) * PS + c * 4;
          double* Vout = V + (d & 1) * VEC + c + 2;
          double* PVout = PV + (d & 1) * PS + (c + 2) * 4;
          const double dt = pre[sp::PRE_DT * 32];
          if constexpr (M <= 5) fail = cell_update_body<M>(S, D, cpp, dt, Vout, PVout, &bad);
          else fail = cell_update_call<M>(S, D, cpp, dt, Vout, PVout, &bad);
        }
        if (valid && fail) {
          const int i = b.i_up ? ir : f.nx - 1 - ir, j = b.j_up ? jr : f.ny - 1 - jr;
          tc::raise(err, tc::code_for(fail), fail, i, j, bad);
        }
        const bool ok = valid && fail == W_NONE;
        s_ok[d & 1][c] = ok ? 1 : 0;
        if (tr) s_tr[4] += sp::gtimer() - s_tr[0];
      } else if (warp == 1) {
        if (d + 1 <= dlast)
          sp::band_pre<M, BW>(f, ctx, b, d + 1, O + ((d + 1) & 3) * VEC, PO + ((d + 1) & 3) * PS,
                              smem + LY::PRE + ((d + 1) & 1) * sp::PRE_N * 32);
      } else if (warp == 2) {
        const int stop_now = c == 0 ? sp::band_stop(err) : 0;
        if (has_rhs && d + 1 <= dlast) rhs_project<M, BW>(rhsf, b, d + 1, PO + ((d + 1) & 3) * PS, R);
        if (c == 0) s_stop = stop_now;
      } else if (warp <= 4) {
        // publication of step d-2 (stored a step ago), write-back of step d-1
        if (d > dfirst) {
          const int c0 = (BW / 2) * (warp - 3);
          sp::sched_jitter(plan.jitter, (unsigned)d);
          if (d - 2 >= dfirst && c < BW / 2) {
            const int cl = b.cell(c0 + c, d - 2);
            if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, false);
          }
          rb2_writeback<M>(f, b, d - 1, V + ((d - 1) & 1) * VEC, PV + ((d - 1) & 1) * PS, s_ok[(d - 1) & 1], c0, BW / 2);
          __syncwarp();
        }
      } else if (warp <= 6) {
        // old(d+3) is read from the next step on (as old(d'+2)): copied in
        // during this phase, under the update
        if (d + 1 <= dlast) {
          band_load_async<M, AM>(fa, b, d + 3, NS, nold, O + ((d + 3) & 3) * VEC, PO + ((d + 3) & 3) * PS, warp - 5, 2,
                                 err, plan.poll_ns, plan.jitter, ahead);
          ahead = band_counters_ahead<AM>(fa, b, d + 4, NS, nold, warp - 5, 2);
        }
        cp_async_wait();
      } else {
        // band k-1's columns -1 and -2 of diagonal d (slots 1, 0 of new(d))
        if (k > 0 && d + 1 <= dlast) {
          const int c1 = b.cell(-1, d), c2 = b.cell(-2, d);
          sp::sched_jitter(plan.jitter, (unsigned)d);
          if (c == 0 && c1 >= 0) poll_acquire(fa.vptr(c1), nold + 1u, c1, b.nx, err, plan.poll_ns);
          if (c == 1 && c2 >= 0) poll_acquire(fa.vptr(c2), nold + 1u, c2, b.nx, err, plan.poll_ns);
          __syncwarp();
          load_slot<M>(fa, c1, V + (d & 1) * VEC, PV + (d & 1) * PS, 1);
          load_slot<M>(fa, c2, V + (d & 1) * VEC, PV + (d & 1) * PS, 0);
        }
      }
      __syncthreads();
      if (tr) s_tr[5] += sp::gtimer() - s_tr[0];
      if (s_stop) return;
    }
    rb2_writeback<M>(f, b, dlast, V + (dlast & 1) * VEC, PV + (dlast & 1) * PS, s_ok[dlast & 1], (BW / 8) * warp,
                     BW / 8);
    __syncthreads();
    if (warp == 1) {
      const int cp_ = dlast > dfirst && c < BW ? b.cell(c, dlast - 1) : -1;  // (written back during step dlast)
      if (cp_ >= 0) st_release_s(fa.vptr(cp_), ep + (unsigned)s + 1u, false);
      const int cl = c < BW ? b.cell(c, dlast) : -1;
      if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, false);
    }
    if (tr) {
      unsigned long long* o = plan.trace + (size_t)task * 32;
      o[0] = t0;
      o[1] = sp::gtimer();
      o[2] = (unsigned long long)(dlast - dfirst + 1) | ((unsigned long long)s << 20) | ((unsigned long long)k << 28);
      for (int t = 3; t < 32; ++t) o[t] = 0;
      o[4] = s_tr[2];
      o[12] = s_tr[3];
      o[5] = s_tr[4];
      o[7] = s_tr[5];
    }
  }
}

template <int M, int BW>
void rb2_launch_impl(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err, const BandPlan& plan,
                     cudaStream_t st) {
  static int nsm = 0;
  if (!nsm) {
    cudaFuncSetAttribute(k9_band<M, BW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)R2Layout<M, BW>::bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int nb = nsm;  // one CTA per SM (smem-bound); tasks are claimed dynamically
  if (nb > plan.nsweeps * plan.nk) nb = plan.nsweeps * plan.nk;
  nb = rb_grid_cap(nb, plan.nk);  // (kernels_impl.cuh: one CTA per TPC while the tasks allow it)
  k9_band<M, BW><<<nb, RT, R2Layout<M, BW>::bytes, st>>>(f, rhs, ctx, err, plan);
}

}  // namespace rb
}  // namespace momg_gpu
