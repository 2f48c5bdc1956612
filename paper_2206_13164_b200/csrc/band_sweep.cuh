// Band-persistent exact fast sweep, first order, M <= 5, no rhs (k5_band;
// sweeps with an FAS right-hand side run the wavefront items of split_cell.cuh).
//
// fast_sweep_step (single_level.cpp:121-166) visits the cells of each sweep
// in lexicographic order (i outer, j inner, in the sweep's direction).  In
// the sweep's rotated frame (ir, jr) a cell depends on the NEW states of
// (ir-1, jr) and (ir, jr-1) and the OLD (previous sweep) states of (ir+1, jr)
// and (ir, jr+1): the anti-diagonals d = ir + jr are the wavefronts.
//
// A task is one band of 32 rotated columns (ir = 32k + lane) of one sweep,
// walked diagonal by diagonal by one CTA (the 512-thread split layout of
// split_cell.cuh: 4 face groups x 4 partitions, lane = cell).  Everything a
// step needs except one cell is already on chip:
//   * the new states of diagonal d-1 are the previous step's update output
//     (V), shifted by one lane for the x-upstream face;
//   * the old states of diagonals d and d+1 were prefetched one and two
//     steps earlier (OLD1 / X), by the 12 warps that are idle while face
//     group 0 runs the cell update;
//   * only lane 0's x-upstream neighbour comes from band k-1 (HALO), polled
//     on its per-cell counter during the previous step's update.
// So the critical path of a step is copies + face phases + update, with no
// global round trip on it.  Tasks are handed out in (sweep, band) order by
// an atomic counter: every dependency of a task (band k-1 of the same sweep,
// any band of earlier sweeps) belongs to an earlier task, which is running
// or finished, so the schedule cannot deadlock and needs no co-residency.
// The per-cell counters (rule in sweep_persistent.cuh) still gate every
// global read, so tasks of consecutive sweeps overlap safely.
#pragma once

#include "split_cell.cuh"
#include "strips.h"

namespace momg_gpu {
namespace sp {

// Global addresses of a cell handle (ST: strip table; else one flat field)
template <bool ST = false>
struct CellAddr {
  static constexpr bool kStrips = ST;
  const StripTab* st;
  double* c;
  double* p;
  unsigned* ver;
  template <class T>
  static __device__ __forceinline__ T* tab(T* const* a, int h) {
    return (T*)__ldg((const unsigned long long*)&a[h >> kStripShift]);
  }
  __device__ __forceinline__ double* cptr(int h, int NP) const {
    if constexpr (ST) return tab(st->c, h) + (size_t)(h & kStripMask) * NP;
    else return c + (size_t)h * NP;
  }
  __device__ __forceinline__ double* pptr(int h) const {
    if constexpr (ST) return tab(st->p, h) + (size_t)(h & kStripMask) * 4;
    else return p + (size_t)h * 4;
  }
  __device__ __forceinline__ unsigned* vptr(int h) const {
    if constexpr (ST) return tab(st->ver, h) + (h & kStripMask);
    else return ver + h;
  }
  __device__ __forceinline__ double* ocptr(int h, int NP, double* flat) const {
    if constexpr (ST) return tab(st->oc, h) + (size_t)(h & kStripMask) * NP;
    else return flat + (size_t)h * NP;
  }
  __device__ __forceinline__ double* opptr(int h, double* flat) const {
    if constexpr (ST) return tab(st->op, h) + (size_t)(h & kStripMask) * 4;
    else return flat + (size_t)h * 4;
  }
};

struct BandPlan {
  unsigned* ver;       // per-cell sweep counters (zeroed per launch)
  unsigned* next;      // task counter (zeroed per launch)
  int nsweeps;         // <= 16
  int nbands;          // ceil(nx / 32)
  int dirs[16];
  unsigned dirbits;  // dirs[s] = (dirbits >> 2s) & 3 (no runtime-indexed param array)
  int poll_ns;
  unsigned jitter;  // schedule perturbation seed (race stress tests; 0 = off)
  unsigned long long* trace;  // optional per-task [8] stamps (debug)
  long long trace_cap;
  int nchunks, clen;  // residual mode: diagonal chunks per band and their length
  // strips (nullptr: one flat field).  A launch runs the tasks of the rotated
  // bands [kb, kb + nk) of every sweep, kb = kb_up for i-ascending sweeps and
  // kb_dn for i-descending ones (a rank's own strips); the counters then count
  // from `epoch` (need = epoch + s) and are never reset, and `sys` selects
  // system-scope polls / releases (strips on peer GPUs)
  const StripTab* strips;
  unsigned epoch;
  int kb_up, kb_dn, nk;
  int sys;
  // blocked mode (SolveContext.threads = T > 1 on band-aligned blocks; the
  // reference's threads > 1 sweep, single_level.cpp:130-161, realised
  // deterministically): korder[f * nbands + pos] = the band claimed at
  // position pos of a sweep in frame f (0: i ascending, 1: descending) --
  // blocks in descending rotated order, bands ascending inside a block;
  // bflags[f * nbands + k]: 1 = the band starts a block (its x-upstream halo
  // is the OLD state, that block runs later), 2 = it ends one (the next
  // band's first column is the NEW state, that block ran earlier)
  const short* korder;
  const unsigned char* bflags;
  // the second-order / rhs register kernel (reg_band2.cuh): spatial order 1 | 2, FAS right-hand side
  int order, has_rhs;
};

template <int M>
struct BandLayout {
  static constexpr int N = Gen<M>::N;
  static constexpr int VEC = N * SPV;
  // vectors: 0..11 face groups (L, U, F), 12 S, 13 X, 14 OLD1; the update's
  // V / D are group 1's L / U (update_split)
  static constexpr int V_V = 3, V_S = 12, V_X = 13, V_OLD1 = 14;
  static constexpr int PO = 15 * VEC;  // params of OLD1 [33][4]
  static constexpr int PX = PO + 132;  // params of X [33][4]
  static constexpr int PV = PX + 132;  // params of V [32][4]
  static constexpr int HALO = PV + 128;  // band k-1 new state [N] + params [4]
  static constexpr int HALOP = HALO + N;
  static constexpr int PRE = HALOP + 4;  // 2 blocks [PRE_N][32] of precomputed update scalars
  static constexpr size_t bytes = (size_t)(PRE + 2 * PRE_N * 32) * sizeof(double);
};

template <bool ST = false>
struct BandGeo {
  int nx, ny, k, bw;
  bool i_up, j_up;
  const StripTab* st = nullptr;
  // strip of the halo column (slot -1), of the band's own columns and of the
  // next band's first column (slot bw): strips are whole bands, so a task
  // touches at most these three (set per task by strips_init)
  int r0 = 0, r1 = 0, r2 = 0, i00 = 0, i01 = 0, i02 = 0, w0 = 0, w1 = 0, w2 = 0;
  __device__ __forceinline__ void strip_of(int slot, int* r, int* i0, int* w) const {
    const int ir = min(max(bw * k + slot, 0), nx - 1);
    const int i = i_up ? ir : nx - 1 - ir;
    const int n = __ldg(&st->n);
    int q = 0;
#pragma unroll 1
    for (int t = 1; t < n; ++t) q += i >= __ldg(&st->i0[t]) ? 1 : 0;
    *r = q;
    *i0 = __ldg(&st->i0[q]);
    *w = __ldg(&st->i0[q + 1]) - *i0;
  }
  __device__ __forceinline__ void strips_init() {
    if constexpr (!ST) return;
    strip_of(-1, &r0, &i00, &w0);
    strip_of(0, &r1, &i01, &w1);
    strip_of(bw, &r2, &i02, &w2);
  }
  // rotated cell (ir = 32k + slot, jr = dd - ir) -> cell handle, or -1
  __device__ __forceinline__ int cell(int slot, int dd) const {
    const int ir = bw * k + slot, jr = dd - ir;
    if (ir < 0 || ir >= nx || jr < 0 || jr >= ny) return -1;
    const int i = i_up ? ir : nx - 1 - ir, j = j_up ? jr : ny - 1 - jr;
    if constexpr (!ST) return j * nx + i;
    const int r = slot < 0 ? r0 : (slot >= bw ? r2 : r1);
    const int i0 = slot < 0 ? i00 : (slot >= bw ? i02 : i01);
    const int w = slot < 0 ? w0 : (slot >= bw ? w2 : w1);
    return (r << kStripShift) | (j * w + i - i0);
  }
};

// back-off of the prologue poll (a task may wait for half a sweep; tight
// spinning by the waiting CTAs would load the L2 the running tasks use)
constexpr int kPrologueSleepNs = 512;

// race stress: a pseudo-random 0-2 us sleep of the calling warp (seed != 0)
__device__ __forceinline__ void sched_jitter(unsigned seed, unsigned site) {
  if (!seed) return;
  unsigned h = (unsigned)gtimer() ^ (seed * 0x9e3779b9u) ^ (site * 0x85ebca6bu) ^ (blockIdx.x * 0xc2b2ae35u);
  h ^= h >> 15;
  h *= 0x2c1b3c6du;
  h ^= h >> 12;
  __nanosleep(h & 2047u);
}

__device__ __forceinline__ bool band_stop(const DevErr* err) {
  return *((volatile const int*)&err->code) != 0;
}

// Warp wi of nw loads slots s0 + wi, s0 + wi + nw, ... (< s0 + ns) of
// diagonal dd: coefficient records into vec[k * vstride + (slot - s0)] and
// parameters into prm[(slot - s0) * 4 ..], once the cell's counter reaches
// `need` (0: no wait).  All of a warp's polls, then all of its loads, are in
// flight together.
template <int M, int MAXS, class Addr, class Geo>
__device__ __forceinline__ void band_load(const Addr& fld, const Geo& b, int dd, int s0, int ns,
                                          unsigned need, double* vec, int vstride, double* prm, int wi, int nw,
                                          DevErr* err, int poll_ns, unsigned jit = 0, bool sys = false,
                                          int hi_slot = 1 << 30, unsigned hi_need = 0) {
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3, H = (N + 31) / 32;
  static_assert(MAXS <= 32, "one polling lane per slot");
  constexpr int PR = (4 * MAXS + 31) / 32;  // rounds of parameter loads (4 lanes per slot)
  const int lane = threadIdx.x & 31;
  int my_cell = -1;
  unsigned my_need = need;
  if (lane < MAXS) {
    const int slot = s0 + wi + lane * nw;
    if (slot < s0 + ns) my_cell = b.cell(slot, dd);
    if (slot >= hi_slot) my_need = hi_need;  // (the next band's columns in blocked mode)
  }
  if (jit && need) sched_jitter(jit, (unsigned)dd);
  if (my_need && my_cell >= 0) {
    // relaxed polling, one acquire once satisfied (an acquire per poll
    // measured slower: the spinning warps slow the SM's memory pipeline)
    const unsigned* a = fld.vptr(my_cell);
    long long polls = 0;
    while (ld_relaxed_s(a, Addr::kStrips && sys) < my_need) {
      if (band_stop(err)) break;
      if (++polls > (1LL << 26)) {
        tc::raise(err, E_ERROR, W_DEADLOCK, my_cell % b.nx, my_cell / b.nx, (double)my_need);
        break;
      }
      if (poll_ns) __nanosleep(poll_ns);
    }
    (void)ld_acquire_s(a, Addr::kStrips && sys);
  }
  __syncwarp();
  double r[MAXS][H];
  double pr[PR];
#pragma unroll
  for (int t = 0; t < MAXS; ++t) {
    const int cl = __shfl_sync(0xffffffffu, my_cell, t);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int kk = lane + 32 * h;
      r[t][h] = (cl >= 0 && kk < N) ? __ldcg(fld.cptr(cl, NP) + kk) : 0.0;
    }
  }
#pragma unroll
  for (int rr = 0; rr < PR; ++rr) {
    const int t = (lane + 32 * rr) >> 2;
    const int cl = __shfl_sync(0xffffffffu, my_cell, t < MAXS ? t : 0);
    pr[rr] = (t < MAXS && cl >= 0) ? __ldcg(fld.pptr(cl) + (lane & 3)) : 0.0;
  }
#pragma unroll
  for (int t = 0; t < MAXS; ++t) {
    const int slot = s0 + wi + t * nw;
    if (slot >= s0 + ns) continue;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int kk = lane + 32 * h;
      if (kk < N) vec[kk * vstride + (slot - s0)] = r[t][h];
    }
  }
#pragma unroll
  for (int rr = 0; rr < PR; ++rr) {
    const int t = (lane + 32 * rr) >> 2;
    const int slot = s0 + wi + t * nw;
    if (t < MAXS && slot < s0 + ns && prm) prm[(slot - s0) * 4 + (lane & 3)] = pr[rr];
  }
}

// Update scalars (cell_scalars) of the cells of diagonal dd, whose states
// and bases are in OLD1 / PO, into a PRE block: one step ahead of the cell
// update, by a warp that is otherwise idle, so that pow / sqrt / divisions
// are off the critical path.
template <int M, int BW, class Geo>
__device__ __forceinline__ void band_pre(const DevField& f, const DevCtx& ctx, const Geo& b, int dd,
                                         const double* OLD1, const double* PO, double* pre) {
  const int c = threadIdx.x & 31;
  const int ir = BW * b.k + c, jr = dd - ir;
  const bool valid = c < BW && ir < f.nx && jr >= 0 && jr < f.ny;
  double dt = 0.0, nu = 0.0, qv[3] = {0.0, 0.0, 0.0}, idx = 1.0, idy = 1.0;
  int fail = W_NONE;
  if (valid) {
    const int i = b.i_up ? ir : f.nx - 1 - ir, j = b.j_up ? jr : f.ny - 1 - jr;
    const double dxi = f.dx[i], dyj = f.dy[j];
    P4 cp;
#pragma unroll
    for (int t = 0; t < 4; ++t) cp.v[t] = PO[c * 4 + t];
    fail = cell_scalars(ctx, OLD1 + c, cp, dxi, dyj, &dt, &nu, qv);
    idx = 1.0 / dxi;
    idy = 1.0 / dyj;
  }
  pre[PRE_DT * 32 + c] = dt;
  pre[PRE_NU * 32 + c] = nu;
  pre[PRE_Q0 * 32 + c] = qv[0];
  pre[PRE_Q0 * 32 + 32 + c] = qv[1];
  pre[PRE_Q0 * 32 + 64 + c] = qv[2];
  pre[PRE_FAIL * 32 + c] = (double)fail;
  pre[PRE_IDX * 32 + c] = idx;
  pre[PRE_IDY * 32 + c] = idy;
}

// Write-back of the cells of diagonal dd updated by the previous step: new
// states V (group 1's L, interleaved) and bases PV, for the lanes whose
// update succeeded (ok).  Warp w of 16 stores cells 2w and 2w+1, lane =
// coefficient (coalesced).  Runs at the start of the next step on all warps,
// so the update's critical path ends with its last projection pass.
template <int M, class Addr, class Geo>
__device__ __forceinline__ void band_writeback(const Addr& f, const Geo& b, int dd, const double* V,
                                               const double* PV, const int* ok, int warp) {
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int cc = 2 * warp + t;
    const int cl = ok[cc] ? b.cell(cc, dd) : -1;
    if (cl < 0) continue;
    double* dst = f.cptr(cl, NP);
    double r[(N + 31) / 32];
#pragma unroll
    for (int h = 0; h < (N + 31) / 32; ++h) {
      const int k = lane + 32 * h;
      r[h] = k < N ? V[k * SPV + cc] : 0.0;
    }
#pragma unroll
    for (int h = 0; h < (N + 31) / 32; ++h) {
      const int k = lane + 32 * h;
      if (k < N) __stcg(dst + k, r[h]);
    }
    if (lane < 4) __stcg(f.pptr(cl) + lane, PV[cc * 4 + lane]);
  }
}

// RES = true: the residual (spatial.cpp:135-159) with the same staging and
// face machinery.  Every neighbour is an old state, nothing waits on a
// counter, tasks are (band, chunk of diagonals) so all SMs have work, and the
// previous diagonal's states (V) are the old ones, copied there by group 0
// after it assembles R = Q - sum of the face fluxes, which it stores to `out`.
template <int M, int BW, bool RES = false, bool ST = false>
__global__ void __launch_bounds__(THREADS, 1) k5_band(DevField f, DevCtx ctx, DevErr* err, BandPlan plan,
                                                      DevField out) {
  static_assert(BW == 16 || BW == 32, "band width: 16 or 32 columns");
  constexpr int NS = BW + 1;  // slots of the old-state vectors (one column of band k+1)
  extern __shared__ __align__(128) double smem[];
  __shared__ int s_task, s_stop;
  __shared__ int s_ok[32];  // per-lane success of the last cell update (write-back pending)
  __shared__ unsigned long long s_tr[16];  // debug trace accumulators (thread 0)
  __shared__ unsigned long long s_ph[4];   // debug: face phase stamps of group 0
  __shared__ unsigned long long s_warr[16];  // debug: per-warp arrival at the end-of-step barrier
  using LY = BandLayout<M>;
  constexpr int N = LY::N, VEC = LY::VEC;
  constexpr int NE = NS * N;                         // elements of one NS-slot vector
  constexpr int EPT = (NE + THREADS - 1) / THREADS;  // per thread in the copy phase
  const int tid = threadIdx.x;
  const int warp = tid >> 5, g = warp / P, q = warp % P, c = tid & 31;
  // sweep tasks (sweep, band), then residual tasks (chunk, band): the
  // standalone residual (RES) has only the latter; a fused sweep+residual
  // launch (plan.nchunks > 0) appends them, polling for the final version
  const int sweep_tasks = RES ? 0 : plan.nsweeps * plan.nk;
  const int ntasks = sweep_tasks + plan.nchunks * plan.nk;
  const unsigned ep = plan.epoch;  // counters count from here (0: zeroed per launch)
  const unsigned rneed = RES ? 0u : ep + (unsigned)plan.nsweeps;
  const bool sys = ST && plan.sys != 0;
  const CellAddr<ST> fa{plan.strips, f.c, f.p, plan.ver};
  for (;;) {
    if (tid == 0) {
      sched_jitter(plan.jitter, 1u);
      s_task = (int)atomicAdd(plan.next, 1u);
      s_stop = band_stop(err);
    }
    __syncthreads();
    const int task = s_task;
    if (task >= ntasks || s_stop) return;
    const bool res = task >= sweep_tasks;  // uniform per task
    const int rtask = task - sweep_tasks;
    const int s = res ? plan.nsweeps - 1 : task / plan.nk;
    // residual tasks walk the frame of the last sweep, whose wavefront they follow
    const int dir = (int)((plan.dirbits >> (2 * s)) & 3u);
    const int frame = dir == 0 || dir == 3 ? 0 : 1;
    const int pos = (res ? rtask : task) % plan.nk;
    const int k = (!res && plan.korder) ? (int)plan.korder[frame * plan.nbands + pos]
                                        : (frame == 0 ? plan.kb_up : plan.kb_dn) + pos;
    const int bfl = (!res && plan.bflags) ? (int)plan.bflags[frame * plan.nbands + k] : 0;
    const bool bstart = (bfl & 1) != 0, bend = (bfl & 2) != 0;  // blocked mode (see BandPlan)
    BandGeo<ST> b;
    b.nx = f.nx;
    b.ny = f.ny;
    b.k = k;
    b.bw = BW;
    b.i_up = dir == 0 || dir == 3;  // kSweepDirs (single_level.cpp:116-117)
    b.j_up = dir == 0 || dir == 1;
    b.st = plan.strips;
    b.strips_init();
    const int ir = BW * k + c;
    int dfirst = BW * k, dlast = min(BW * k + BW - 1, f.nx - 1) + f.ny - 1;
    if (res) {
      dfirst += (rtask / plan.nk) * plan.clen;
      dlast = min(dlast, dfirst + plan.clen - 1);
      if (dfirst > dlast) {  // empty chunk of a partial band
        __syncthreads();
        continue;
      }
    }
    const bool tr = plan.trace && 4 * task + 3 < plan.trace_cap && tid == 0;
    if (tr) {
      s_tr[0] = gtimer();
      for (int t = 2; t < 16; ++t) s_tr[t] = 0;
    }
    if (plan.trace && 4 * task + 3 < plan.trace_cap && c == 0) s_warr[warp] = 0;
    // prologue: warp 0 alone waits (with back-off) for the cells of the
    // first two diagonals and band k-1's halo cell, then every warp loads
    // OLD1 <- old(dfirst), X <- old(dfirst+1), HALO <- band k-1 at dfirst-1
    if (!res && warp == 0) {
      for (int e = c; e < 2 * NS + 1; e += 32) {
        const int cl = e < 2 * NS ? b.cell(e % NS, dfirst + e / NS) : (k > 0 ? b.cell(-1, dfirst - 1) : -1);
        // halo: new (old at a block start); row dfirst+1's slot NS-1: old (new at a block end)
        const unsigned need = ep + (e < 2 * NS ? (unsigned)s + (bend && e == 2 * NS - 1 ? 1u : 0u)
                                                : (unsigned)s + (bstart ? 0u : 1u));
        if (cl >= 0 && need) {
          long long polls = 0;
          const unsigned* a = fa.vptr(cl);
          while (ld_relaxed_s(a, ST && sys) < need) {
            if (band_stop(err)) break;
            if (++polls > (1LL << 26)) {
              tc::raise(err, E_ERROR, W_DEADLOCK, cl % f.nx, cl / f.nx, (double)need);
              break;
            }
            __nanosleep(kPrologueSleepNs);
          }
          (void)ld_acquire_s(a, ST && sys);
        }
      }
    }
    __syncthreads();
    const unsigned pn = res ? rneed : 0u;  // sweep tasks polled above
    band_load<M, 4>(fa, b, dfirst, 0, NS, pn, smem + LY::V_OLD1 * VEC, SPV, smem + LY::PO, warp, 16, err,
                    kPrologueSleepNs);
    band_load<M, 4>(fa, b, dfirst + 1, 0, NS, pn, smem + LY::V_X * VEC, SPV, smem + LY::PX, warp, 16, err,
                    kPrologueSleepNs);
    if (k > 0 && warp == 15)
      band_load<M, 1>(fa, b, dfirst - 1, -1, 1, pn, smem + LY::HALO, 1, smem + LY::HALOP, 0, 1, err,
                      kPrologueSleepNs);
    if (res)  // a chunk may start mid-band: its upstream states are old(dfirst-1)
      band_load<M, 2>(fa, b, dfirst - 1, 0, BW, pn, smem + LY::V_V * VEC, SPV, smem + LY::PV, warp, 16,
                      err, kPrologueSleepNs);
    __syncthreads();
    if (warp == 4)
      band_pre<M, BW>(f, ctx, b, dfirst, smem + LY::V_OLD1 * VEC, smem + LY::PO, smem + LY::PRE + (dfirst & 1) * PRE_N * 32);
    __syncthreads();  // (A) of the first step overwrites OLD1 / PO
    if (tr) {
      s_tr[1] = gtimer();
      s_tr[10] = clock64();
    }
    for (int d = dfirst; d <= dlast; ++d) {
      if (tr) s_tr[3] = gtimer();
      // write-back of step d-1 (V is read here before (A) overwrites it)
      if (!res && d > dfirst) band_writeback<M>(fa, b, d - 1, smem + LY::V_V * VEC, smem + LY::PV, s_ok, warp);
      // ---- (A) stage the step's face states.  Sources: OLD1 (own old
      // states), X (old states of diagonal d+1), V (= L of group 1: new
      // states of d-1) and HALO.  Every destination except group 1's L is
      // written at once; those values are held over one barrier because
      // group 1's L is where V lives.
      double hold[EPT];
      {
        const double* OLD1 = smem + LY::V_OLD1 * VEC;
        const double* X = smem + LY::V_X * VEC;
        const double* Vv = smem + LY::V_V * VEC;
        const double* HALO = smem + LY::HALO;
        const int gux = b.i_up ? 0 : 1, guy = b.j_up ? 2 : 3;  // upstream face groups
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
          const int e = tid + r * THREADS;
          hold[r] = 0.0;
          if (e < NE) {
            const int kk = e / NS, sl = e - kk * NS;
            const int o = kk * SPV + sl;
            const double x = X[o];
            if (sl < BW) {
              const double self = OLD1[o];
              const double xu = sl ? Vv[o - 1] : HALO[kk];
              const double yu = Vv[o];
              const double xd = X[o + 1];
              const int irs = BW * k + sl, jrs = d - irs;
              const bool sxu = irs >= 1, sxd = irs + 1 < f.nx, syu = jrs >= 1, syd = jrs + 1 < f.ny;
              smem[LY::V_S * VEC + o] = self;
              // face group gg: the neighbour is the lower cell of a low face
              // (L) and the upper cell of a high face (U); walls take L = self
#pragma unroll
              for (int gg = 0; gg < 4; ++gg) {
                const bool up = gg == ((gg >> 1) == 0 ? gux : guy);
                const bool has = (gg >> 1) == 0 ? (up ? sxu : sxd) : (up ? syu : syd);
                const double nbv = (gg >> 1) == 0 ? (up ? xu : xd) : (up ? yu : x);
                const bool low = (gg & 1) == 0;
                const double lv = (has && low) ? nbv : self;
                if (gg != 1) smem[(gg * 3) * VEC + o] = lv;
                else hold[r] = lv;
                smem[(gg * 3 + 1) * VEC + o] = low ? self : nbv;
              }
            }
            smem[LY::V_OLD1 * VEC + o] = x;
          }
        }
      }
      // this lane's parameters and geometry
      const int jr = d - ir;
      const bool valid = c < BW && ir < f.nx && jr >= 0 && jr < f.ny;
      const int i = valid ? (b.i_up ? ir : f.nx - 1 - ir) : 0;
      const int j = valid ? (b.j_up ? jr : f.ny - 1 - jr) : 0;
      P4 cp, lp, rp;
      int branch;
      {
        const int axis = g >> 1;
        const bool up = g == (axis == 0 ? (b.i_up ? 0 : 1) : (b.j_up ? 2 : 3));
        const bool has_nb = axis == 0 ? (up ? ir >= 1 : ir + 1 < f.nx) : (up ? jr >= 1 : jr + 1 < f.ny);
        // neighbour parameters: upstream = new (PV / HALOP), downstream = old (PX)
        const int off = up ? (axis == 0 ? (c ? LY::PV + (c - 1) * 4 : LY::HALOP) : LY::PV + c * 4)
                           : LY::PX + (axis == 0 ? c + 1 : c) * 4;
        P4 nb;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          cp.v[t] = smem[LY::PO + c * 4 + t];
          nb.v[t] = smem[off + t];
        }
        branch = !valid ? B_NONE : (has_nb ? B_HALF : B_WALL);
        const bool low = (g & 1) == 0;  // low face: L is the neighbour
        lp = low ? nb : cp;
        rp = low ? cp : nb;
      }
      const double dxi = 1.0, dyj = 1.0;  // the update takes 1/dx, 1/dy and dt from PRE
      __syncthreads();
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const int e = tid + r * THREADS;
        if (e < NE) {
          const int kk = e / NS, sl = e - kk * NS;
          if (sl < BW) smem[3 * VEC + kk * SPV + sl] = hold[r];
        }
      }
      if (tid < 4 * NS) smem[LY::PO + tid] = smem[LY::PX + tid];
      __syncthreads();
      if (tr) s_tr[4] += gtimer() - s_tr[3];
      // ---- (B) face fluxes (face_flux / wall_flux, back into the cell basis)
      {
        double* L = smem + (g * 3) * VEC + c;
        const int w = face_core<M>(ctx, g, q, g >> 1, g & 1, branch, W_NONE, lp, rp, cp, L, L + VEC, L + 2 * VEC,
                                   tr && g == 0 ? s_ph : nullptr);
        if (w && valid && q == 0) tc::raise(err, tc::code_for(w), w, i, j, 0.0);
      }
      __syncthreads();
      if (tr) {
        s_tr[5] += gtimer() - s_tr[3];
        s_tr[8] += s_ph[1] - s_tr[3];
        s_tr[9] += s_ph[2] - s_tr[3];
      }
      // ---- (C) face group 0: cell update (update_split); groups 1-3:
      // publish the previous step's cells, band k-1's new cell and old(d+2)
      // for the next step, update scalars of d+1
      if (res && g == 0) {
        // residual: R = Q - sum of the face fluxes into D (group 1's U) and
        // V <- S (old states of d for the next diagonal's upstream faces)
        const double* pre = smem + LY::PRE + (d & 1) * PRE_N * 32 + c;
        const int w = valid ? (int)pre[PRE_FAIL * 32] : W_NONE;
        double* S = smem + LY::V_S * VEC + c;
        double* V = smem + LY::V_V * VEC + c;
        double* D = V + VEC;
        if (valid && w == W_NONE) {
          const double qv[3] = {pre[PRE_Q0 * 32], pre[PRE_Q0 * 32 + 32], pre[PRE_Q0 * 32 + 64]};
#define RS_AS(Q)                                                                                              \
  Part<M, Q>::assemble(S, nullptr, smem + 2 * VEC + c, smem + 5 * VEC + c, smem + 8 * VEC + c,                \
                       smem + 11 * VEC + c, pre[PRE_NU * 32], ctx.collision == 2, ctx.shakhov_w, qv,         \
                       pre[PRE_IDX * 32], pre[PRE_IDY * 32], 0.0, false, D, V)
          SP_DISPATCH(q, RS_AS)
#undef RS_AS
        }
        if (w && valid && q == 0) tc::raise(err, tc::code_for(w), w, i, j, 0.0);
#define RS_CP(Q) Part<M, Q>::copy(S, V)
        SP_DISPATCH(q, RS_CP)
#undef RS_CP
        gbar(0);
        {  // coalesced store of R: warp q stores cells 8q..8q+7, lane = coefficient
          constexpr int NP = (N + 3) & ~3;
          const bool ok = valid && w == W_NONE;
          const int cell = valid ? b.cell(c, d) : 0;
          if (ok && q == 0) {
            double* op = fa.opptr(cell, out.p);
            __stcg(reinterpret_cast<double2*>(op), make_double2(cp.v[0], cp.v[1]));
            __stcg(reinterpret_cast<double2*>(op) + 1, make_double2(cp.v[2], cp.v[3]));
          }
          const double* Db = D - c;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int cc = 8 * q + t;
            const int okc = __shfl_sync(0xffffffffu, ok ? 1 : 0, cc);
            const int bc = __shfl_sync(0xffffffffu, cell, cc);
            if (!okc) continue;
            double* dst = fa.ocptr(bc, NP, out.c);
#pragma unroll
            for (int h = 0; h < (N + 31) / 32; ++h) {
              const int kq = c + 32 * h;
              if (kq < N) __stcg(dst + kq, Db[kq * SPV + cc]);
            }
          }
        }
        if (q == 0 && c < BW) {
#pragma unroll
          for (int t = 0; t < 4; ++t) smem[LY::PV + c * 4 + t] = cp.v[t];
        }
      } else if (!res && g <= 1) {
        // residual assembly (update_split's first half) on face groups 0 and 1,
        // each taking half of every partition's elements; then group 0 updates.
        // Group 1 first publishes step d-1 (its write-back happened before the
        // last CTA barrier, so this release orders it: fence cumulativity; the
        // earlier the publication, the shorter band k+1's halo wait)
        if (g == 1 && q == 0 && d > dfirst && c < BW) {
          sched_jitter(plan.jitter, (unsigned)d);
          const int cl = b.cell(c, d - 1);
          if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, ST && sys);
        }
        {
          const double* pre = smem + LY::PRE + (d & 1) * PRE_N * 32 + c;
          if (valid && (int)pre[PRE_FAIL * 32] == W_NONE) {
            const double qv[3] = {pre[PRE_Q0 * 32], pre[PRE_Q0 * 32 + 32], pre[PRE_Q0 * 32 + 64]};
            double* S = smem + LY::V_S * VEC + c;
            double* V = smem + LY::V_V * VEC + c;
#define B8_AS(Q)                                                                                                \
  {                                                                                                             \
    using PQ = Part<M, Q>;                                                                                      \
    if (g == 0)                                                                                                 \
      PQ::template assemble<0, PQ::CNT / 2>(S, nullptr, smem + 2 * VEC + c, smem + 5 * VEC + c,               \
                                            smem + 8 * VEC + c, smem + 11 * VEC + c, pre[PRE_NU * 32],        \
                                            ctx.collision == 2, ctx.shakhov_w, qv, pre[PRE_IDX * 32],         \
                                            pre[PRE_IDY * 32], pre[PRE_DT * 32], false, V + VEC, V);          \
    else                                                                                                        \
      PQ::template assemble<PQ::CNT / 2, PQ::CNT>(S, nullptr, smem + 2 * VEC + c, smem + 5 * VEC + c,         \
                                                  smem + 8 * VEC + c, smem + 11 * VEC + c, pre[PRE_NU * 32],  \
                                                  ctx.collision == 2, ctx.shakhov_w, qv, pre[PRE_IDX * 32],   \
                                                  pre[PRE_IDY * 32], pre[PRE_DT * 32], false, V + VEC, V);    \
  }
            SP_DISPATCH(q, B8_AS)
#undef B8_AS
          }
          asm volatile("barrier.cta.sync 6, 256;" ::: "memory");  // groups 0 and 1
        }
        if (g == 1 && q == 1 && d + 1 <= dlast)  // OLD1 / PO hold diagonal d+1 since (A)
          band_pre<M, BW>(f, ctx, b, d + 1, smem + LY::V_OLD1 * VEC, smem + LY::PO,
                          smem + LY::PRE + ((d + 1) & 1) * PRE_N * 32);
      }
      if (!res && g == 0) {
        double bad = 0.0;
        P4 np = cp;
        const int w = update_split<M>(f, nullptr, ctx, q, valid, i, j, smem, &bad, cp, dxi, dyj, &np,
                                      tr ? s_tr + 3 : nullptr, smem + LY::PRE + (d & 1) * PRE_N * 32 + c, s_ok,
                                      true);
        if (w && valid && q == 0) tc::raise(err, tc::code_for(w), w, i, j, bad);
        if (tr) s_tr[7] += gtimer() - s_tr[3];
        if (q == 0 && c < BW) {
#pragma unroll
          for (int t = 0; t < 4; ++t) smem[LY::PV + c * 4 + t] = np.v[t];
        }
      } else if (res ? g >= 1 : g >= 2) {
        // prefetch warps: groups 1-3 in residual mode, 2-3 in the sweep
        const int pw0 = res ? 4 : 8, npw = 16 - pw0;
        const int wi = warp - pw0;
        const int stop_now = wi == 0 && c == 0 ? band_stop(err) : 0;  // issued early, consumed last
        // publish step d-1: its write-back happened before the last CTA
        // barrier, so this release orders it (fence cumulativity) and the
        // update's critical path carries no memory fence

        if (d + 1 <= dlast)
          band_load<M, 5>(fa, b, d + 2, 0, NS, res ? rneed : ep + (unsigned)s, smem + LY::V_X * VEC, SPV,
                          smem + LY::PX, wi, npw, err, plan.poll_ns, plan.jitter, sys,
                          bend ? NS - 1 : 1 << 30, ep + (unsigned)s + 1u);
        if (res && wi == 0 && d + 1 <= dlast)  // (the sweep: group 1 does this)
          band_pre<M, BW>(f, ctx, b, d + 1, smem + LY::V_OLD1 * VEC, smem + LY::PO,
                          smem + LY::PRE + ((d + 1) & 1) * PRE_N * 32);
        // band k-1's new cell last: by then it is (nearly always) published
        if (k > 0 && wi == npw - 1 && d + 1 <= dlast)
          band_load<M, 1>(fa, b, d, -1, 1, res ? rneed : ep + (unsigned)s + (bstart ? 0u : 1u), smem + LY::HALO, 1,
                          smem + LY::HALOP, 0, 1, err, plan.poll_ns, plan.jitter, sys);
        if (wi == 0 && c == 0) {
          s_stop = stop_now;
          if (plan.trace && 4 * task + 3 < plan.trace_cap) s_tr[2] += gtimer() - s_tr[3];
        }
      }
      if (plan.trace && 4 * task + 3 < plan.trace_cap && c == 0) s_warr[warp] += gtimer() - s_tr[3];
      __syncthreads();
      if (tr) s_tr[6] += gtimer() - s_tr[3];
      if (s_stop) return;
    }
    if (!res) band_writeback<M>(fa, b, dlast, smem + LY::V_V * VEC, smem + LY::PV, s_ok, warp);
    __syncthreads();
    if (!res && warp == 4 && c < BW) {  // publish the last step
      const int cl = b.cell(c, dlast);
      if (cl >= 0) st_release_s(fa.vptr(cl), ep + (unsigned)s + 1u, ST && sys);
    }
    if (tr) {
      unsigned long long* o = plan.trace + (size_t)task * 32;
      // [loop start, end, steps | s << 20 | k << 28, sums from step start
      //  to: copies, faces, update, prefetch, step end]
      o[0] = s_tr[1];
      o[1] = gtimer();
      s_tr[10] = clock64() - s_tr[10];  // SM cycles over the loop (effective clock)
      o[2] = (unsigned long long)(dlast - dfirst + 1) | ((unsigned long long)s << 20) | ((unsigned long long)k << 28);
      o[3] = s_tr[4];
      o[4] = s_tr[5];
      o[5] = s_tr[7];
      o[6] = s_tr[2];
      o[7] = s_tr[6];
      for (int t = 8; t < 16; ++t) o[t] = s_tr[t];
      for (int t = 0; t < 16; ++t) o[16 + t] = s_warr[t];
    }
  }
}

}  // namespace sp
}  // namespace momg_gpu
