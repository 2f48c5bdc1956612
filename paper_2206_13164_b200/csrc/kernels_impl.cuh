// Templated per-cell kernels of the hot path (instantiated once per moment
// order in kernels_m<M>.cu so the orders compile in parallel).
//
//   K1 k_residual        residual()            spatial.cpp:135-159
//   K2 k_sweep_diag      fast_sweep_step()     single_level.cpp:121-166
//      (one anti-diagonal per launch; the default is the persistent dataflow
//       sweep of sweep_persistent.cuh)
//   K3 k_restrict_sol    restrict_solution()   multigrid.cpp:67-112
//      k_restrict_res    restrict_residual()   multigrid.cpp:114-142
//   K4 k_fas_correct     fas_correct()         multigrid.cpp:144-164
//   K6 k_norm_partial    residual_norm()       multigrid.cpp:202-218
//   K7 k_defect          nmg_cycle's defect    multigrid.cpp:178-185
//
// One warp per cell, WPB warps per block; every kernel early-exits when the
// device error record is set, so the host may defer error checks to where the
// reference's exceptions would surface.
#pragma once

#include "momg_cell.cuh"
#include "runtime.h"
#include "sweep_persistent.cuh"
#include "kernels_v3.cuh"
#include "split_cell.cuh"
#include "band_sweep.cuh"
#include "reg_band.cuh"
#include "transfer.cuh"
#include "band2.h"

namespace momg_gpu {

constexpr int WPB = 4;  // warps per block for the per-cell kernels

// ------------------------------------------------------------------- K1
template <int M, int ORDER>
__global__ void __launch_bounds__(WPB * 32) k_residual(DevField f, DevField out, DevCtx ctx,
                                                       DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M, ORDER>(smem_raw, &ctx, &f, &out, nullptr, nullptr);
  WarpBuf<M, ORDER>& sb = warp_buf<M, ORDER>(bv);
  const DevField* F = &bv.hdr->f;
  const int cells = f.nx * f.ny;
  for (int cell = blockIdx.x * WPB + (threadIdx.x >> 5); cell < cells; cell += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int i = cell % f.nx, j = cell / f.nx;
    load_stencil<M, ORDER>(F, i, j, sb);
    double R[Cfg<M>::T];
    const int w = cell_residual<M, ORDER>(F, &bv.hdr->ctx, bv.tab, i, j, sb, R);
    if (w) {
      if (lane_id() == 0) raise_err(err, code_of(w), w, i, j, 0.0);
      return;
    }
    store_cell_regs<M>(&bv.hdr->g, cell, R, sb.cp[0]);
    __syncwarp();
  }
}

// ------------------------------------------------------------------- K2
// One anti-diagonal of sweep direction (i_up, j_up): the cells with
// ii + jj = d, ii = i_up ? i : nx-1-i, jj = j_up ? j : ny-1-j.  Cells on one
// anti-diagonal are independent (cross stencil), so successive launches give
// exactly the lexicographic Gauss-Seidel order of single_level.cpp:146-153.
template <int M, int ORDER>
__global__ void __launch_bounds__(WPB * 32) k_sweep_diag(DevField f, DevField rhs, int has_rhs,
                                                         DevCtx ctx, DevErr* err, int i_up,
                                                         int j_up, int d, int ii0, int count) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (err_set(err)) return;
  const BlockView bv = block_setup<M, ORDER>(smem_raw, &ctx, &f, &rhs, nullptr, nullptr);
  const int q = blockIdx.x * WPB + (threadIdx.x >> 5);
  if (q >= count) return;
  WarpBuf<M, ORDER>& sb = warp_buf<M, ORDER>(bv);
  const int ii = ii0 + q, jj = d - ii;
  const int i = i_up ? ii : f.nx - 1 - ii;
  const int j = j_up ? jj : f.ny - 1 - jj;
  double bad = 0.0;
  load_stencil<M, ORDER>(&bv.hdr->f, i, j, sb);
  const int w = sweep_cell<M, ORDER>(&bv.hdr->f, has_rhs ? &bv.hdr->g : nullptr, &bv.hdr->ctx,
                                     bv.tab, i, j, sb, &bad);
  if (w && lane_id() == 0) raise_err(err, code_of(w), w, i, j, bad);
}

// ------------------------------------------------------------------- K3
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_restrict_sol(DevField fine, DevField coarse,
                                                           DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M, 1>(smem_raw, nullptr, &fine, &coarse, nullptr, nullptr);
  WarpBuf<M, 1>& sb = warp_buf<M, 1>(bv);
  constexpr int T = Cfg<M>::T;
  const int lane = lane_id();
  const int cells = coarse.nx * coarse.ny;
  for (int K = blockIdx.x * WPB + (threadIdx.x >> 5); K < cells; K += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int I = K % coarse.nx, J = K / coarse.nx;
    double area[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      area[c] = fine.dx[i] * fine.dy[j];
      load_cell_async<M>(&bv.hdr->f, (size_t)j * fine.nx + i, sb.cell[c], sb.cp[c]);
    }
    __syncwarp();
    // conservation of mass, momentum, energy over the children (multigrid.cpp:83-93)
    double S = 0.0, mass = 0.0, energy = 0.0, mom[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double rho = sb.cell[c][0];
      const double* u = sb.cp[c];
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
      if (lane == 0) raise_err(err, E_NONPHYSICAL, W_RESTRICT, I, J, rho_H);
      return;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) proj_coeffs<M>(p4(sb.cp[c]), basis, sb.c[c]);
    __syncwarp();
    double acc[T], v[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = 0.0;
    for (int c = 0; c < 4; ++c) {
      project_apply<M>(bv.tab, sb.cell[c], sb.X1, sb.X2, sb.c[c], pass_mask(p4(sb.cp[c]), basis), v);
      const double wgt = area[c] / S;
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] = fma(wgt, v[t], acc[t]);
    }
    __syncwarp();
    store_items<M>(sb.LA, acc);
    if (lane < 4) sb.par[lane] = basis.v[lane];
    __syncwarp();
    double bad = 0.0;
    const double* res;
    const int w = grad_normalize<M, 1>(bv.tab, sb, sb.LA, sb.X1, sb.X2, sb.par, acc, &bad, &res);
    if (w) {
      if (lane == 0) raise_err(err, code_of(w), w, I, J, bad);
      return;
    }
    store_cell_regs<M>(&bv.hdr->g, K, acc, sb.par);
    __syncwarp();
  }
}

template <int M>
__global__ void __launch_bounds__(WPB * 32) k_restrict_res(DevField arrays, DevField coarse,
                                                           DevField out, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M, 1>(smem_raw, nullptr, &arrays, &coarse, &out, nullptr);
  WarpBuf<M, 1>& sb = warp_buf<M, 1>(bv);
  constexpr int T = Cfg<M>::T;
  const int lane = lane_id();
  const int cells = coarse.nx * coarse.ny;
  for (int K = blockIdx.x * WPB + (threadIdx.x >> 5); K < cells; K += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int I = K % coarse.nx, J = K / coarse.nx;
    P4 basis;
#pragma unroll
    for (int q = 0; q < 4; ++q) basis.v[q] = ldg_cg(coarse.p + (size_t)K * 4 + q);
    double S = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      S += arrays.dx[i] * arrays.dy[j];
      load_cell_async<M>(&bv.hdr->f, (size_t)j * arrays.nx + i, sb.cell[c], sb.cp[c]);
    }
    __syncwarp();
    if (!(basis.v[3] > 0.0)) {
      if (lane == 0) raise_err(err, E_NONPHYSICAL, W_PROJ_SPREAD, I, J, basis.v[3]);
      return;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) proj_coeffs<M>(p4(sb.cp[c]), basis, sb.c[c]);
    __syncwarp();
    double acc[T], v[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = 0.0;
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      project_apply<M>(bv.tab, sb.cell[c], sb.X1, sb.X2, sb.c[c], pass_mask(p4(sb.cp[c]), basis), v);
      const double wgt = (arrays.dx[i] * arrays.dy[j]) / S;
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] = fma(wgt, v[t], acc[t]);
    }
    store_cell_regs<M>(&bv.hdr->h, K, acc, basis.v);
    __syncwarp();
  }
}

// ------------------------------------------------------------------- K4
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_fas_correct(DevField fine, DevField before,
                                                          DevField after, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M, 1>(smem_raw, nullptr, &fine, &before, &after, nullptr);
  WarpBuf<M, 1>& sb = warp_buf<M, 1>(bv);
  constexpr int T = Cfg<M>::T;
  const int lane = lane_id();
  const int cells = fine.nx * fine.ny;
  for (int k = blockIdx.x * WPB + (threadIdx.x >> 5); k < cells; k += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int i = k % fine.nx, j = k / fine.nx;
    const size_t K = (size_t)(j / 2) * before.nx + (i / 2);
    load_cell_async<M>(&bv.hdr->f, k, sb.cell[0], sb.cp[0]);
    load_cell_async<M>(&bv.hdr->h, K, sb.cell[1], sb.cp[1]);
    load_cell_async<M>(&bv.hdr->g, K, sb.cell[2], sb.cp[2]);
    __syncwarp();
    const P4 cp = p4(sb.cp[0]), ap = p4(sb.cp[1]), bp = p4(sb.cp[2]);
    if (!(cp.v[3] > 0.0)) {
      if (lane == 0) raise_err(err, E_NONPHYSICAL, W_PROJ_SPREAD, i, j, cp.v[3]);
      return;
    }
    proj_coeffs<M>(ap, cp, sb.c[0]);
    proj_coeffs<M>(bp, cp, sb.c[1]);
    __syncwarp();
    double va[T], vb[T];
    const double *pa, *pb;
    project_apply2<M>(bv.tab, sb.cell[1], sb.X1, sb.X2, sb.c[0], pass_mask(ap, cp), va,
                      sb.cell[2], sb.Y1, sb.Y2, sb.c[1], pass_mask(bp, cp), vb, &pa, &pb);
    double v[T];
#pragma unroll
    for (int t = 0; t < T; ++t) v[t] = sb.cell[0][item_pos<M>(t)] + (va[t] - vb[t]);
    __syncwarp();
    store_items<M>(sb.LA, v);
    if (lane < 4) sb.par[lane] = cp.v[lane];
    __syncwarp();
    double bad = 0.0;
    const double* res;
    int w = grad_normalize<M, 1>(bv.tab, sb, sb.LA, sb.X1, sb.X2, sb.par, v, &bad, &res);
    if (w) {
      if (code_of(w) == E_NONPHYSICAL) w = W_FAS;
      if (lane == 0) raise_err(err, code_of(w), w, i, j, bad);
      return;
    }
    store_cell_regs<M>(&bv.hdr->f, k, v, sb.par);
    __syncwarp();
  }
}

// ------------------------------------------------------------------- K7
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_defect(DevField res, DevField rhs, int has_rhs,
                                                     DevField out, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M, 1>(smem_raw, nullptr, &res, &rhs, &out, nullptr);
  WarpBuf<M, 1>& sb = warp_buf<M, 1>(bv);
  constexpr int T = Cfg<M>::T;
  const int lane = lane_id();
  const int cells = res.nx * res.ny;
  for (int k = blockIdx.x * WPB + (threadIdx.x >> 5); k < cells; k += gridDim.x * WPB) {
    if (err_set(err)) return;
    load_cell_async<M>(&bv.hdr->f, k, sb.cell[0], sb.cp[0]);
    if (has_rhs) load_cell_async<M>(&bv.hdr->g, k, sb.cell[1], sb.cp[1]);
    __syncwarp();
    double v[T];
    if (!has_rhs) {
#pragma unroll
      for (int t = 0; t < T; ++t) v[t] = -sb.cell[0][item_pos<M>(t)];
    } else {
      const P4 rp = p4(sb.cp[0]), hp = p4(sb.cp[1]);
      if (!(rp.v[3] > 0.0)) {
        if (lane == 0) raise_err(err, E_NONPHYSICAL, W_PROJ_SPREAD, k % res.nx, k / res.nx, rp.v[3]);
        return;
      }
      proj_coeffs<M>(hp, rp, sb.c[0]);
      __syncwarp();
      project_apply<M>(bv.tab, sb.cell[1], sb.X1, sb.X2, sb.c[0], pass_mask(hp, rp), v);
#pragma unroll
      for (int t = 0; t < T; ++t) v[t] = v[t] - sb.cell[0][item_pos<M>(t)];
    }
    store_cell_regs<M>(&bv.hdr->h, k, v, sb.cp[0]);
    __syncwarp();
  }
}

// ---------------------------------------------------------- euler_step
// euler_step (single_level.cpp:74-97) for the warp-per-cell orders (7, 8):
// one warp per cell, dt from the device global_dt reduction, the dt/2 retry
// of apply_update (:44-61).
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_euler(DevField f, DevField res, DevField rhs, int has_rhs,
                                                    const double* dt_dev, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M, 1>(smem_raw, nullptr, &f, &res, &rhs, nullptr);
  WarpBuf<M, 1>& sb = warp_buf<M, 1>(bv);
  constexpr int T = Cfg<M>::T;
  const int lane = lane_id();
  const int cells = f.nx * f.ny;
  for (int k = blockIdx.x * WPB + (threadIdx.x >> 5); k < cells; k += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int i = k % f.nx, j = k / f.nx;
    const double dt = ldg_cg(dt_dev);
    load_cell_async<M>(&bv.hdr->f, k, sb.cell[0], sb.cp[0]);
    load_cell_async<M>(&bv.hdr->g, k, sb.cell[1], sb.cp[1]);
    __syncwarp();
    double R[T];
#pragma unroll
    for (int t = 0; t < T; ++t) R[t] = sb.cell[1][item_pos<M>(t)];
    if (has_rhs) {  // update_delta (single_level.cpp:63-70)
      load_cell<M>(&bv.hdr->h, k, sb.UB, sb.par);
      const P4 rp = p4(sb.par), cp = p4(sb.cp[0]);
      proj_coeffs<M>(rp, cp, sb.c[1]);
      __syncwarp();
      double pr[T];
      project_apply<M>(bv.tab, sb.UB, sb.Y1, sb.Y2, sb.c[1], pass_mask(rp, cp), pr);
#pragma unroll
      for (int t = 0; t < T; ++t) R[t] -= pr[t];
    }
    int w = W_NONE;
    double bad = 0.0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      const double step = attempt == 0 ? dt : 0.5 * dt;
      double v[T];
#pragma unroll
      for (int t = 0; t < T; ++t) v[t] = fma(step, R[t], sb.cell[0][item_pos<M>(t)]);
      __syncwarp();
      store_items<M>(sb.X1, v);
      if (lane < 4) sb.par[lane] = sb.cp[0][lane];
      __syncwarp();
      const double* rr;
      w = grad_normalize<M, 1>(bv.tab, sb, sb.X1, sb.X2, sb.Y1, sb.par, v, &bad, &rr);
      if (w == W_NONE) {
        store_cell_regs<M>(&bv.hdr->f, k, v, sb.par);
        __syncwarp();
        break;
      }
      if (code_of(w) != E_NONPHYSICAL) break;
    }
    if (w != W_NONE) {
      if (code_of(w) == E_NONPHYSICAL) w = W_DT_HALVING;
      if (lane == 0) raise_err(err, code_of(w), w, i, j, bad);
      return;
    }
  }
}

// ------------------------------------------------------------------- K6
// residual_norm partials: block b sums the row-major cell chunk b of
// area * sum_k alpha! theta^|alpha| R_k^2 in a fixed order (one warp per cell).
template <int M>
__global__ void k_norm_partial(DevField res, DevField field, double* partial) {
  __shared__ double sh[32];
  const int cells = res.nx * res.ny;
  const int chunk = (cells + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * chunk, hi = min(cells, lo + chunk);
  const int warps = blockDim.x / 32, wid = threadIdx.x >> 5, lane = lane_id();
  double fact[Cfg<M>::T];
  int deg[Cfg<M>::T];
  bool valid[Cfg<M>::T];
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    const int k = lane + 32 * t;
    valid[t] = k < Cfg<M>::N;
    int a1 = 0, a2 = 0, a3 = 0;
    if (valid[t]) decode(k, a1, a2, a3);
    double f = 1.0;
    for (int q = 2; q <= a1; ++q) f *= q;
    for (int q = 2; q <= a2; ++q) f *= q;
    for (int q = 2; q <= a3; ++q) f *= q;
    fact[t] = f;
    deg[t] = a1 + a2 + a3;
  }
  double v = 0.0;
  for (int k = lo + wid; k < hi; k += warps) {
    const int i = k % res.nx, j = k / res.nx;
    const double theta = field.p[(size_t)k * 4 + 3];
    double cell = 0.0;
#pragma unroll
    for (int t = 0; t < Cfg<M>::T; ++t) {
      if (!valid[t]) continue;
      double tp = 1.0;
#pragma unroll
      for (int e = 1; e <= M; ++e)
        if (e <= deg[t]) tp *= theta;
      const double r = res.c[(size_t)k * Cfg<M>::NP + lane + 32 * t];
      cell += fact[t] * tp * r * r;
    }
    for (int o = 16; o > 0; o >>= 1) cell += __shfl_xor_sync(FULL, cell, o);
    if (lane == 0) v += cell * (res.dx[i] * res.dy[j]);
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < warps ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(FULL, t, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}

inline int grid_blocks(int cells) {
  const int need = (cells + WPB - 1) / WPB;
  return need < 148 * 16 ? need : 148 * 16;
}

template <typename K>
inline void set_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Thread-granular path (kernels_v3.cuh) for orders 3..6; warp-per-cell above
// for orders 7, 8 (their per-thread vectors would not fit shared memory).
template <int M>
constexpr bool use_tc() { return M <= 6; }

int tc_sweep_blocks(const void* kernel, size_t smem, int threads = tc::VS);
tc::SegPlan tc_seg_plan(momg_field* f, int seg = tc::SEG);
template <int M>
constexpr bool use_split() { return M <= 5; }
unsigned long long* trace_buffer(long long* cap);
unsigned sched_jitter_seed();
bool blocked_plan(int T, int nx, int band, const short** korder, const unsigned char** bflags);
void band_scratch(momg_field* f, unsigned** ver, unsigned** next);
// the band kernels for M <= 5 (momg_set_sweep_mode 1, the default); mode 2
// runs the thread-per-face / warp-per-cell kernels, mode 0 per-diagonal launches
bool band_sweep_enabled();
// the register-resident band kernel (reg_band.cuh) for first-order exact
// sweeps / residuals of M <= 5 (momg_set_band_kernel: 1 default, 0 k5_band)
bool rb_enabled();
// Resident CTAs of a register-resident band sweep: the exact order keeps
// ~0.8 nk band tasks running (nk = bands per sweep), the CTAs beyond that hold
// tasks that wait for their first dependency.  Two CTAs on the SMs of one TPC
// slow each other down (the 155 KB step loop streams through the shared
// instruction path: 2048^2 fused launch 122 ms at 148 CTAs, 96-98 ms at
// 88-100; the waiting CTAs' polling is not the cause: a 8x longer back-off
// changes nothing), so the grid is capped at min(1.5 nk, 0.65 SMs) and the
// hardware spreads it over the TPCs first.  MOMG_RB_GRID overrides the cap.
int rb_grid_cap(int nb, int nk);

// rb::k9_band (reg_band2.cuh, own translation units rb2_m<M>.cu)
void rb2_launch_m3(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err, const sp::BandPlan& plan,
                   cudaStream_t st);
void rb2_launch_m4(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err, const sp::BandPlan& plan,
                   cudaStream_t st);
void rb2_launch_m5(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err, const sp::BandPlan& plan,
                   cudaStream_t st);
void rb2_launch_m6(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err, const sp::BandPlan& plan,
                   cudaStream_t st);  // 16-column bands

// launch of rb::k8_band (grid: one CTA per SM, at most one per task)
template <int M, bool RES>
void rb_launch(const DevField& f, const DevCtx& ctx, const sp::BandPlan& bp, const DevField& out) {
  static bool attr = false;
  if (!attr) {
    set_smem(rb::k8_band<M, RES>, rb::RLayout<M>::bytes);
    attr = true;
  }
  int nb = tc_sweep_blocks((const void*)rb::k8_band<M, RES>, rb::RLayout<M>::bytes, rb::RT);
  const int tasks = (RES ? 0 : bp.nsweeps * bp.nk) + bp.nchunks * bp.nk;
  if (nb > tasks) nb = tasks;
  if (!RES) nb = rb_grid_cap(nb, bp.nk);
  if (nb < 1) nb = 1;
  rb::k8_band<M, RES><<<nb, rb::RT, rb::RLayout<M>::bytes, momg_rt::stream()>>>(f, ctx, momg_rt::err_dev(), bp,
                                                                                   out);
  momg_rt::count_launch(1);
}

// ---------------------------------------------------- templated launchers
template <int M>
struct Launch {
  static size_t smem(int order) {
    return order == 2 ? BlockSmem<M, 2>::bytes(WPB) : BlockSmem<M, 1>::bytes(WPB);
  }
  static void attrs() {
    static bool done = false;
    if (done) return;
    set_smem(k_residual<M, 1>, smem(1));
    set_smem(k_residual<M, 2>, smem(2));
    set_smem(k_sweep_diag<M, 1>, smem(1));
    set_smem(k_sweep_diag<M, 2>, smem(2));
    set_smem(k_restrict_sol<M>, smem(1));
    set_smem(k_restrict_res<M>, smem(1));
    set_smem(k_fas_correct<M>, smem(1));
    set_smem(k_defect<M>, smem(1));
    set_smem(k_euler<M>, smem(1));
    done = true;
  }
  static void tc_attrs() {
    if constexpr (use_tc<M>()) {
      static bool done = false;
      if (done) return;
      const size_t s = tc::TSmem<M>::bytes;
      set_smem(tc::k3_residual<M, 1>, s);
      set_smem(tc::k3_residual<M, 2>, s);
      set_smem(tc::k3_sweep<M, 1>, s);
      set_smem(tc::k3_sweep<M, 2>, s);
      set_smem(tc::k3_sweep_diag<M, 1>, s);
      set_smem(tc::k3_sweep_diag<M, 2>, s);
      set_smem(tc::k3_restrict_sol<M>, s);
      set_smem(tc::k3_restrict_res<M>, s);
      set_smem(tc::k3_fas<M>, s);
      set_smem(tc::k3_defect<M>, s);
      set_smem(tc::k3_euler<M>, s);
      done = true;
    }
  }
  static int tc_grid(int work, int per_block) {
    const int need = (work + per_block - 1) / per_block;
    return need < 148 * 8 ? need : 148 * 8;
  }
  // fast_sweep_step followed by residual (nmg_cycle, multigrid.cpp:170-176)
  // as ONE band launch: the residual tasks follow the last sweep's wavefront
  // on the SMs the sweep's dependency DAG leaves idle.  Returns false when
  // the fused path does not apply (the caller runs the two operations).
  static bool sweep_res(const DevCtx& ctx, momg_field* f, const int* order, momg_field* out, int iters) {
    if constexpr (use_split<M>()) {
      if (ctx.order == 1 && iters >= 1 && iters <= 4 && band_sweep_enabled() && ctx.collision != 1) {
        static bool battr = false;
        if (!battr) {
          set_smem(sp::k5_band<M, 32>, sp::BandLayout<M>::bytes);
          battr = true;
        }
        sp::BandPlan bp{};
        band_scratch(f, &bp.ver, &bp.next);
        bp.nsweeps = 4 * iters;
        bp.nbands = (f->nx + 31) / 32;
        bp.nk = bp.nbands;
        bp.dirbits = 0;
        for (int s = 0; s < 16; ++s) {
          bp.dirs[s] = order[s & 3];
          bp.dirbits |= (unsigned)(order[s & 3] & 3) << (2 * s);
        }
            bp.jitter = sched_jitter_seed();
        blocked_plan(ctx.threads, f->nx, 32, &bp.korder, &bp.bflags);
        const int ndiag = std::min(31, f->nx - 1) + f->ny;
        bp.nchunks = std::max(1, (2 * 148 + bp.nbands - 1) / bp.nbands);
        bp.clen = (ndiag + bp.nchunks - 1) / bp.nchunks;
        bp.nchunks = (ndiag + bp.clen - 1) / bp.clen;
        if (rb_enabled() && !bp.korder) {
          rb_launch<M, false>(f->dev(), ctx, bp, out->dev());
          return true;
        }
        int nb = tc_sweep_blocks((const void*)sp::k5_band<M, 32>, sp::BandLayout<M>::bytes, sp::THREADS);
        const int tasks = (bp.nsweeps + bp.nchunks) * bp.nbands;
        if (nb > tasks) nb = tasks;
        DevCtx c = ctx;
        sp::k5_band<M, 32><<<nb, sp::THREADS, sp::BandLayout<M>::bytes, momg_rt::stream()>>>(
            f->dev(), c, momg_rt::err_dev(), bp, out->dev());
        momg_rt::count_launch(1);
        return true;
      }
    }
    (void)ctx;
    (void)f;
    (void)order;
    (void)out;
    (void)iters;
    return false;
  }
  static void residual(const DevCtx& ctx, const momg_field* f, momg_field* out) {
    if constexpr (use_split<M>()) {
      if (ctx.order == 1 && band_sweep_enabled() && ctx.collision != 1) {
        // the band kernel in residual mode: (band, diagonal chunk) tasks
        static bool rattr = false;
        if (!rattr) {
          set_smem(sp::k5_band<M, 32, true>, sp::BandLayout<M>::bytes);
          rattr = true;
        }
        sp::BandPlan bp{};
        band_scratch(out, &bp.ver, &bp.next);
        bp.nsweeps = 1;
        bp.nbands = (f->nx + 31) / 32;
        bp.nk = bp.nbands;
        const int ndiag = std::min(31, f->nx - 1) + f->ny;
        bp.nchunks = std::max(1, (2 * 148 + bp.nbands - 1) / bp.nbands);
        bp.clen = (ndiag + bp.nchunks - 1) / bp.nchunks;
        bp.nchunks = (ndiag + bp.clen - 1) / bp.clen;
        if (rb_enabled()) {
          rb_launch<M, true>(f->dev(), ctx, bp, out->dev());
          return;
        }
        const int tasks = bp.nbands * bp.nchunks;
        const int nb = tasks < 148 ? tasks : 148;
        DevCtx c = ctx;
        sp::k5_band<M, 32, true><<<nb, sp::THREADS, sp::BandLayout<M>::bytes, momg_rt::stream()>>>(
            f->dev(), c, momg_rt::err_dev(), bp, out->dev());
        momg_rt::count_launch(1);
        return;
      }
    }
    if constexpr (use_tc<M>()) {
      tc_attrs();
      const int g = tc_grid(f->nx * f->ny, tc::SEG);
      if (ctx.order == 2)
        tc::k3_residual<M, 2><<<g, tc::VS, tc::TSmem<M>::bytes, momg_rt::stream()>>>(f->dev(), out->dev(), ctx, momg_rt::err_dev());
      else
        tc::k3_residual<M, 1><<<g, tc::VS, tc::TSmem<M>::bytes, momg_rt::stream()>>>(f->dev(), out->dev(), ctx, momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    attrs();
    const int g = grid_blocks(f->nx * f->ny);
    if (ctx.order == 2)
      k_residual<M, 2><<<g, WPB * 32, smem(2), momg_rt::stream()>>>(f->dev(), out->dev(), ctx,
                                                                   momg_rt::err_dev());
    else
      k_residual<M, 1><<<g, WPB * 32, smem(1), momg_rt::stream()>>>(f->dev(), out->dev(), ctx,
                                                                   momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void sweep(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int* order) {
    sweep_n(ctx, f, rhs, order, 1);
  }
  // `iters` consecutive fast_sweep_step calls (identical results; the split
  // persistent kernel runs them as one launch so the sweeps overlap)
  static void sweep_n(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int* order, int iters) {
    if constexpr (use_split<M>()) {
      if (!band_sweep_enabled() || ctx.collision == 1 || iters > 4) {
        for (int it = 0; it < iters; ++it) sweep1(ctx, f, rhs, order, 1);
        return;
      }
    } else {
      if constexpr (M == 6) {
        // the register-resident band kernel with 16-column bands (rb2_m6.cu):
        // every exact-order BGK / Shakhov sweep of M = 6 (first or second
        // order, with or without rhs), up to four FS iterations per launch
        if (band_sweep_enabled() && rb_enabled() && ctx.collision != 1 && ctx.threads <= 1 && iters <= 4) {
          sp::BandPlan bp{};
          band_scratch(f, &bp.ver, &bp.next);
          bp.nsweeps = 4 * iters;
          bp.nbands = (f->nx + 15) / 16;
          bp.nk = bp.nbands;
          bp.dirbits = 0;
          for (int s = 0; s < 16; ++s) {
            bp.dirs[s] = order[s & 3];
            bp.dirbits |= (unsigned)(order[s & 3] & 3) << (2 * s);
          }
          bp.order = ctx.order;
          bp.has_rhs = rhs != nullptr;
          bp.jitter = sched_jitter_seed();
          bp.trace = trace_buffer(&bp.trace_cap);
          const DevField fd = f->dev();
          rb2_launch_m6(fd, rhs ? rhs->dev() : fd, ctx, momg_rt::err_dev(), bp, momg_rt::stream());
          momg_rt::count_launch(1);
          return;
        }
      }
      for (int it = 0; it < iters; ++it) sweep1(ctx, f, rhs, order, 1);
      return;
    }
    sweep1(ctx, f, rhs, order, iters);
  }
  static void sweep1(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int* order, int iters) {
    if constexpr (use_tc<M>()) {
      tc_attrs();
      const DevField fd = f->dev();
      const DevField rd = rhs ? rhs->dev() : fd;
      int has_rhs = rhs != nullptr;
      DevErr* err = momg_rt::err_dev();
      DevCtx c = ctx;
      if constexpr (use_split<M>()) {
        // the band kernels (BGK / Shakhov); ES-BGK runs the thread-per-face kernels
        if (band_sweep_enabled() && ctx.collision != 1) {
          if (ctx.order == 1 && !rhs) {
            static bool battr = false;
            if (!battr) {
              set_smem(sp::k5_band<M, 32>, sp::BandLayout<M>::bytes);
              battr = true;
            }
            const int bw = 32;  // columns per band task (16 measured no faster per step: latency-bound)
            sp::BandPlan bp{};
            band_scratch(f, &bp.ver, &bp.next);
            bp.nsweeps = 4 * iters;
            bp.nbands = (f->nx + bw - 1) / bw;
            bp.nk = bp.nbands;
            bp.dirbits = 0;
            for (int s = 0; s < 16; ++s) {
              bp.dirs[s] = order[s & 3];
              bp.dirbits |= (unsigned)(order[s & 3] & 3) << (2 * s);
            }
            bp.jitter = sched_jitter_seed();
            blocked_plan(ctx.threads, f->nx, 32, &bp.korder, &bp.bflags);
            bp.trace = trace_buffer(&bp.trace_cap);
            bp.nchunks = 0;  // no fused residual tasks
            bp.clen = 1;
            if (rb_enabled() && !bp.korder) {
              rb_launch<M, false>(fd, c, bp, fd);
              return;
            }
            int nb = tc_sweep_blocks((const void*)sp::k5_band<M, 32>, sp::BandLayout<M>::bytes, sp::THREADS);
            if (nb > bp.nsweeps * bp.nbands) nb = bp.nsweeps * bp.nbands;
            sp::k5_band<M, 32><<<nb, sp::THREADS, sp::BandLayout<M>::bytes, momg_rt::stream()>>>(fd, c, err, bp, fd);
            momg_rt::count_launch(1);
            return;
          }
          if (rb_enabled() && ctx.threads <= 1) {
            // second order and/or an FAS rhs, exact order: the register-resident kernel
            sp::BandPlan bp{};
            band_scratch(f, &bp.ver, &bp.next);
            bp.nsweeps = 4 * iters;
            bp.nbands = (f->nx + 31) / 32;
            bp.nk = bp.nbands;
            bp.dirbits = 0;
            for (int s = 0; s < 16; ++s) {
              bp.dirs[s] = order[s & 3];
              bp.dirbits |= (unsigned)(order[s & 3] & 3) << (2 * s);
            }
            bp.order = ctx.order;
            bp.has_rhs = rhs != nullptr;
            bp.jitter = sched_jitter_seed();
            bp.trace = trace_buffer(&bp.trace_cap);
            if constexpr (M == 3) rb2_launch_m3(fd, rd, c, err, bp, momg_rt::stream());
            else if constexpr (M == 4) rb2_launch_m4(fd, rd, c, err, bp, momg_rt::stream());
            else rb2_launch_m5(fd, rd, c, err, bp, momg_rt::stream());
            momg_rt::count_launch(1);
            return;
          }
          {
            // second order and/or an FAS rhs: the 16-column band sweep
            sp::Band2Plan bp{};
            band_scratch(f, &bp.ver, &bp.next);
            bp.nsweeps = 4 * iters;
            bp.nbands = (f->nx + 15) / 16;
            bp.nk = bp.nbands;
            bp.dirbits = 0;
            for (int s = 0; s < 16; ++s) bp.dirbits |= (unsigned)(order[s & 3] & 3) << (2 * s);
            bp.order = ctx.order;
            bp.has_rhs = rhs != nullptr;
            blocked_plan(ctx.threads, f->nx, 16, &bp.korder, &bp.bflags);
            bp.jitter = sched_jitter_seed();
            if constexpr (M == 3) band2_launch_m3(fd, rd, c, err, bp, momg_rt::stream());
            else if constexpr (M == 4) band2_launch_m4(fd, rd, c, err, bp, momg_rt::stream());
            else band2_launch_m5(fd, rd, c, err, bp, momg_rt::stream());
            momg_rt::count_launch(1);
            return;
          }
        }
      }
      if (persistent_sweep_enabled()) {
        tc::SegPlan plan = tc_seg_plan(f);
        plan.nsweeps = 4;
        for (int s = 0; s < 8; ++s) plan.dirs[s] = order[s & 3];
        const void* kern = ctx.order == 2 ? (const void*)tc::k3_sweep<M, 2> : (const void*)tc::k3_sweep<M, 1>;
        int nb = tc_sweep_blocks(kern, tc::TSmem<M>::bytes);
        DevField fa = fd, ra = rd;
        void* args[] = {&fa, &ra, &has_rhs, &c, &err, &plan};
        momg_rt::note_launch(cudaLaunchCooperativeKernel(kern, dim3(nb), dim3(tc::VS), args, tc::TSmem<M>::bytes,
                                    momg_rt::stream()));
        momg_rt::count_launch(1);
        return;
      }
      static const int dirs4[4][2] = {{1, 1}, {0, 1}, {0, 0}, {1, 0}};
      const int nx = f->nx, ny = f->ny;
      for (int s = 0; s < 4; ++s) {
        const int* dir = dirs4[order[s]];
        for (int d = 0; d <= nx + ny - 2; ++d) {
          const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
          const int hi = d < nx - 1 ? d : nx - 1;
          const int count = hi - lo + 1;
          const int g = (count + tc::SEG - 1) / tc::SEG;
          if (ctx.order == 2)
            tc::k3_sweep_diag<M, 2><<<g, tc::VS, tc::TSmem<M>::bytes, momg_rt::stream()>>>(
                fd, rd, has_rhs, ctx, err, dir[0], dir[1], d, lo, count);
          else
            tc::k3_sweep_diag<M, 1><<<g, tc::VS, tc::TSmem<M>::bytes, momg_rt::stream()>>>(
                fd, rd, has_rhs, ctx, err, dir[0], dir[1], d, lo, count);
        }
        momg_rt::count_launch(nx + ny - 1);
      }
      return;
    }
    if (persistent_sweep_enabled()) {
      if (ctx.order == 2)
        PersistentSweep<M, 2>::run(ctx, f, rhs, order);
      else
        PersistentSweep<M, 1>::run(ctx, f, rhs, order);
      return;
    }
    attrs();
    static const int dirs[4][2] = {{1, 1}, {0, 1}, {0, 0}, {1, 0}};  // single_level.cpp:116-117
    const DevField fd = f->dev();
    const DevField rd = rhs ? rhs->dev() : fd;
    const int nx = f->nx, ny = f->ny;
    for (int s = 0; s < 4; ++s) {
      const int* dir = dirs[order[s]];
      for (int d = 0; d <= nx + ny - 2; ++d) {
        const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
        const int hi = d < nx - 1 ? d : nx - 1;
        const int count = hi - lo + 1;
        const int g = (count + WPB - 1) / WPB;
        if (ctx.order == 2)
          k_sweep_diag<M, 2><<<g, WPB * 32, smem(2), momg_rt::stream()>>>(
              fd, rd, rhs != nullptr, ctx, momg_rt::err_dev(), dir[0], dir[1], d, lo, count);
        else
          k_sweep_diag<M, 1><<<g, WPB * 32, smem(1), momg_rt::stream()>>>(
              fd, rd, rhs != nullptr, ctx, momg_rt::err_dev(), dir[0], dir[1], d, lo, count);
      }
      momg_rt::count_launch(nx + ny - 1);
    }
  }
  static int xf_grid(int cells) {
    const int need = (cells + xf::XT - 1) / xf::XT;
    return need < 148 * 8 ? need : 148 * 8;
  }
  static void xf_attrs() {
    if constexpr (use_split<M>()) {
      static bool done = false;
      if (done) return;
      done = true;
    }
  }
  static void restrict_sol(const momg_field* fine, momg_field* coarse) {
    if constexpr (use_split<M>()) {  // warp-staged records (transfer.cuh)
      xf_attrs();
      xf::xf_restrict_sol<M><<<xf_grid(coarse->nx * coarse->ny), xf::XT, 0, momg_rt::stream()>>>(
          fine->dev(), coarse->dev(), momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    if constexpr (use_tc<M>()) {
      tc_attrs();
      tc::k3_restrict_sol<M><<<tc_grid(coarse->nx * coarse->ny, tc::VS), tc::VS, tc::TSmem<M>::bytes,
                               momg_rt::stream()>>>(fine->dev(), coarse->dev(), momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    attrs();
    k_restrict_sol<M><<<grid_blocks(coarse->nx * coarse->ny), WPB * 32, smem(1),
                        momg_rt::stream()>>>(fine->dev(), coarse->dev(), momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void restrict_res(const momg_field* arrays, const momg_field* coarse, momg_field* out) {
    if constexpr (use_split<M>()) {
      xf_attrs();
      xf::xf_restrict_res<M><<<xf_grid(coarse->nx * coarse->ny), xf::XT, 0, momg_rt::stream()>>>(
          arrays->dev(), coarse->dev(), out->dev(), momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    if constexpr (use_tc<M>()) {
      tc_attrs();
      tc::k3_restrict_res<M><<<tc_grid(coarse->nx * coarse->ny, tc::VS), tc::VS, tc::TSmem<M>::bytes,
                               momg_rt::stream()>>>(arrays->dev(), coarse->dev(), out->dev(),
                                                    momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    attrs();
    k_restrict_res<M><<<grid_blocks(coarse->nx * coarse->ny), WPB * 32, smem(1),
                        momg_rt::stream()>>>(arrays->dev(), coarse->dev(), out->dev(),
                                             momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void fas(momg_field* fine, const momg_field* before, const momg_field* after) {
    if constexpr (use_split<M>()) {
      xf_attrs();
      xf::xf_fas<M><<<xf_grid(fine->nx * fine->ny), xf::XT, 0, momg_rt::stream()>>>(
          fine->dev(), before->dev(), after->dev(), momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    if constexpr (use_tc<M>()) {
      tc_attrs();
      tc::k3_fas<M><<<tc_grid(fine->nx * fine->ny, tc::VS), tc::VS, tc::TSmem<M>::bytes, momg_rt::stream()>>>(
          fine->dev(), before->dev(), after->dev(), momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    attrs();
    k_fas_correct<M><<<grid_blocks(fine->nx * fine->ny), WPB * 32, smem(1), momg_rt::stream()>>>(
        fine->dev(), before->dev(), after->dev(), momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void defect(const momg_field* res, const momg_field* rhs, momg_field* out) {
    if constexpr (use_tc<M>()) {
      tc_attrs();
      tc::k3_defect<M><<<tc_grid(res->nx * res->ny, tc::VS), tc::VS, tc::TSmem<M>::bytes, momg_rt::stream()>>>(
          res->dev(), rhs ? rhs->dev() : res->dev(), rhs != nullptr, out->dev(), momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    attrs();
    k_defect<M><<<grid_blocks(res->nx * res->ny), WPB * 32, smem(1), momg_rt::stream()>>>(
        res->dev(), rhs ? rhs->dev() : res->dev(), rhs != nullptr, out->dev(),
        momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  // euler_step: dt_dev = device scalar of the global_dt reduction
  static void euler(const momg_field* f_, const momg_field* res, const momg_field* rhs, const double* dt_dev) {
    momg_field* f = const_cast<momg_field*>(f_);
    if constexpr (use_tc<M>()) {
      tc_attrs();
      tc::k3_euler<M><<<tc_grid(f->nx * f->ny, tc::VS), tc::VS, tc::TSmem<M>::bytes, momg_rt::stream()>>>(
          f->dev(), res->dev(), rhs ? rhs->dev() : res->dev(), rhs != nullptr, dt_dev, momg_rt::err_dev());
      momg_rt::count_launch(1);
      return;
    }
    attrs();
    k_euler<M><<<grid_blocks(f->nx * f->ny), WPB * 32, smem(1), momg_rt::stream()>>>(
        f->dev(), res->dev(), rhs ? rhs->dev() : res->dev(), rhs != nullptr, dt_dev, momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void norm_partial(const momg_field* res, const momg_field* field, double* partial,
                           int blocks) {
    k_norm_partial<M><<<blocks, 256, 0, momg_rt::stream()>>>(res->dev(), field->dev(), partial);
    momg_rt::count_launch(1);
  }
  // FS iterations (+ the residual, first order) over a strip partition: one
  // launch for this process's strips (M <= 5, BGK / Shakhov, no rhs): the
  // first-order band kernel, or the second-order one with 16-column bands
  static bool strips_sweep(const DevCtx& ctx, const StripLaunch& L) {
    if constexpr (use_split<M>()) {
      if (ctx.collision == 1 || L.iters < 1 || L.iters > 4 || (ctx.order != 1 && L.with_res)) return false;
      DevCtx c = ctx;
      if (ctx.order == 2) {
        sp::Band2Plan bp{};
        bp.next = L.next;
        bp.nsweeps = 4 * L.iters;
        bp.nbands = 2 * L.nbands;
        for (int s = 0; s < 16; ++s) bp.dirbits |= (unsigned)(L.order[s & 3] & 3) << (2 * s);
        bp.order = 2;
        bp.has_rhs = 0;
        bp.jitter = sched_jitter_seed();
        bp.strips = (const sp::StripTab*)L.tab;
        bp.epoch = L.epoch;
        bp.kb_up = 2 * L.kb_up;
        bp.kb_dn = 2 * L.kb_dn;
        bp.nk = 2 * L.nk;
        bp.sys = L.sys;
        if constexpr (M == 3) band2_strips_launch_m3(L.geo, c, momg_rt::err_dev(), bp, momg_rt::stream());
        else if constexpr (M == 4) band2_strips_launch_m4(L.geo, c, momg_rt::err_dev(), bp, momg_rt::stream());
        else band2_strips_launch_m5(L.geo, c, momg_rt::err_dev(), bp, momg_rt::stream());
        momg_rt::note_launch(cudaGetLastError());
        momg_rt::count_launch(1);
        return true;
      }
      static bool battr = false;
      if (!battr) {
        set_smem(sp::k5_band<M, 32, false, true>, sp::BandLayout<M>::bytes);
        battr = true;
      }
      sp::BandPlan bp{};
      bp.next = L.next;
      bp.nsweeps = 4 * L.iters;
      bp.nbands = L.nbands;
      bp.dirbits = 0;
      for (int s = 0; s < 16; ++s) {
        bp.dirs[s] = L.order[s & 3];
        bp.dirbits |= (unsigned)(L.order[s & 3] & 3) << (2 * s);
      }
      bp.jitter = sched_jitter_seed();
      const int ndiag = std::min(31, L.geo.nx - 1) + L.geo.ny;
      if (L.with_res) {
        bp.nchunks = std::max(1, (2 * 148 + L.nk - 1) / L.nk);
        bp.clen = (ndiag + bp.nchunks - 1) / bp.nchunks;
        bp.nchunks = (ndiag + bp.clen - 1) / bp.clen;
      } else {
        bp.nchunks = 0;
        bp.clen = 1;
      }
      bp.strips = (const sp::StripTab*)L.tab;
      bp.epoch = L.epoch;
      bp.kb_up = L.kb_up;
      bp.kb_dn = L.kb_dn;
      bp.nk = L.nk;
      bp.sys = L.sys;
      int nb = tc_sweep_blocks((const void*)sp::k5_band<M, 32, false, true>, sp::BandLayout<M>::bytes, sp::THREADS);
      const int tasks = (bp.nsweeps + bp.nchunks) * bp.nk;
      if (nb > tasks) nb = tasks;
      DevField none = L.geo;
      none.c = none.p = nullptr;
      sp::k5_band<M, 32, false, true><<<nb, sp::THREADS, sp::BandLayout<M>::bytes, momg_rt::stream()>>>(
          L.geo, c, momg_rt::err_dev(), bp, none);
      momg_rt::note_launch(cudaGetLastError());
      momg_rt::count_launch(1);
      return true;
    }
    (void)ctx;
    (void)L;
    return false;
  }
  static const Ops* ops() {
    static const Ops o = {residual, sweep, restrict_sol, restrict_res, fas, defect, norm_partial, sweep_n, sweep_res,
                          euler, strips_sweep};
    return &o;
  }
};

}  // namespace momg_gpu

#define MOMG_INSTANTIATE(Mv)                                                          \
  namespace momg_gpu {                                                                \
  const Ops* ops_m##Mv() { return Launch<Mv>::ops(); }                                \
  }
