// Templated per-cell kernels of the hot path (instantiated once per moment
// order in kernels_m<M>.cu so the orders compile in parallel).
//
//   K1 k_residual        residual()            spatial.cpp:135-159
//   K2 k_sweep_diag      fast_sweep_step()     single_level.cpp:121-166
//      (one anti-diagonal of one sweep direction per launch; see also the
//       persistent dataflow sweep in sweep_persistent.cuh)
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

namespace momg_gpu {

constexpr int WPB = 4;  // warps per block for the per-cell kernels

// ------------------------------------------------------------------- K1
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_residual(DevField f, DevField out, DevCtx ctx,
                                                       DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M>(smem_raw, &ctx, &f, &out, nullptr, nullptr);
  WarpBuf<M>& sb = warp_buf<M>(bv);
  const DevField* F = &bv.hdr->f;
  const int cells = f.nx * f.ny;
  for (int cell = blockIdx.x * WPB + (threadIdx.x >> 5); cell < cells; cell += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int i = cell % f.nx, j = cell / f.nx;
    load_cell<M>(F, cell, sb.S, sb.cp);
    const int w = cell_residual_smem<M>(F, &bv.hdr->ctx, bv.alpha, i, j, sb.cp, sb);
    if (w) {
      if (lane_id() == 0) raise_err(err, code_of(w), w, i, j, 0.0);
      return;
    }
    store_cell<M>(&bv.hdr->g, cell, sb.R, sb.cp);
  }
}

// ------------------------------------------------------------------- K2
// One anti-diagonal of sweep direction (i_up, j_up): the cells with
// ii + jj = d, ii = i_up ? i : nx-1-i, jj = j_up ? j : ny-1-j.  Cells on one
// anti-diagonal are independent (cross stencil), so successive launches give
// exactly the lexicographic Gauss-Seidel order of single_level.cpp:146-153.
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_sweep_diag(DevField f, DevField rhs, int has_rhs,
                                                         DevCtx ctx, DevErr* err, int i_up,
                                                         int j_up, int d, int ii0, int count) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (err_set(err)) return;
  const BlockView bv = block_setup<M>(smem_raw, &ctx, &f, &rhs, nullptr, nullptr);
  const int q = blockIdx.x * WPB + (threadIdx.x >> 5);
  if (q >= count) return;
  WarpBuf<M>& sb = warp_buf<M>(bv);
  const int ii = ii0 + q, jj = d - ii;
  const int i = i_up ? ii : f.nx - 1 - ii;
  const int j = j_up ? jj : f.ny - 1 - jj;
  double bad = 0.0;
  const int w = sweep_cell_smem<M>(&bv.hdr->f, has_rhs ? &bv.hdr->g : nullptr, &bv.hdr->ctx,
                                   bv.alpha, i, j, sb, &bad);
  if (w && lane_id() == 0) raise_err(err, code_of(w), w, i, j, bad);
}

// ------------------------------------------------------------------- K3
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_restrict_sol(DevField fine, DevField coarse,
                                                           DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M>(smem_raw, nullptr, &fine, &coarse, nullptr, nullptr);
  WarpBuf<M>& sb = warp_buf<M>(bv);
  const DevField* Fi = &bv.hdr->f;
  const int lane = lane_id();
  const int cells = coarse.nx * coarse.ny;
  for (int K = blockIdx.x * WPB + (threadIdx.x >> 5); K < cells; K += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int I = K % coarse.nx, J = K / coarse.nx;
    size_t child[4];
    double area[4];
    double S = 0.0, mass = 0.0, energy = 0.0, mom[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      child[c] = (size_t)j * fine.nx + i;
      area[c] = fine.dx[i] * fine.dy[j];
      const double rho = ldg_cg(fine.c + child[c] * Cfg<M>::NP);
      double u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = ldg_cg(fine.p + child[c] * 4 + q);
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
    for (int k = lane; k < Cfg<M>::N; k += 32) sb.R[k] = 0.0;
    for (int c = 0; c < 4; ++c) {
      load_cell<M>(Fi, child[c], sb.A, sb.par);
      project_smem<M>(bv.alpha, sb.A, sb.A2, p4(sb.par), basis, sb.A);
      const double wgt = area[c] / S;
      for (int k = lane; k < Cfg<M>::N; k += 32) sb.R[k] = fma(wgt, sb.A[k], sb.R[k]);
      __syncwarp();
    }
    if (lane < 4) sb.cp[lane] = basis.v[lane];
    __syncwarp();
    double bad = 0.0;
    const int w = grad_normalize_smem<M>(bv.alpha, sb.R, sb.A2, sb.cp, &bad);
    if (w) {
      if (lane == 0) raise_err(err, code_of(w), w, I, J, bad);
      return;
    }
    store_cell<M>(&bv.hdr->g, K, sb.R, sb.cp);
  }
}

template <int M>
__global__ void __launch_bounds__(WPB * 32) k_restrict_res(DevField arrays, DevField coarse,
                                                           DevField out, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M>(smem_raw, nullptr, &arrays, &coarse, &out, nullptr);
  WarpBuf<M>& sb = warp_buf<M>(bv);
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
    }
    for (int k = lane; k < Cfg<M>::N; k += 32) sb.R[k] = 0.0;
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      load_cell<M>(&bv.hdr->f, (size_t)j * arrays.nx + i, sb.A, sb.par);
      if (!project_smem<M>(bv.alpha, sb.A, sb.A2, p4(sb.par), basis, sb.A)) {
        if (lane == 0) raise_err(err, E_NONPHYSICAL, W_PROJ_SPREAD, I, J, basis.v[3]);
        return;
      }
      const double wgt = (arrays.dx[i] * arrays.dy[j]) / S;
      for (int k = lane; k < Cfg<M>::N; k += 32) sb.R[k] = fma(wgt, sb.A[k], sb.R[k]);
      __syncwarp();
    }
    if (lane < 4) sb.cp[lane] = basis.v[lane];
    __syncwarp();
    store_cell<M>(&bv.hdr->h, K, sb.R, sb.cp);
  }
}

// ------------------------------------------------------------------- K4
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_fas_correct(DevField fine, DevField before,
                                                          DevField after, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M>(smem_raw, nullptr, &fine, &before, &after, nullptr);
  WarpBuf<M>& sb = warp_buf<M>(bv);
  const int lane = lane_id();
  const int cells = fine.nx * fine.ny;
  for (int k = blockIdx.x * WPB + (threadIdx.x >> 5); k < cells; k += gridDim.x * WPB) {
    if (err_set(err)) return;
    const int i = k % fine.nx, j = k / fine.nx;
    const size_t K = (size_t)(j / 2) * before.nx + (i / 2);
    load_cell<M>(&bv.hdr->f, k, sb.S, sb.cp);
    load_cell<M>(&bv.hdr->h, K, sb.A, sb.par);
    load_cell<M>(&bv.hdr->g, K, sb.B, sb.par + 4);
    if (!project_smem<M>(bv.alpha, sb.A, sb.A2, p4(sb.par), p4(sb.cp), sb.A) ||
        !project_smem<M>(bv.alpha, sb.B, sb.B2, p4(sb.par + 4), p4(sb.cp), sb.B)) {
      if (lane == 0) raise_err(err, E_NONPHYSICAL, W_PROJ_SPREAD, i, j, sb.cp[3]);
      return;
    }
    for (int q = lane; q < Cfg<M>::N; q += 32) sb.S[q] += sb.A[q] - sb.B[q];
    __syncwarp();
    double bad = 0.0;
    int w = grad_normalize_smem<M>(bv.alpha, sb.S, sb.A2, sb.cp, &bad);
    if (w) {
      if (code_of(w) == E_NONPHYSICAL) w = W_FAS;
      if (lane == 0) raise_err(err, code_of(w), w, i, j, bad);
      return;
    }
    store_cell<M>(&bv.hdr->f, k, sb.S, sb.cp);
  }
}

// ------------------------------------------------------------------- K7
template <int M>
__global__ void __launch_bounds__(WPB * 32) k_defect(DevField res, DevField rhs, int has_rhs,
                                                     DevField out, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M>(smem_raw, nullptr, &res, &rhs, &out, nullptr);
  WarpBuf<M>& sb = warp_buf<M>(bv);
  const int lane = lane_id();
  const int cells = res.nx * res.ny;
  for (int k = blockIdx.x * WPB + (threadIdx.x >> 5); k < cells; k += gridDim.x * WPB) {
    if (err_set(err)) return;
    load_cell<M>(&bv.hdr->f, k, sb.S, sb.cp);
    if (!has_rhs) {
      for (int q = lane; q < Cfg<M>::N; q += 32) sb.R[q] = -sb.S[q];
    } else {
      load_cell<M>(&bv.hdr->g, k, sb.A, sb.par);
      if (!project_smem<M>(bv.alpha, sb.A, sb.A2, p4(sb.par), p4(sb.cp), sb.A)) {
        if (lane == 0) raise_err(err, E_NONPHYSICAL, W_PROJ_SPREAD, k % res.nx, k / res.nx, sb.cp[3]);
        return;
      }
      for (int q = lane; q < Cfg<M>::N; q += 32) sb.R[q] = sb.A[q] - sb.S[q];
    }
    __syncwarp();
    store_cell<M>(&bv.hdr->h, k, sb.R, sb.cp);
  }
}

// ------------------------------------------------------------------- K6
// residual_norm partials: block b sums the row-major cell chunk b of
// area * sum_k alpha! theta^|alpha| R_k^2 in a fixed order (one warp per cell).
template <int M>
__global__ void k_norm_partial(DevField res, DevField field, double* partial) {
  __shared__ double sh[32];
  __shared__ uint32_t alpha[Cfg<M>::N];
  build_alpha<M>(alpha);
  __syncthreads();
  const Items<M> it(alpha);
  const int cells = res.nx * res.ny;
  const int chunk = (cells + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * chunk, hi = min(cells, lo + chunk);
  const int warps = blockDim.x / 32, wid = threadIdx.x >> 5, lane = lane_id();
  double fact[Cfg<M>::T];
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    double f = 1.0;
    for (int q = 2; q <= it.a1(t); ++q) f *= q;
    for (int q = 2; q <= it.a2(t); ++q) f *= q;
    for (int q = 2; q <= it.a3(t); ++q) f *= q;
    fact[t] = f;
  }
  double v = 0.0;
  for (int k = lo + wid; k < hi; k += warps) {
    const int i = k % res.nx, j = k / res.nx;
    const double theta = field.p[(size_t)k * 4 + 3];
    double cell = 0.0;
#pragma unroll
    for (int t = 0; t < Cfg<M>::T; ++t) {
      if (!it.v(t)) continue;
      double tp = 1.0;
      const int dg = it.deg(t);
#pragma unroll
      for (int e = 1; e <= M; ++e)
        if (e <= dg) tp *= theta;
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

// ---------------------------------------------------- templated launchers
template <int M>
struct Launch {
  static size_t smem() { return BlockSmem<M>::bytes(WPB); }
  static void attrs() {
    static bool done = false;
    if (done) return;
    const int s = (int)smem();
    cudaFuncSetAttribute(k_residual<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
    cudaFuncSetAttribute(k_sweep_diag<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
    cudaFuncSetAttribute(k_restrict_sol<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
    cudaFuncSetAttribute(k_restrict_res<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
    cudaFuncSetAttribute(k_fas_correct<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
    cudaFuncSetAttribute(k_defect<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
    done = true;
  }
  static void residual(const DevCtx& ctx, const momg_field* f, momg_field* out) {
    attrs();
    k_residual<M><<<grid_blocks(f->nx * f->ny), WPB * 32, smem(), momg_rt::stream()>>>(
        f->dev(), out->dev(), ctx, momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void sweep(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int* order) {
    if (persistent_sweep_enabled()) {
      PersistentSweep<M>::run(ctx, f, rhs, order);
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
        k_sweep_diag<M><<<(count + WPB - 1) / WPB, WPB * 32, smem(), momg_rt::stream()>>>(
            fd, rd, rhs != nullptr, ctx, momg_rt::err_dev(), dir[0], dir[1], d, lo, count);
      }
      momg_rt::count_launch(nx + ny - 1);
    }
  }
  static void restrict_sol(const momg_field* fine, momg_field* coarse) {
    attrs();
    k_restrict_sol<M><<<grid_blocks(coarse->nx * coarse->ny), WPB * 32, smem(),
                        momg_rt::stream()>>>(fine->dev(), coarse->dev(), momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void restrict_res(const momg_field* arrays, const momg_field* coarse, momg_field* out) {
    attrs();
    k_restrict_res<M><<<grid_blocks(coarse->nx * coarse->ny), WPB * 32, smem(),
                        momg_rt::stream()>>>(arrays->dev(), coarse->dev(), out->dev(),
                                             momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void fas(momg_field* fine, const momg_field* before, const momg_field* after) {
    attrs();
    k_fas_correct<M><<<grid_blocks(fine->nx * fine->ny), WPB * 32, smem(), momg_rt::stream()>>>(
        fine->dev(), before->dev(), after->dev(), momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void defect(const momg_field* res, const momg_field* rhs, momg_field* out) {
    attrs();
    k_defect<M><<<grid_blocks(res->nx * res->ny), WPB * 32, smem(), momg_rt::stream()>>>(
        res->dev(), rhs ? rhs->dev() : res->dev(), rhs != nullptr, out->dev(),
        momg_rt::err_dev());
    momg_rt::count_launch(1);
  }
  static void norm_partial(const momg_field* res, const momg_field* field, double* partial,
                           int blocks) {
    k_norm_partial<M><<<blocks, 256, 0, momg_rt::stream()>>>(res->dev(), field->dev(), partial);
    momg_rt::count_launch(1);
  }
  static const Ops* ops() {
    static const Ops o = {residual, sweep, restrict_sol, restrict_res, fas, defect, norm_partial};
    return &o;
  }
};

}  // namespace momg_gpu

#define MOMG_INSTANTIATE(Mv)                                                          \
  namespace momg_gpu {                                                                \
  const Ops* ops_m##Mv() { return Launch<Mv>::ops(); }                                \
  }
