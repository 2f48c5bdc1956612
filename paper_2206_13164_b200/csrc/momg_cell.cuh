// Per-cell warp routines: face fluxes, collision, cell residual, the local
// update with grad_normalize and the dt/2 retry, and the transfer-operator
// bodies.  Each routine is executed by one full warp on one cell; vectors
// live in the warp's shared-memory buffers (WarpBuf), problem constants and
// field descriptors in the block header (BlockHdr), both in shared memory.
#pragma once

#include "momg_device.cuh"

namespace momg_gpu {

template <int M>
struct WarpBuf {
  static constexpr int NP = Cfg<M>::NP, KT = Cfg<M>::KT;
  double S[NP];   // the cell's own state
  double A[NP];   // face state / projection scratch
  double A2[NP];
  double B[NP];
  double B2[NP];
  double F1[NP];  // face fluxes in the cell basis
  double F2[NP];
  double R[NP];   // residual accumulator
  double Kup[KT];
  double Klo[KT];
  double cp[4];   // the cell's basis params
  double par[8];  // face-state / scratch params shared by the lanes
};

struct BlockHdr {
  DevCtx ctx;
  DevField f, g, h, o;
};

template <int M>
struct BlockSmem {
  static constexpr size_t alpha_bytes = ((Cfg<M>::N * 4 + 31) / 32) * 32;
  static constexpr size_t hdr_bytes = ((sizeof(BlockHdr) + 31) / 32) * 32;
  static constexpr size_t bytes(int warps) {
    return hdr_bytes + alpha_bytes + sizeof(WarpBuf<M>) * (size_t)warps;
  }
};

struct BlockView {
  BlockHdr* hdr;
  uint32_t* alpha;
  unsigned char* warps;
};

template <int M>
__device__ __forceinline__ BlockView block_view(unsigned char* raw) {
  BlockView v;
  v.hdr = reinterpret_cast<BlockHdr*>(raw);
  v.alpha = reinterpret_cast<uint32_t*>(raw + BlockSmem<M>::hdr_bytes);
  v.warps = raw + BlockSmem<M>::hdr_bytes + BlockSmem<M>::alpha_bytes;
  return v;
}
template <int M>
__device__ __forceinline__ WarpBuf<M>& warp_buf(const BlockView& v) {
  return reinterpret_cast<WarpBuf<M>*>(v.warps)[threadIdx.x >> 5];
}

// Block prologue: copy the launch descriptors to shared memory and build the
// multi-index table.
template <int M>
__device__ __forceinline__ BlockView block_setup(unsigned char* raw, const DevCtx* ctx,
                                                 const DevField* f, const DevField* g,
                                                 const DevField* h, const DevField* o) {
  BlockView v = block_view<M>(raw);
  if (threadIdx.x == 0) {
    if (ctx) v.hdr->ctx = *ctx;
    if (f) v.hdr->f = *f;
    if (g) v.hdr->g = *g;
    if (h) v.hdr->h = *h;
    if (o) v.hdr->o = *o;
  }
  build_alpha<M>(v.alpha);
  __syncthreads();
  return v;
}

__device__ __forceinline__ void raise_err(DevErr* e, int code, int what, int i, int j,
                                          double value) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->what = what;
    e->i = i;
    e->j = j;
    e->value = value;
    __threadfence();
  }
}

__device__ __forceinline__ bool err_set(const DevErr* e) {
  return *((volatile const int*)&e->code) != 0;
}

__device__ __forceinline__ int code_of(int what) {
  switch (what) {
    case W_NONE: return E_OK;
    case W_GRAD_CAP: return E_ERROR;
    case W_DT_HALVING:
    case W_FAS: return E_SOLVER;
    case W_ES_UNSUPPORTED: return E_CONFIG;
    default: return E_NONPHYSICAL;
  }
}

// L2-coherent global loads/stores: values written by other SMs during a
// persistent sweep are observed after the flag acquire.
__device__ __forceinline__ double ldg_cg(const double* p) { return __ldcg(p); }

// Loads a cell's coefficients into smem `dst` and its params into `prm`
// (smem, 4 doubles); synced on return.
template <int M>
__device__ __forceinline__ void load_cell(const DevField* f, size_t cell, double* dst, double* prm) {
  constexpr int NP = Cfg<M>::NP;
  const double* src = f->c + cell * NP;
  const int lane = lane_id();
  for (int k = lane; k < Cfg<M>::N; k += 32) dst[k] = ldg_cg(src + k);
  if (lane < 4) prm[lane] = ldg_cg(f->p + cell * 4 + lane);
  __syncwarp();
}

template <int M>
__device__ __forceinline__ void store_cell(const DevField* f, size_t cell, const double* src,
                                           const double* prm) {
  constexpr int NP = Cfg<M>::NP;
  const int lane = lane_id();
  double* dst = f->c + cell * NP;
  for (int k = lane; k < Cfg<M>::N; k += 32) __stcg(dst + k, src[k]);
  if (lane < 4) __stcg(f->p + cell * 4 + lane, prm[lane]);
  __syncwarp();
}

__device__ __forceinline__ P4 p4(const double* p) {
  P4 r;
  r.v[0] = p[0];
  r.v[1] = p[1];
  r.v[2] = p[2];
  r.v[3] = p[3];
  return r;
}

// Face state of cell (i, j) on its (axis, high) face (spatial.cpp:34-80) into
// dst / prm: order 1 -> the cell; order 2 -> central slope from the
// neighbours along the axis (zero at wall-adjacent cells), with the
// nonpositive-temperature fallback to the cell value (safe_face_state,
// spatial.cpp:53-60).
template <int M>
__device__ __noinline__ void face_state(const DevField* f, int order, int i, int j, int axis,
                                        bool high, double* dst, double* prm) {
  constexpr int NP = Cfg<M>::NP;
  const size_t cell = (size_t)j * f->nx + i;
  load_cell<M>(f, cell, dst, prm);
  if (order == 1) return;
  const int m = axis == 0 ? i : j;
  const int last = (axis == 0 ? f->nx : f->ny) - 1;
  if (m == 0 || m == last) return;  // zero slope: w = cell (+ off * 0)
  const size_t lo = axis == 0 ? cell - 1 : cell - f->nx;
  const size_t hi = axis == 0 ? cell + 1 : cell + f->nx;
  const double h = axis == 0 ? f->xc[i + 1] - f->xc[i - 1] : f->yc[j + 1] - f->yc[j - 1];
  const double off = (high ? 0.5 : -0.5) * (axis == 0 ? f->dx[i] : f->dy[j]);
  const double wsp = prm[3] + off * ((ldg_cg(f->p + hi * 4 + 3) - ldg_cg(f->p + lo * 4 + 3)) / h);
  if (!(wsp > 0.0)) return;  // NonphysicalReconstruction -> first order
  const int lane = lane_id();
  const double rh = 1.0 / h;
  for (int k = lane; k < Cfg<M>::N; k += 32) {
    const double s = (ldg_cg(f->c + hi * NP + k) - ldg_cg(f->c + lo * NP + k)) * rh;
    dst[k] = fma(off, s, dst[k]);
  }
  __syncwarp();
  if (lane < 3) prm[lane] = prm[lane] + off * ((ldg_cg(f->p + hi * 4 + lane) - ldg_cg(f->p + lo * 4 + lane)) / h);
  if (lane == 3) prm[3] = wsp;
  __syncwarp();
}

// ------------------------------------------------------------ grad_normalize
// projection.hpp:96-121 on the vector in smem X with basis prm (smem, updated
// in place); Y is scratch.  Returns W_NONE or the failure kind.
template <int M>
__device__ __noinline__ int grad_normalize_smem(const uint32_t* alpha, double* X, double* Y,
                                                double* prm, double* bad) {
  const double rel_tol = 1e-12;
  for (int iter = 0; iter < 30; ++iter) {
    const double rho = X[0];
    if (!isfinite(rho) || !(rho > 0.0)) {
      *bad = rho;
      return W_GRAD_RHO;
    }
    if (grad_defect(X) <= rel_tol) return W_NONE;
    P4 to;
    to.v[0] = rep_u(X, prm, 0);
    to.v[1] = rep_u(X, prm, 1);
    to.v[2] = rep_u(X, prm, 2);
    to.v[3] = rep_theta(X, prm);
    if (!isfinite(to.v[3]) || !(to.v[3] > 0.0)) {
      *bad = to.v[3];
      return W_GRAD_THETA;
    }
    if (!isfinite(to.v[0]) || !isfinite(to.v[1]) || !isfinite(to.v[2])) return W_GRAD_U;
    project_smem<M>(alpha, X, Y, p4(prm), to, X);
    if (lane_id() < 4) prm[lane_id()] = to.v[lane_id()];
    __syncwarp();
  }
  if (grad_defect(X) > rel_tol) return W_GRAD_CAP;
  return W_NONE;
}

// ----------------------------------------------------------------- collision
// collision_coeffs (collision.hpp:120-127): dst = nu (f_eq - f) in the cell's
// own basis, BGK or Shakhov (extract_macro moment_rep.hpp:116-146).
template <int M>
__device__ __noinline__ int collision_smem(const uint32_t* alpha, const double* S,
                                           const double* cp, const DevCtx* ctx, double* dst) {
  const double rho = S[0];
  if (!(rho > 0.0)) return W_MACRO_RHO;
  const double theta = cp[3];
  if (!(theta > 0.0)) return W_MACRO_RHO;  // maxwellian_rep precondition
  if (ctx->collision == 1) return W_ES_UNSUPPORTED;
  const double nu = ctx->nu_coef * rho * pow(theta, ctx->nu_exp);
  double q[3] = {0.0, 0.0, 0.0};
  const bool shakhov = ctx->collision == 2;
  if (shakhov) {
    // q_i = 2 f_{3e_i} + sum_d f_{2e_d + e_i}
    q[0] = 2.0 * S[flat3(3, 0, 0)] + S[flat3(3, 0, 0)] + S[flat3(1, 2, 0)] + S[flat3(1, 0, 2)];
    q[1] = 2.0 * S[flat3(0, 3, 0)] + S[flat3(2, 1, 0)] + S[flat3(0, 3, 0)] + S[flat3(0, 1, 2)];
    q[2] = 2.0 * S[flat3(0, 0, 3)] + S[flat3(2, 0, 1)] + S[flat3(0, 2, 1)] + S[flat3(0, 0, 3)];
  }
  const Items<M> it(alpha);
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    if (!it.v(t)) continue;
    const int k = lane + 32 * t;
    double eq = k == 0 ? rho : 0.0;
    const int a1 = it.a1(t), a2 = it.a2(t), a3 = it.a3(t);
    if (shakhov && a1 + a2 + a3 == 3 && !(a1 == 1 && a2 == 1 && a3 == 1)) {
      const int d = (a1 & 1) ? 0 : ((a2 & 1) ? 1 : 2);
      eq = ctx->shakhov_w * q[d];
    }
    dst[k] = nu * (eq - S[k]);
  }
  __syncwarp();
  return W_NONE;
}

// ----------------------------------------------------------------- face flux
// Flux through face (axis, high) of cell (i, j), projected into the cell
// basis cp (the `face` lambda of cell_residual, spatial.cpp:106-124), into
// dst.  The cell's own state is in sb.S.  Returns W_NONE or a failure kind.
template <int M>
__device__ __noinline__ int cell_face(const DevField* f, const DevCtx* ctx, const uint32_t* alpha,
                                      int i, int j, int axis, bool high, const double* cp,
                                      WarpBuf<M>& sb, double* dst) {
  const int lane = lane_id();
  const bool at_wall = axis == 0 ? (high ? i == f->nx - 1 : i == 0)
                                 : (high ? j == f->ny - 1 : j == 0);
  P4 fp;
  if (at_wall) {
    // wall_flux, flux.cpp:105-130
    const int w = axis == 0 ? (high ? 1 : 0) : (high ? 3 : 2);
    fp.v[0] = fp.v[1] = fp.v[2] = 0.0;
    fp.v[axis == 0 ? 1 : 0] = ctx->wall_speed[w];
    fp.v[3] = ctx->wall_theta[w];
    if (!(fp.v[3] > 0.0)) return W_PROJ_SPREAD;
    const double rs = sqrt(fp.v[3]);
    half_kernels<M>(0.0, rs, sb.Kup, sb.Klo);
    vcopy<M>(sb.A, sb.S);
    project_smem<M>(alpha, sb.A, sb.A2, p4(cp), fp, sb.A);
    const double* Kout = high ? sb.Kup : sb.Klo;
    const double* Kin = high ? sb.Klo : sb.Kup;
    half_sum<M>(alpha, sb.A, Kout, nullptr, nullptr, axis, rs, sb.B);
    const double o0 = sb.B[0];
    const double in0 = Kin[0];
    if (in0 == 0.0) return W_WALL_DEGEN;
    const double wall_rho = -o0 / in0;
    if (!(wall_rho > 0.0)) return W_WALL_RHO;
    // incoming unit-wall half flux: nonzero only at beta = p e_n
    if (lane <= M) {
      const int p = lane;
      double v = Kin[p];
      for (int e = 1; e <= p; ++e) v = v * rs * rcp_int(e);
      const int k = flat3(axis == 0 ? p : 0, axis == 1 ? p : 0, axis == 2 ? p : 0);
      sb.B[k] = fma(wall_rho, v, sb.B[k]);
    }
    __syncwarp();
    if (lane == 0) sb.B[0] = 0.0;
    __syncwarp();
    if (!project_smem<M>(alpha, sb.B, sb.B2, fp, p4(cp), dst)) return W_PROJ_SPREAD;
    return W_NONE;
  }
  // interior face, flux.cpp:77-97 with the geometric lo/hi roles of
  // spatial.cpp:114-121
  const int ni = axis == 0 ? (high ? i + 1 : i - 1) : i;
  const int nj = axis == 1 ? (high ? j + 1 : j - 1) : j;
  double* lp = sb.par;
  double* rp = sb.par + 4;
  face_state<M>(f, ctx->order, high ? i : ni, high ? j : nj, axis, true, sb.A, lp);
  face_state<M>(f, ctx->order, high ? ni : i, high ? nj : j, axis, false, sb.B, rp);
  const double ul = rep_u(sb.A, lp, axis), ur = rep_u(sb.B, rp, axis);
  const double cl = ctx->c_bound * sqrt(rep_theta(sb.A, lp));
  const double cr = ctx->c_bound * sqrt(rep_theta(sb.B, rp));
  const double lminus = smin(ul - cl, ur - cr);
  const double lplus = smax(ul + cl, ur + cr);
#pragma unroll
  for (int q = 0; q < 4; ++q) fp.v[q] = 0.5 * (lp[q] + rp[q]);
  const P4 lpv = p4(lp), rpv = p4(rp);
  if (lminus >= 0.0 || lplus <= 0.0) {
    double* X = lminus >= 0.0 ? sb.A : sb.B;
    double* Y = lminus >= 0.0 ? sb.A2 : sb.B2;
    if (!project_smem<M>(alpha, X, Y, lminus >= 0.0 ? lpv : rpv, fp, X)) return W_PROJ_SPREAD;
    full_flux<M>(alpha, X, fp.v[axis], fp.v[3], axis, Y);
    return project_smem<M>(alpha, Y, X, fp, p4(cp), dst) ? W_NONE : W_PROJ_SPREAD;
  }
  if (!(fp.v[3] > 0.0)) return W_HALF_SPREAD;
  const double rs = sqrt(fp.v[3]);
  half_kernels<M>(fp.v[axis], rs, sb.Kup, sb.Klo);
  if (!project_smem<M>(alpha, sb.A, sb.A2, lpv, fp, sb.A)) return W_PROJ_SPREAD;
  project_smem<M>(alpha, sb.B, sb.B2, rpv, fp, sb.B);
  half_sum<M>(alpha, sb.A, sb.Kup, sb.B, sb.Klo, axis, rs, sb.A2);
  if (!project_smem<M>(alpha, sb.A2, sb.B2, fp, p4(cp), dst)) return W_PROJ_SPREAD;
  return W_NONE;
}

// cell_residual (spatial.cpp:98-133): R = Q - (F_x+ - F_x-)/dx - (F_y+ - F_y-)/dy
// in the cell basis, into sb.R.  The cell state must be in sb.S with params cp.
template <int M>
__device__ __noinline__ int cell_residual_smem(const DevField* f, const DevCtx* ctx,
                                               const uint32_t* alpha, int i, int j,
                                               const double* cp, WarpBuf<M>& sb) {
  int w = collision_smem<M>(alpha, sb.S, cp, ctx, sb.R);
  if (w) return w;
  if ((w = cell_face<M>(f, ctx, alpha, i, j, 0, true, cp, sb, sb.F1))) return w;
  if ((w = cell_face<M>(f, ctx, alpha, i, j, 0, false, cp, sb, sb.F2))) return w;
  const int lane = lane_id();
  const double dx = f->dx[i], dy = f->dy[j];
  for (int k = lane; k < Cfg<M>::N; k += 32) sb.R[k] -= (sb.F1[k] - sb.F2[k]) / dx;
  __syncwarp();
  if ((w = cell_face<M>(f, ctx, alpha, i, j, 1, true, cp, sb, sb.F1))) return w;
  if ((w = cell_face<M>(f, ctx, alpha, i, j, 1, false, cp, sb, sb.F2))) return w;
  for (int k = lane; k < Cfg<M>::N; k += 32) sb.R[k] -= (sb.F1[k] - sb.F2[k]) / dy;
  __syncwarp();
  return W_NONE;
}

// local_dt (single_level.cpp:18-24)
__device__ __forceinline__ int local_dt(const DevCtx* ctx, const double* cp, double dx, double dy,
                                        double* dt) {
  const double theta = cp[3];
  if (!(theta > 0.0)) return W_DT_THETA;
  const double c = ctx->cfl_c_bound * sqrt(theta);
  *dt = ctx->cfl / ((fabs(cp[0]) + c) / dx + (fabs(cp[1]) + c) / dy);
  return W_NONE;
}

// sweep_cell (single_level.cpp:103-111) + update_delta / apply_update
// (:44-70).  rhs may be null (empty RhsField).  Writes the updated cell, or
// leaves it unchanged and returns the failure kind.
template <int M>
__device__ __noinline__ int sweep_cell_smem(const DevField* f, const DevField* rhs,
                                            const DevCtx* ctx, const uint32_t* alpha, int i, int j,
                                            WarpBuf<M>& sb, double* bad) {
  const size_t cell = (size_t)j * f->nx + i;
  load_cell<M>(f, cell, sb.S, sb.cp);
  double dt;
  int w = local_dt(ctx, sb.cp, f->dx[i], f->dy[j], &dt);
  if (w) return w;
  w = cell_residual_smem<M>(f, ctx, alpha, i, j, sb.cp, sb);
  if (w) return w;
  const int lane = lane_id();
  if (rhs) {
    load_cell<M>(rhs, cell, sb.A, sb.par);
    if (!project_smem<M>(alpha, sb.A, sb.A2, p4(sb.par), p4(sb.cp), sb.F1)) return W_PROJ_SPREAD;
    for (int k = lane; k < Cfg<M>::N; k += 32) sb.R[k] -= sb.F1[k];
    __syncwarp();
  }
  // apply_update: f += dt*delta; grad_normalize; retry at dt/2 on NonphysicalState
  for (int attempt = 0; attempt < 2; ++attempt) {
    const double step = attempt == 0 ? dt : 0.5 * dt;
    for (int k = lane; k < Cfg<M>::N; k += 32) sb.A[k] = fma(step, sb.R[k], sb.S[k]);
    if (lane < 4) sb.par[lane] = sb.cp[lane];
    __syncwarp();
    w = grad_normalize_smem<M>(alpha, sb.A, sb.A2, sb.par, bad);
    if (w == W_NONE) {
      store_cell<M>(f, cell, sb.A, sb.par);
      return W_NONE;
    }
    if (code_of(w) != E_NONPHYSICAL) return w;  // plain Error propagates
  }
  return W_DT_HALVING;
}

}  // namespace momg_gpu
