// Per-cell warp routines: stencil prefetch, face fluxes, collision, the cell
// residual, the local update with grad_normalize and the dt/2 retry.  One
// full warp works on one cell; vectors live in the warp's shared-memory
// buffers (WarpBuf), descriptors in the block header (BlockHdr).
#pragma once

#include "es_bgk.cuh"
#include "momg_device.cuh"

namespace momg_gpu {

// Stencil slots: 0 self, 1 x-, 2 x+, 3 y-, 4 y+, 5 x--, 6 x++, 7 y--, 8 y++.
template <int ORDER>
struct Stencil {
  static constexpr int NCELL = ORDER == 2 ? 9 : 5;
};

template <int M, int ORDER>
struct WarpBuf {
  using C = Cfg<M>;
  static constexpr int NB = C::NB;
  double cell[Stencil<ORDER>::NCELL][NB];  // prefetched stencil (slot N = 0)
  double LA[NB], UB[NB];                   // reconstructed face states / flux scratch
  double X1[NB], X2[NB], Y1[NB], Y2[NB];   // projection ping-pong scratch
  double Kup[C::KT], Klo[C::KT];           // folded half-flux kernels
  double c[4][C::PC];                      // projection coefficients
  double cp[Stencil<ORDER>::NCELL][4];     // stencil params
  double par[8];                           // face-state params (lower, upper)
};

struct BlockHdr {
  DevCtx ctx;
  DevField f, g, h, o;
};

template <int M, int ORDER>
struct BlockSmem {
  static constexpr size_t tab_bytes = ((Cfg<M>::WORDS * 32 * 4 + 127) / 128) * 128;
  static constexpr size_t hdr_bytes = ((sizeof(BlockHdr) + 127) / 128) * 128;
  static constexpr size_t bytes(int warps) {
    return hdr_bytes + tab_bytes + sizeof(WarpBuf<M, ORDER>) * (size_t)warps;
  }
};

struct BlockView {
  BlockHdr* hdr;
  uint32_t* tab;
  unsigned char* warps;
};

template <int M, int ORDER>
__device__ __forceinline__ WarpBuf<M, ORDER>& warp_buf(const BlockView& v) {
  return reinterpret_cast<WarpBuf<M, ORDER>*>(v.warps)[threadIdx.x >> 5];
}

// Block prologue: launch descriptors to shared memory, index tables, zero
// slots of every warp buffer.
template <int M, int ORDER>
__device__ __forceinline__ BlockView block_setup(unsigned char* raw, const DevCtx* ctx,
                                                 const DevField* f, const DevField* g,
                                                 const DevField* h, const DevField* o) {
  using S = BlockSmem<M, ORDER>;
  BlockView v;
  v.hdr = reinterpret_cast<BlockHdr*>(raw);
  v.tab = reinterpret_cast<uint32_t*>(raw + S::hdr_bytes);
  v.warps = raw + S::hdr_bytes + S::tab_bytes;
  if (threadIdx.x == 0) {
    if (ctx) v.hdr->ctx = *ctx;
    if (f) v.hdr->f = *f;
    if (g) v.hdr->g = *g;
    if (h) v.hdr->h = *h;
    if (o) v.hdr->o = *o;
  }
  build_tables<M>(v.tab);
  // zero the whole warp area once: zero slots stay zero forever
  double* z = reinterpret_cast<double*>(v.warps);
  const int nz = (int)(sizeof(WarpBuf<M, ORDER>) / 8) * (blockDim.x / 32);
  for (int q = threadIdx.x; q < nz; q += blockDim.x) z[q] = 0.0;
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
    case W_NON_SPD: return E_NONSPD;
    default: return E_NONPHYSICAL;
  }
}

// L2-coherent global access (values written by other SMs during a persistent
// sweep are observed after the flag acquire).
__device__ __forceinline__ double ldg_cg(const double* p) { return __ldcg(p); }

// Issues the loads of one cell record into smem (no sync).
template <int M>
__device__ __forceinline__ void load_cell_async(const DevField* f, size_t cell, double* dst,
                                                double* prm) {
  const double* src = f->c + cell * Cfg<M>::NP;
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    const int k = lane + 32 * t;
    if (t < Cfg<M>::T - 1 || k < Cfg<M>::N) dst[k] = ldg_cg(src + k);
  }
  if (lane < 4) prm[lane] = ldg_cg(f->p + cell * 4 + lane);
}

template <int M>
__device__ __forceinline__ void load_cell(const DevField* f, size_t cell, double* dst, double* prm) {
  load_cell_async<M>(f, cell, dst, prm);
  __syncwarp();
}

// Writes registers v (+ params prm) to global memory.
template <int M>
__device__ __forceinline__ void store_cell_regs(const DevField* f, size_t cell, const double* v,
                                                const double* prm) {
  const int lane = lane_id();
  double* dst = f->c + cell * Cfg<M>::NP;
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    const int k = lane + 32 * t;
    if (t < Cfg<M>::T - 1 || k < Cfg<M>::N) __stcg(dst + k, v[t]);
  }
  if (lane < 4) __stcg(f->p + cell * 4 + lane, prm[lane]);
}

__device__ __forceinline__ P4 p4(const double* p) {
  P4 r;
  r.v[0] = p[0];
  r.v[1] = p[1];
  r.v[2] = p[2];
  r.v[3] = p[3];
  return r;
}

// Prefetches the stencil of cell (i, j) (radius 1 or 2 cross) into sb.cell
// with one batch of independent loads; synced on return.
template <int M, int ORDER>
__device__ __forceinline__ void load_stencil(const DevField* f, int i, int j,
                                             WarpBuf<M, ORDER>& sb) {
  const size_t c = (size_t)j * f->nx + i;
  load_cell_async<M>(f, c, sb.cell[0], sb.cp[0]);
  if (i > 0) load_cell_async<M>(f, c - 1, sb.cell[1], sb.cp[1]);
  if (i < f->nx - 1) load_cell_async<M>(f, c + 1, sb.cell[2], sb.cp[2]);
  if (j > 0) load_cell_async<M>(f, c - f->nx, sb.cell[3], sb.cp[3]);
  if (j < f->ny - 1) load_cell_async<M>(f, c + f->nx, sb.cell[4], sb.cp[4]);
  if (ORDER == 2) {
    if (i > 1) load_cell_async<M>(f, c - 2, sb.cell[5 % Stencil<ORDER>::NCELL], sb.cp[5 % Stencil<ORDER>::NCELL]);
    if (i < f->nx - 2) load_cell_async<M>(f, c + 2, sb.cell[6 % Stencil<ORDER>::NCELL], sb.cp[6 % Stencil<ORDER>::NCELL]);
    if (j > 1) load_cell_async<M>(f, c - 2 * (size_t)f->nx, sb.cell[7 % Stencil<ORDER>::NCELL], sb.cp[7 % Stencil<ORDER>::NCELL]);
    if (j < f->ny - 2) load_cell_async<M>(f, c + 2 * (size_t)f->nx, sb.cell[8 % Stencil<ORDER>::NCELL], sb.cp[8 % Stencil<ORDER>::NCELL]);
  }
  __syncwarp();
}

// face_state + safe_face_state (spatial.cpp:34-80) of the stencil cell in
// slot `s` on its (axis, high) face, for second order: central slope from
// slots `lo`/`hi`, zero slope at wall-adjacent cells (position m == 0 or
// last), nonpositive-temperature fallback to the cell.  Returns the buffer
// holding the state (the cell buffer itself when unchanged) and writes the
// params to prm.
template <int M, int ORDER>
__device__ __forceinline__ const double* face_state(const DevField* f, WarpBuf<M, ORDER>& sb, int s,
                                                    int lo, int hi, int m, int last, double h,
                                                    double off, double* dst, double* prm) {
  const int lane = lane_id();
  if (ORDER == 1 || m == 0 || m == last) {
    if (lane < 4) prm[lane] = sb.cp[s][lane];
    return sb.cell[s];
  }
  const double* cs = sb.cell[s];
  const double* cl = sb.cell[lo];
  const double* ch = sb.cell[hi];
  const double wsp = sb.cp[s][3] + off * ((sb.cp[hi][3] - sb.cp[lo][3]) / h);
  if (!(wsp > 0.0)) {  // NonphysicalReconstruction -> first-order value
    if (lane < 4) prm[lane] = sb.cp[s][lane];
    return sb.cell[s];
  }
  const double rh = 1.0 / h;
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    const int k = lane + 32 * t;
    if (t < Cfg<M>::T - 1 || k < Cfg<M>::N) dst[k] = fma(off, (ch[k] - cl[k]) * rh, cs[k]);
  }
  if (lane < 3) prm[lane] = sb.cp[s][lane] + off * ((sb.cp[hi][lane] - sb.cp[lo][lane]) / h);
  if (lane == 3) prm[3] = wsp;
  return dst;
}

// ------------------------------------------------------------ grad_normalize
// projection.hpp:96-121 on the vector held in smem `X` and registers v with
// basis prm (smem, updated); Y, Z scratch.  Returns W_NONE or the failure
// kind; on success *out points at the buffer holding the result (== v).
template <int M, int ORDER>
__device__ __forceinline__ int grad_normalize(const uint32_t* tab, WarpBuf<M, ORDER>& sb, double* X,
                                              double* Y, double* Z, double* prm, double* v,
                                              double* bad, const double** out) {
  const double rel_tol = 1e-12;
  const double* cur = X;
  for (int iter = 0; iter < 30; ++iter) {
    const double rho = cur[0];
    if (!isfinite(rho) || !(rho > 0.0)) {
      *bad = rho;
      return W_GRAD_RHO;
    }
    if (grad_defect(cur) <= rel_tol) {
      *out = cur;
      return W_NONE;
    }
    P4 to;
    const P4 from = p4(prm);
    to.v[0] = rep_u(cur, prm, 0);
    to.v[1] = rep_u(cur, prm, 1);
    to.v[2] = rep_u(cur, prm, 2);
    to.v[3] = rep_theta(cur, prm);
    if (!isfinite(to.v[3]) || !(to.v[3] > 0.0)) {
      *bad = to.v[3];
      return W_GRAD_THETA;
    }
    if (!isfinite(to.v[0]) || !isfinite(to.v[1]) || !isfinite(to.v[2])) return W_GRAD_U;
    proj_coeffs<M>(from, to, sb.c[3]);
    __syncwarp();
    if (lane_id() < 4) prm[lane_id()] = to.v[lane_id()];
    double* s1 = cur == X ? Y : (cur == Y ? Z : X);
    double* s2 = cur == X ? Z : (cur == Y ? X : Y);
    cur = project_apply<M>(tab, cur, s1, s2, sb.c[3], pass_mask(from, to), v);
  }
  if (grad_defect(cur) > rel_tol) return W_GRAD_CAP;
  *out = cur;
  return W_NONE;
}

// ----------------------------------------------------------------- collision
// collision_coeffs (collision.hpp:120-127): Q = nu (f_eq - f) in the cell's
// own basis, BGK or Shakhov (extract_macro moment_rep.hpp:116-146), into
// registers.
template <int M>
__device__ __forceinline__ int collision(const uint32_t* tab, const double* S, const double* cp,
                                         const DevCtx* ctx, double* Q, double* scratch) {
  const double rho = S[0];
  if (!(rho > 0.0)) return W_MACRO_RHO;
  const double theta = cp[3];
  if (!(theta > 0.0)) return W_MACRO_RHO;  // maxwellian_rep precondition
  const bool es_bgk = ctx->collision == 1;
  if (es_bgk) {
    // ES-BGK: the Gaussian equilibrium (es_bgk.cuh) built once by lane 0 in
    // the warp's scratch vector, flat coefficient order
    double bad = 0.0;
    if (es::check<1>(S, theta, ctx->prandtl, &bad)) return W_NON_SPD;
    if (lane_id() == 0) es::fill<M, 1>(S, theta, ctx->prandtl, scratch);
    __syncwarp();
  }
  const double nu = ctx->nu_coef * rho * pow(theta, ctx->nu_exp);
  double q[3] = {0.0, 0.0, 0.0};
  const bool shakhov = ctx->collision == 2;
  if (shakhov) {
    // q_i = 2 f_{3e_i} + sum_d f_{2e_d + e_i}
    q[0] = 2.0 * S[flat3(3, 0, 0)] + S[flat3(3, 0, 0)] + S[flat3(1, 2, 0)] + S[flat3(1, 0, 2)];
    q[1] = 2.0 * S[flat3(0, 3, 0)] + S[flat3(2, 1, 0)] + S[flat3(0, 3, 0)] + S[flat3(0, 1, 2)];
    q[2] = 2.0 * S[flat3(0, 0, 3)] + S[flat3(2, 0, 1)] + S[flat3(0, 2, 1)] + S[flat3(0, 0, 3)];
  }
  const int lane = lane_id();
#pragma unroll
  for (int t = 0; t < Cfg<M>::T; ++t) {
    const int k = lane + 32 * t;
    double eq = k == 0 ? rho : 0.0;
    if (es_bgk && k < Cfg<M>::N) eq = scratch[item_pos<M>(t)];
    if (shakhov) {
      const uint32_t ms = misc<M>(tab, t);
      const int a1 = byte_of(ms, 0), a2 = byte_of(ms, 1), a3 = byte_of(ms, 2);
      if (a1 + a2 + a3 == 3 && !(a1 == 1 && a2 == 1 && a3 == 1) && k < Cfg<M>::N) {
        const int d = (a1 & 1) ? 0 : ((a2 & 1) ? 1 : 2);
        eq = ctx->shakhov_w * q[d];
      }
    }
    Q[t] = nu * (eq - S[item_pos<M>(t)]);
  }
  return W_NONE;
}

// ----------------------------------------------------------------- face flux
// Flux through face (axis, high) of cell (i, j), projected into the cell
// basis (the `face` lambda of cell_residual, spatial.cpp:106-124), into
// registers F.  Stencil in sb.cell / sb.cp.  Returns W_NONE or a failure.
template <int M, int ORDER>
__device__ __forceinline__ int cell_face(const DevField* f, const DevCtx* ctx, const uint32_t* tab,
                                         int i, int j, int axis, bool high, WarpBuf<M, ORDER>& sb,
                                         double* F) {
  constexpr int T = Cfg<M>::T;
  const int lane = lane_id();
  const bool at_wall = axis == 0 ? (high ? i == f->nx - 1 : i == 0)
                                 : (high ? j == f->ny - 1 : j == 0);
  const P4 cp = p4(sb.cp[0]);
  double out[T];
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
    proj_coeffs<M>(cp, fp, sb.c[0]);
    proj_coeffs<M>(fp, cp, sb.c[2]);
    __syncwarp();
    double v[T];
    const double* in_w = project_apply<M>(tab, sb.cell[0], sb.X1, sb.X2, sb.c[0], pass_mask(cp, fp), v);
    const double* Kout = high ? sb.Kup : sb.Klo;
    const double* Kin = high ? sb.Klo : sb.Kup;
    half_sum<M>(tab, in_w, Kout, nullptr, nullptr, axis, out);
    const double o0 = __shfl_sync(FULL, out[0], 0);
    const double in0 = Kin[0];
    if (in0 == 0.0) return W_WALL_DEGEN;
    const double wall_rho = -o0 / in0;
    if (!(wall_rho > 0.0)) return W_WALL_RHO;
    // incoming unit-wall half flux: rs^p/p! K(0,p) at beta = p e_axis
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const uint32_t ms = misc<M>(tab, t);
      const int p = byte_of(ms, axis);
      const int tan = byte_of(ms, 0) + byte_of(ms, 1) + byte_of(ms, 2) - p;
      if (tan == 0 && (t < T - 1 || lane + 32 * t < Cfg<M>::N)) out[t] = fma(wall_rho, Kin[p], out[t]);
    }
    if (lane == 0) out[0] = 0.0;
    store_items<M>(sb.LA, out);
    __syncwarp();
    project_apply<M>(tab, sb.LA, sb.X1, sb.X2, sb.c[2], pass_mask(fp, cp), F);
    return W_NONE;
  }
  // interior face, flux.cpp:77-97, lo/hi roles of spatial.cpp:114-121
  const int s_nb = axis == 0 ? (high ? 2 : 1) : (high ? 4 : 3);     // neighbour slot
  const int s_nb2 = axis == 0 ? (high ? 6 : 5) : (high ? 8 : 7);    // neighbour's far slot
  const int s_opp = axis == 0 ? (high ? 1 : 2) : (high ? 3 : 4);    // own opposite slot
  const int pos = axis == 0 ? i : j;
  const int last = (axis == 0 ? f->nx : f->ny) - 1;
  const double* xc = axis == 0 ? f->xc : f->yc;
  const double* dd = axis == 0 ? f->dx : f->dy;
  double* lp = sb.par;
  double* rp = sb.par + 4;
  const double* L;
  const double* U;
  if (high) {
    // lower = self (slope from opp -> nb), upper = nb (slope from self -> nb2)
    L = face_state<M, ORDER>(f, sb, 0, s_opp, s_nb, pos, last,
                             ORDER == 2 && pos > 0 && pos < last ? xc[pos + 1] - xc[pos - 1] : 1.0,
                             0.5 * dd[pos], sb.LA, lp);
    U = face_state<M, ORDER>(f, sb, s_nb, 0, s_nb2 % Stencil<ORDER>::NCELL, pos + 1, last,
                             ORDER == 2 && pos + 1 < last ? xc[pos + 2] - xc[pos] : 1.0,
                             -0.5 * dd[pos + 1], sb.UB, rp);
  } else {
    L = face_state<M, ORDER>(f, sb, s_nb, s_nb2 % Stencil<ORDER>::NCELL, 0, pos - 1, last,
                             ORDER == 2 && pos - 1 > 0 ? xc[pos] - xc[pos - 2] : 1.0,
                             0.5 * dd[pos - 1], sb.LA, lp);
    U = face_state<M, ORDER>(f, sb, 0, s_nb, s_opp, pos, last,
                             ORDER == 2 && pos > 0 && pos < last ? xc[pos + 1] - xc[pos - 1] : 1.0,
                             -0.5 * dd[pos], sb.UB, rp);
  }
  __syncwarp();
  const double ul = rep_u(L, lp, axis), ur = rep_u(U, rp, axis);
  const double cl = ctx->c_bound * sqrt(rep_theta(L, lp));
  const double cr = ctx->c_bound * sqrt(rep_theta(U, rp));
  const double lminus = smin(ul - cl, ur - cr);
  const double lplus = smax(ul + cl, ur + cr);
  const P4 lpv = p4(lp), rpv = p4(rp);
#pragma unroll
  for (int q = 0; q < 4; ++q) fp.v[q] = 0.5 * (lpv.v[q] + rpv.v[q]);
  if (!(fp.v[3] > 0.0)) return W_PROJ_SPREAD;
  if (lminus >= 0.0 || lplus <= 0.0) {
    const bool left = lminus >= 0.0;
    proj_coeffs<M>(left ? lpv : rpv, fp, sb.c[0]);
    proj_coeffs<M>(fp, cp, sb.c[2]);
    __syncwarp();
    double v[T];
    const double* st = project_apply<M>(tab, left ? L : U, sb.X1, sb.X2, sb.c[0],
                                        pass_mask(left ? lpv : rpv, fp), v);
    full_flux<M>(tab, st, fp.v[axis], fp.v[3], axis, out);
  } else {
    const double rs = sqrt(fp.v[3]);
    half_kernels<M>(fp.v[axis], rs, sb.Kup, sb.Klo);
    proj_coeffs<M>(lpv, fp, sb.c[0]);
    proj_coeffs<M>(rpv, fp, sb.c[1]);
    proj_coeffs<M>(fp, cp, sb.c[2]);
    __syncwarp();
    double va[T], vb[T];
    const double *pa, *pb;
    project_apply2<M>(tab, L, sb.X1, sb.X2, sb.c[0], pass_mask(lpv, fp), va, U, sb.Y1, sb.Y2,
                      sb.c[1], pass_mask(rpv, fp), vb, &pa, &pb);
    half_sum<M>(tab, pa, sb.Kup, pb, sb.Klo, axis, out);
  }
  __syncwarp();
  store_items<M>(sb.LA, out);
  __syncwarp();
  project_apply<M>(tab, sb.LA, sb.X1, sb.X2, sb.c[2], pass_mask(fp, cp), F);
  return W_NONE;
}

// cell_residual (spatial.cpp:98-133) into registers R, stencil prefetched.
template <int M, int ORDER>
__device__ __forceinline__ int cell_residual(const DevField* f, const DevCtx* ctx, const uint32_t* tab,
                                             int i, int j, WarpBuf<M, ORDER>& sb, double* R) {
  constexpr int T = Cfg<M>::T;
  int w = collision<M>(tab, sb.cell[0], sb.cp[0], ctx, R, sb.X1);
  if (w) return w;
  double Fp[T], Fm[T];
  if ((w = cell_face<M, ORDER>(f, ctx, tab, i, j, 0, true, sb, Fp))) return w;
  if ((w = cell_face<M, ORDER>(f, ctx, tab, i, j, 0, false, sb, Fm))) return w;
  const double dx = f->dx[i], dy = f->dy[j];
#pragma unroll
  for (int t = 0; t < T; ++t) R[t] -= (Fp[t] - Fm[t]) / dx;
  if ((w = cell_face<M, ORDER>(f, ctx, tab, i, j, 1, true, sb, Fp))) return w;
  if ((w = cell_face<M, ORDER>(f, ctx, tab, i, j, 1, false, sb, Fm))) return w;
#pragma unroll
  for (int t = 0; t < T; ++t) R[t] -= (Fp[t] - Fm[t]) / dy;
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
// (:44-70) for cell (i, j) whose stencil is prefetched.  rhs may be null.
// Writes the updated cell, or leaves it and returns the failure kind.
template <int M, int ORDER>
__device__ __forceinline__ int sweep_cell(const DevField* f, const DevField* rhs, const DevCtx* ctx,
                                          const uint32_t* tab, int i, int j, WarpBuf<M, ORDER>& sb,
                                          double* bad) {
  constexpr int T = Cfg<M>::T;
  const size_t cell = (size_t)j * f->nx + i;
  double dt;
  int w = local_dt(ctx, sb.cp[0], f->dx[i], f->dy[j], &dt);
  if (w) return w;
  double R[T];
  w = cell_residual<M, ORDER>(f, ctx, tab, i, j, sb, R);
  if (w) return w;
  const int lane = lane_id();
  if (rhs) {
    load_cell<M>(rhs, cell, sb.UB, sb.par);
    const P4 rp = p4(sb.par), cp = p4(sb.cp[0]);
    proj_coeffs<M>(rp, cp, sb.c[1]);
    __syncwarp();
    double pr[T];
    project_apply<M>(tab, sb.UB, sb.Y1, sb.Y2, sb.c[1], pass_mask(rp, cp), pr);
#pragma unroll
    for (int t = 0; t < T; ++t) R[t] -= pr[t];
  }
  // apply_update: f += dt*delta; grad_normalize; retry at dt/2 on NonphysicalState
  for (int attempt = 0; attempt < 2; ++attempt) {
    const double step = attempt == 0 ? dt : 0.5 * dt;
    double v[T];
#pragma unroll
    for (int t = 0; t < T; ++t) v[t] = fma(step, R[t], sb.cell[0][item_pos<M>(t)]);
    __syncwarp();
    store_items<M>(sb.X1, v);
    if (lane < 4) sb.par[lane] = sb.cp[0][lane];
    __syncwarp();
    const double* res;
    w = grad_normalize<M, ORDER>(tab, sb, sb.X1, sb.X2, sb.Y1, sb.par, v, bad, &res);
    if (w == W_NONE) {
      store_cell_regs<M>(f, cell, v, sb.par);
      __syncwarp();
      return W_NONE;
    }
    if (code_of(w) != E_NONPHYSICAL) return w;  // plain Error propagates
  }
  return W_DT_HALVING;
}

}  // namespace momg_gpu
