// Thread-granular kernels (moment orders 3..6): residual, the persistent
// exact-order sweep, and the transfer operators.  See thread_cell.cuh.
#pragma once

#include "runtime.h"
#include "sweep_persistent.cuh"
#include "thread_cell.cuh"

namespace momg_gpu {
namespace tc {

template <int M>
struct TSmem {
  static constexpr size_t vec = (size_t)Gen<M>::N * VS * sizeof(double);  // one vector per thread
  static constexpr size_t bytes = 2 * vec;                                  // L and U
};

__device__ __forceinline__ void raise(DevErr* e, int code, int what, int i, int j, double value) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->what = what;
    e->i = i;
    e->j = j;
    e->value = value;
    __threadfence();
  }
}
__device__ __forceinline__ bool err_on(const DevErr* e) { return *((volatile const int*)&e->code) != 0; }
__device__ __forceinline__ int code_for(int what) {
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

// face phase for thread tid of a 16-cell segment: cell (i, j) valid?
template <int M, int ORDER, bool CG>
__device__ __forceinline__ int face_phase(const DevField& f, const DevCtx& ctx, int i, int j,
                                          double* L, double* U) {
  const int tid = threadIdx.x;
  const bool high = (tid >> 4) & 1;
  if (tid < 32) return face<M, ORDER, 0, CG>(f, ctx, i, j, high, L, U);
  return face<M, ORDER, 1, CG>(f, ctx, i, j, high, L, U);
}

// --------------------------------------------------------------- residual
template <int M, int ORDER>
__global__ void __launch_bounds__(VS) k3_residual(DevField f, DevField out, DevCtx ctx, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x;
  double* L = base + tid;
  double* U = base + (size_t)Gen<M>::N * VS + tid;
  const int cells = f.nx * f.ny;
  const int tiles = (cells + SEG - 1) / SEG;
  constexpr int NP = (Gen<M>::N + 3) & ~3;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    if (err_on(err)) return;
    const int cell = tile * SEG + (tid & 15);
    const bool valid = cell < cells;
    const int i = valid ? cell % f.nx : 0, j = valid ? cell / f.nx : 0;
    if (valid) {
      const int w = face_phase<M, ORDER, false>(f, ctx, i, j, L, U);
      if (w) raise(err, code_for(w), w, i, j, 0.0);
    }
    __syncthreads();
    if (tid < SEG && valid && !err_on(err)) {
      double* S = U;                         // own U (x-low thread)
      double* D = base + (size_t)Gen<M>::N * VS + 16 + tid;  // U of the x-high thread
      load_vec<M, false>(f.c + (size_t)cell * NP, S);
      const P4 cp = ldp<false>(f.p + (size_t)cell * 4);
      double nu, q[3];
      const int w = collision_scalars<M>(S, cp, ctx, &nu, q);
      if (w) {
        raise(err, code_for(w), w, i, j, w == W_NON_SPD ? q[0] : 0.0);
      } else {
        assemble<M>(S, nu, q, ctx.collision == 2, ctx.shakhov_w, base + tid, base + 16 + tid,
                    base + 32 + tid, base + 48 + tid, f.dx[i], f.dy[j], nullptr, D, ctx.collision == 1, cp.v[3],
                    ctx.prandtl);
        store_vec<M>(D, out.c + (size_t)cell * NP);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) out.p[(size_t)cell * 4 + q4] = cp.v[q4];
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------ update (one cell)
// sweep_cell (single_level.cpp:103-111) + apply_update / update_delta
// (:44-70) after the face phase; executed by thread tid < 16 for cell (i, j).
template <int M, bool CG>
__device__ __forceinline__ int update_cell(const DevField& f, const DevField* rhs, const DevCtx& ctx,
                                           int i, int j, double* base, double* bad) {
  constexpr int NP = (Gen<M>::N + 3) & ~3;
  constexpr int N = Gen<M>::N;
  const int tid = threadIdx.x;
  const size_t cell = (size_t)j * f.nx + i;
  double* Ubase = base + (size_t)N * VS;
  double* S = Ubase + tid;        // cell state
  double* R = Ubase + 16 + tid;   // rhs projected
  double* D = Ubase + 32 + tid;   // assembled residual - rhs
  double* V = Ubase + 48 + tid;   // updated state
  load_vec<M, CG>(f.c + cell * NP, S);
  const P4 cp = ldp<CG>(f.p + cell * 4);
  // local_dt (single_level.cpp:18-24)
  if (!(cp.v[3] > 0.0)) return W_DT_THETA;
  const double cc = ctx.cfl_c_bound * sqrt(cp.v[3]);
  const double dt = ctx.cfl / ((fabs(cp.v[0]) + cc) / f.dx[i] + (fabs(cp.v[1]) + cc) / f.dy[j]);
  double nu, q[3];
  int w = collision_scalars<M>(S, cp, ctx, &nu, q);
  if (w) {
    if (w == W_NON_SPD) *bad = q[0];
    return w;
  }
  if (rhs) {
    load_vec<M, CG>(rhs->c + cell * NP, R);
    const P4 rp = ldp<CG>(rhs->p + cell * 4);
    project<M>(R, rp, cp);
  }
  assemble<M>(S, nu, q, ctx.collision == 2, ctx.shakhov_w, base + tid, base + 16 + tid,
              base + 32 + tid, base + 48 + tid, f.dx[i], f.dy[j], rhs ? R : nullptr, D, ctx.collision == 1,
              cp.v[3], ctx.prandtl);
  for (int attempt = 0; attempt < 2; ++attempt) {
    const double step = attempt == 0 ? dt : 0.5 * dt;
#pragma unroll
    for (int k = 0; k < N; ++k) V[k * VS] = fma(step, D[k * VS], S[k * VS]);
    P4 prm = cp;
    w = grad_normalize<M>(V, prm, bad);
    if (w == W_NONE) {
      store_vec<M>(V, f.c + cell * NP);
      __stcg(reinterpret_cast<double2*>(f.p + cell * 4), make_double2(prm.v[0], prm.v[1]));
      __stcg(reinterpret_cast<double2*>(f.p + cell * 4) + 1, make_double2(prm.v[2], prm.v[3]));
      return W_NONE;
    }
    if (code_for(w) != E_NONPHYSICAL) return w;
  }
  return W_DT_HALVING;
}

// ------------------------------------------- persistent exact-order sweep
// Work items are 16-cell segments of one anti-diagonal of one sweep,
// enumerated sweep-major then diagonal-major (a topological order); block b
// of the resident grid takes items b, b+G, ...  Per-cell completion counters
// give the exact lexicographic Gauss-Seidel dependencies (see
// sweep_persistent.cuh for the rule and the memory-ordering argument).
struct SegPlan {
  const int* diag_lo;     // first ii of anti-diagonal d
  const int* seg_start;   // prefix count of segments before diagonal d (size nd+1)
  unsigned* ver;
  int nd;                 // number of anti-diagonals
  int nsweeps;
  int dirs[8];
};

template <int M, int ORDER>
__global__ void __launch_bounds__(VS) k3_sweep(DevField f, DevField rhs, int has_rhs, DevCtx ctx,
                                               DevErr* err, SegPlan plan) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x;
  double* L = base + tid;
  double* U = base + (size_t)Gen<M>::N * VS + tid;
  const int per_sweep = plan.seg_start[plan.nd];
  const long long total = (long long)per_sweep * plan.nsweeps;
  constexpr int radius = ORDER == 2 ? 2 : 1;
  for (long long item = blockIdx.x; item < total; item += gridDim.x) {
    const int s = (int)(item / per_sweep);
    const int r = (int)(item - (long long)s * per_sweep);
    // diagonal of segment r: binary search in seg_start
    int lo = 0, hi = plan.nd - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (plan.seg_start[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int d = lo;
    const int seg = r - plan.seg_start[d];
    const int dlo = plan.diag_lo[d];
    const int dhi = d < f.nx - 1 ? d : f.nx - 1;
    const int ii = dlo + seg * SEG + (tid & 15);
    const bool valid = ii <= dhi;
    const int jj = d - ii;
    const int dir = plan.dirs[s & 7];
    const bool i_up = dir == 0 || dir == 3, j_up = dir == 0 || dir == 1;  // kSweepDirs
    const int i = valid ? (i_up ? ii : f.nx - 1 - ii) : 0;
    const int j = valid ? (j_up ? jj : f.ny - 1 - jj) : 0;
    // dependencies of this thread's face (+ self for the x-low thread)
    if (valid) {
      const int axis = tid >> 5, side = (tid >> 4) & 1;
      const int c = j * f.nx + i;
      bool ok = false;
      long long polls = 0;
      while (!ok) {
        ok = true;
        if (axis == 0 && side == 0 && ld_acquire(plan.ver + c) < (unsigned)s) ok = false;
#pragma unroll
        for (int dist = 1; dist <= radius; ++dist) {
          const int ni = axis == 0 ? (side ? i + dist : i - dist) : i;
          const int nj = axis == 1 ? (side ? j + dist : j - dist) : j;
          if (ni >= 0 && ni < f.nx && nj >= 0 && nj < f.ny) {
            const bool before = axis == 0 ? (i_up ? ni < i : ni > i) : (j_up ? nj < j : nj > j);
            if (ld_acquire(plan.ver + nj * f.nx + ni) < (unsigned)s + (before ? 1u : 0u)) ok = false;
          }
        }
        if (!ok) {
          if (err_on(err)) break;
          if (++polls > (1LL << 26)) {  // deadlock guard: fail loudly, never hang
            raise(err, E_ERROR, W_DEADLOCK, i, j, (double)s);
            break;
          }
          __nanosleep(64);
        }
      }
    }
    __syncthreads();
    if (err_on(err)) return;
    if (valid) {
      const int w = face_phase<M, ORDER, true>(f, ctx, i, j, L, U);
      if (w) raise(err, code_for(w), w, i, j, 0.0);
    }
    __syncthreads();
    if (err_on(err)) return;
    if (tid < SEG && valid) {
      double bad = 0.0;
      const int w = update_cell<M, true>(f, has_rhs ? &rhs : nullptr, ctx, i, j, base, &bad);
      if (w) raise(err, code_for(w), w, i, j, bad);
      else st_release(plan.ver + j * f.nx + i, (unsigned)s + 1u);
    }
    __syncthreads();
  }
}

// One anti-diagonal per launch (simple strategy, same results).
template <int M, int ORDER>
__global__ void __launch_bounds__(VS) k3_sweep_diag(DevField f, DevField rhs, int has_rhs, DevCtx ctx,
                                                    DevErr* err, int i_up, int j_up, int d, int ii0,
                                                    int count) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x;
  if (err_on(err)) return;
  const int q = blockIdx.x * SEG + (tid & 15);
  const bool valid = q < count;
  const int ii = ii0 + q, jj = d - ii;
  const int i = valid ? (i_up ? ii : f.nx - 1 - ii) : 0;
  const int j = valid ? (j_up ? jj : f.ny - 1 - jj) : 0;
  if (valid) {
    const int w = face_phase<M, ORDER, true>(f, ctx, i, j, base + tid, base + (size_t)Gen<M>::N * VS + tid);
    if (w) raise(err, code_for(w), w, i, j, 0.0);
  }
  __syncthreads();
  if (err_on(err)) return;
  if (tid < SEG && valid) {
    double bad = 0.0;
    const int w = update_cell<M, true>(f, has_rhs ? &rhs : nullptr, ctx, i, j, base, &bad);
    if (w) raise(err, code_for(w), w, i, j, bad);
  }
}

// ------------------------------------------------------------ transfer ops
// restrict_solution (multigrid.cpp:67-112): thread per coarse cell.
template <int M>
__global__ void __launch_bounds__(VS) k3_restrict_sol(DevField fine, DevField coarse, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  double* L = base + threadIdx.x;
  double* A = base + (size_t)N * VS + threadIdx.x;
  const int cells = coarse.nx * coarse.ny;
  for (int K = blockIdx.x * VS + threadIdx.x; K < cells; K += gridDim.x * VS) {
    if (err_on(err)) return;
    const int I = K % coarse.nx, J = K / coarse.nx;
    size_t child[4];
    double area[4];
    P4 cpar[4];
    double S = 0.0, mass = 0.0, energy = 0.0, mom[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      child[c] = (size_t)j * fine.nx + i;
      area[c] = fine.dx[i] * fine.dy[j];
      cpar[c] = ldp<false>(fine.p + child[c] * 4);
      const double rho = __ldg(fine.c + child[c] * NP);
      const double* u = cpar[c].v;
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
      raise(err, E_NONPHYSICAL, W_RESTRICT, I, J, rho_H);
      return;
    }
    for (int c = 0; c < 4; ++c) {
      load_vec<M, false>(fine.c + child[c] * NP, L);
      project<M>(L, cpar[c], basis);
      const double wgt = area[c] / S;
#pragma unroll
      for (int k = 0; k < N; ++k) A[k * VS] = c == 0 ? wgt * L[k * VS] : fma(wgt, L[k * VS], A[k * VS]);
    }
    double bad = 0.0;
    P4 prm = basis;
    const int w = grad_normalize<M>(A, prm, &bad);
    if (w) {
      raise(err, code_for(w), w, I, J, bad);
      return;
    }
    store_vec<M>(A, coarse.c + (size_t)K * NP);
#pragma unroll
    for (int q = 0; q < 4; ++q) coarse.p[(size_t)K * 4 + q] = prm.v[q];
  }
}

// restrict_residual (multigrid.cpp:114-142)
template <int M>
__global__ void __launch_bounds__(VS) k3_restrict_res(DevField arrays, DevField coarse, DevField out,
                                                      DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  double* L = base + threadIdx.x;
  double* A = base + (size_t)N * VS + threadIdx.x;
  const int cells = coarse.nx * coarse.ny;
  for (int K = blockIdx.x * VS + threadIdx.x; K < cells; K += gridDim.x * VS) {
    if (err_on(err)) return;
    const int I = K % coarse.nx, J = K / coarse.nx;
    const P4 basis = ldp<false>(coarse.p + (size_t)K * 4);
    if (!(basis.v[3] > 0.0)) {
      raise(err, E_NONPHYSICAL, W_PROJ_SPREAD, I, J, basis.v[3]);
      return;
    }
    double S = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) S += arrays.dx[2 * I + c % 2] * arrays.dy[2 * J + c / 2];
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + c % 2, j = 2 * J + c / 2;
      const size_t ch = (size_t)j * arrays.nx + i;
      load_vec<M, false>(arrays.c + ch * NP, L);
      project<M>(L, ldp<false>(arrays.p + ch * 4), basis);
      const double wgt = (arrays.dx[i] * arrays.dy[j]) / S;
#pragma unroll
      for (int k = 0; k < N; ++k) A[k * VS] = c == 0 ? wgt * L[k * VS] : fma(wgt, L[k * VS], A[k * VS]);
    }
    store_vec<M>(A, out.c + (size_t)K * NP);
#pragma unroll
    for (int q = 0; q < 4; ++q) out.p[(size_t)K * 4 + q] = basis.v[q];
  }
}

// fas_correct (multigrid.cpp:144-164): thread per fine cell.
template <int M>
__global__ void __launch_bounds__(VS) k3_fas(DevField fine, DevField before, DevField after, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  double* A = base + threadIdx.x;
  double* B = base + (size_t)N * VS + threadIdx.x;
  const int cells = fine.nx * fine.ny;
  for (int k = blockIdx.x * VS + threadIdx.x; k < cells; k += gridDim.x * VS) {
    if (err_on(err)) return;
    const int i = k % fine.nx, j = k / fine.nx;
    const size_t K = (size_t)(j / 2) * before.nx + (i / 2);
    const P4 cp = ldp<false>(fine.p + (size_t)k * 4);
    if (!(cp.v[3] > 0.0)) {
      raise(err, E_NONPHYSICAL, W_PROJ_SPREAD, i, j, cp.v[3]);
      return;
    }
    load_vec<M, false>(after.c + K * NP, A);
    project<M>(A, ldp<false>(after.p + K * 4), cp);
    load_vec<M, false>(before.c + K * NP, B);
    project<M>(B, ldp<false>(before.p + K * 4), cp);
    const double* fc = fine.c + (size_t)k * NP;
#pragma unroll
    for (int q = 0; q < N; ++q) A[q * VS] = __ldg(fc + q) + (A[q * VS] - B[q * VS]);
    double bad = 0.0;
    P4 prm = cp;
    int w = grad_normalize<M>(A, prm, &bad);
    if (w) {
      if (code_for(w) == E_NONPHYSICAL) w = W_FAS;
      raise(err, code_for(w), w, i, j, bad);
      return;
    }
    store_vec<M>(A, fine.c + (size_t)k * NP);
#pragma unroll
    for (int q = 0; q < 4; ++q) fine.p[(size_t)k * 4 + q] = prm.v[q];
  }
}

// euler_step (single_level.cpp:74-97): f <- f + dt (R - project(rhs -> cell
// basis)) with the global dt (device scalar from the global_dt reduction),
// then grad_normalize; a nonphysical result is retried once at dt/2 from the
// saved state (apply_update, :44-61), a second failure is SolverError(i, j).
// Thread per cell; the saved state stays in HBM until the store.
template <int M>
__global__ void __launch_bounds__(VS) k3_euler(DevField f, DevField res, DevField rhs, int has_rhs,
                                               const double* dt_dev, DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  double* D = base + threadIdx.x;
  double* V = base + (size_t)N * VS + threadIdx.x;
  const int cells = f.nx * f.ny;
  for (int k = blockIdx.x * VS + threadIdx.x; k < cells; k += gridDim.x * VS) {
    if (err_on(err)) return;
    const int i = k % f.nx, j = k / f.nx;
    const double dt = __ldcg(dt_dev);
    const P4 cp = ldp<false>(f.p + (size_t)k * 4);
    const double* rc = res.c + (size_t)k * NP;
    const double* fc = f.c + (size_t)k * NP;
    // update_delta (single_level.cpp:63-70)
    if (has_rhs) {
      load_vec<M, false>(rhs.c + (size_t)k * NP, D);
      project<M>(D, ldp<false>(rhs.p + (size_t)k * 4), cp);
#pragma unroll
      for (int q = 0; q < N; ++q) D[q * VS] = __ldg(rc + q) - D[q * VS];
    } else {
#pragma unroll
      for (int q = 0; q < N; ++q) D[q * VS] = __ldg(rc + q);
    }
    int w = W_NONE;
    double bad = 0.0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      const double step = attempt == 0 ? dt : 0.5 * dt;
#pragma unroll
      for (int q = 0; q < N; ++q) V[q * VS] = fma(step, D[q * VS], __ldg(fc + q));
      P4 prm = cp;
      w = grad_normalize<M>(V, prm, &bad);
      if (w == W_NONE) {
        store_vec<M>(V, f.c + (size_t)k * NP);
        __stcg(reinterpret_cast<double2*>(f.p + (size_t)k * 4), make_double2(prm.v[0], prm.v[1]));
        __stcg(reinterpret_cast<double2*>(f.p + (size_t)k * 4) + 1, make_double2(prm.v[2], prm.v[3]));
        break;
      }
      if (code_for(w) != E_NONPHYSICAL) break;  // plain Error propagates
    }
    if (w != W_NONE) {
      if (code_for(w) == E_NONPHYSICAL) w = W_DT_HALVING;
      raise(err, code_for(w), w, i, j, bad);
      return;
    }
  }
}

// nmg_cycle's defect (multigrid.cpp:178-185)
template <int M>
__global__ void __launch_bounds__(VS) k3_defect(DevField res, DevField rhs, int has_rhs, DevField out,
                                                DevErr* err) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* base = reinterpret_cast<double*>(smem_raw);
  constexpr int N = Gen<M>::N, NP = (N + 3) & ~3;
  double* A = base + threadIdx.x;
  const int cells = res.nx * res.ny;
  for (int k = blockIdx.x * VS + threadIdx.x; k < cells; k += gridDim.x * VS) {
    if (err_on(err)) return;
    const P4 rp = ldp<false>(res.p + (size_t)k * 4);
    const double* rc = res.c + (size_t)k * NP;
    double* oc = out.c + (size_t)k * NP;
    if (has_rhs) {
      if (!(rp.v[3] > 0.0)) {
        raise(err, E_NONPHYSICAL, W_PROJ_SPREAD, k % res.nx, k / res.nx, rp.v[3]);
        return;
      }
      load_vec<M, false>(rhs.c + (size_t)k * NP, A);
      project<M>(A, ldp<false>(rhs.p + (size_t)k * 4), rp);
#pragma unroll
      for (int q = 0; q < N; ++q) oc[q] = A[q * VS] - rc[q];
    } else {
#pragma unroll
      for (int q = 0; q < N; ++q) oc[q] = -rc[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) out.p[(size_t)k * 4 + q] = rp.v[q];
  }
}

}  // namespace tc
}  // namespace momg_gpu
