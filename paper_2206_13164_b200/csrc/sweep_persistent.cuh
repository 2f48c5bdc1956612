// K2 (persistent): fast_sweep_step (single_level.cpp:121-166) as ONE
// persistent dataflow kernel that reproduces the exact lexicographic
// Gauss-Seidel dependency order of the reference without per-diagonal
// launches or sweep barriers.
//
// Work items are (sweep s, cell) pairs, enumerated sweep-major and, inside a
// sweep, anti-diagonal by anti-diagonal (a topological order of the sweep's
// dependency DAG).  Warp w of the resident grid takes items w, w+W, w+2W, ...
// Before updating cell c in sweep s it waits, per stencil neighbour n
// (radius 1 at first order, 2 at second order, spatial.cpp:34-50/106-124), on
// the per-cell completion counter ver[n]:
//   ver[n] >= s+1  if n precedes c in sweep s's order (new value, RAW),
//   ver[n] >= s    otherwise (value after sweep s-1),
// and on ver[c] >= s for itself.  A neighbour can never run ahead and
// overwrite a value c still needs: its own next update waits on ver[c] >= s+1.
// The same rule lets sweep s+1 start wherever sweep s has passed, so
// consecutive sweeps (and consecutive FS iterations, nsweeps = 4k) overlap.
// Deadlock freedom: items are taken in a topological order and every warp is
// resident (cooperative launch), so the smallest unfinished item can always
// run.  Counters are reset per launch.
//
// Memory ordering: lane q polls dependency q's counter with ld.acquire.gpu
// (synchronising with that writer's release); a __syncwarp then orders every
// lane's subsequent loads after all the acquires.  The writer stores with
// st.cg, __syncwarp, then lane 0 publishes the counter with st.release.gpu.
#pragma once

#include <cuda_runtime.h>

#include "momg_cell.cuh"
#include "runtime.h"

namespace momg_gpu {

constexpr int PWPB = 4;  // warps per block of the persistent sweep

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// spin-poll read: no L1 invalidation per iteration (ld.acquire emits
// CCTL.IVALL); a successful poll is confirmed with one ld_acquire.
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// system scope: counters and cells shared with peer GPUs over NVLink (row
// strips on several ranks; peer-mapped memory)
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_s(const unsigned* p, bool sys) {
  return sys ? ld_relaxed_sys(p) : ld_relaxed(p);
}
__device__ __forceinline__ unsigned ld_acquire_s(const unsigned* p, bool sys) {
  return sys ? ld_acquire_sys(p) : ld_acquire(p);
}
__device__ __forceinline__ void st_release_s(unsigned* p, unsigned v, bool sys) {
  if (sys) st_release_sys(p, v);
  else st_release(p, v);
}

struct SweepPlan {
  const uint32_t* order;  // diagonal-major (ii | jj << 16) for direction (i+, j+)
  unsigned* ver;          // per-cell completion counters (zeroed per launch)
  int nsweeps;            // 4 per FS iteration
  int dirs[8];            // direction index per sweep (mod 8)
};

template <int M, int ORDER>
__global__ void __launch_bounds__(PWPB * 32) k_sweep_persistent(DevField f, DevField rhs,
                                                                int has_rhs, DevCtx ctx,
                                                                DevErr* err, SweepPlan plan) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BlockView bv = block_setup<M, ORDER>(smem_raw, &ctx, &f, &rhs, nullptr, nullptr);
  WarpBuf<M, ORDER>& sb = warp_buf<M, ORDER>(bv);
  const int lane = lane_id();
  const long long cells = (long long)f.nx * f.ny;
  const long long total = cells * plan.nsweeps;
  const long long W = (long long)gridDim.x * PWPB;
  constexpr int radius = ORDER == 2 ? 2 : 1;
  for (long long item = blockIdx.x * (long long)PWPB + (threadIdx.x >> 5); item < total; item += W) {
    const int s = (int)(item / cells);
    const uint32_t packed = plan.order[item - (long long)s * cells];
    const int ii = packed & 0xffff, jj = packed >> 16;
    const int dir = plan.dirs[s & 7];
    const bool i_up = dir == 0 || dir == 3, j_up = dir == 0 || dir == 1;  // kSweepDirs
    const int i = i_up ? ii : f.nx - 1 - ii;
    const int j = j_up ? jj : f.ny - 1 - jj;
    const size_t c = (size_t)j * f.nx + i;
    // dependency q (lane q < 1 + 4*radius): 0 = self; then x-/x+/y-/y+ at
    // distance 1..radius
    int dn = -1;
    unsigned need = 0;
    if (lane == 0) {
      dn = (int)c;
      need = (unsigned)s;
    } else if (lane <= 4 * radius) {
      const int q = lane - 1;
      const int side = q % 4, dist = q / 4 + 1;
      const int ni = side == 0 ? i - dist : (side == 1 ? i + dist : i);
      const int nj = side == 2 ? j - dist : (side == 3 ? j + dist : j);
      if (ni >= 0 && ni < f.nx && nj >= 0 && nj < f.ny) {
        dn = nj * f.nx + ni;
        const bool before = side < 2 ? (i_up ? ni < i : ni > i) : (j_up ? nj < j : nj > j);
        need = (unsigned)s + (before ? 1u : 0u);
      }
    }
    bool ready = false;
    long long polls = 0;
    while (!ready) {
      bool mine = dn < 0 || ld_acquire(plan.ver + dn) >= need;
      ready = __all_sync(FULL, mine);
      if (!ready) {
        if (err_set(err)) return;
        if (++polls > (1LL << 26)) {  // deadlock guard: fail loudly, never hang
          if (lane == 0) raise_err(err, E_ERROR, W_DEADLOCK, i, j, (double)s);
          return;
        }
        __nanosleep(32);
      }
    }
    // lane q's acquire synchronises with dependency q's writer; the warp
    // barrier orders every lane's following loads after all of them.
    __syncwarp();
    double bad = 0.0;
    load_stencil<M, ORDER>(&bv.hdr->f, i, j, sb);
    const int w = sweep_cell<M, ORDER>(&bv.hdr->f, has_rhs ? &bv.hdr->g : nullptr, &bv.hdr->ctx,
                                       bv.tab, i, j, sb, &bad);
    if (w) {
      if (lane == 0) raise_err(err, code_of(w), w, i, j, bad);
      return;
    }
    __syncwarp();
    if (lane == 0) st_release(plan.ver + c, (unsigned)s + 1u);
  }
}

bool persistent_sweep_enabled();
void set_sweep_mode(int m);
// per-field cached diagonal order + counters
struct SweepScratch {
  uint32_t* order;
  unsigned* ver;
};
SweepScratch sweep_scratch(momg_field* f);

template <int M, int ORDER>
struct PersistentSweep {
  static size_t smem() { return BlockSmem<M, ORDER>::bytes(PWPB); }
  static int blocks() {
    static int nb = 0;
    if (nb) return nb;
    cudaFuncSetAttribute(k_sweep_persistent<M, ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem());
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_persistent<M, ORDER>, PWPB * 32, smem());
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    nb = per_sm * sms;
    return nb;
  }
  // nsweeps = 4 * iterations; order = the 4 direction indices of one FS call
  static void run(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int* order,
                  int iterations = 1) {
    SweepScratch sc = sweep_scratch(f);
    const long long cells = (long long)f->nx * f->ny;
    cudaMemsetAsync(sc.ver, 0, cells * sizeof(unsigned), momg_rt::stream());
    SweepPlan plan;
    plan.order = sc.order;
    plan.ver = sc.ver;
    plan.nsweeps = 4 * iterations;
    for (int s = 0; s < 8; ++s) plan.dirs[s] = order[s & 3];
    long long need = (cells * plan.nsweeps + PWPB - 1) / PWPB;
    int nb = blocks();
    if (need < nb) nb = (int)need;
    DevField fd = f->dev();
    DevField rd = rhs ? rhs->dev() : fd;
    int has_rhs = rhs != nullptr;
    DevErr* err = momg_rt::err_dev();
    DevCtx c = ctx;
    void* args[] = {&fd, &rd, &has_rhs, &c, &err, &plan};
    momg_rt::note_launch(cudaLaunchCooperativeKernel((void*)k_sweep_persistent<M, ORDER>, dim3(nb), dim3(PWPB * 32), args,
                                smem(), momg_rt::stream()));
    momg_rt::count_launch(1);
  }
};

}  // namespace momg_gpu
