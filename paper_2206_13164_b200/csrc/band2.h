// Host-side interface of the second-order / right-hand-side band sweep
// (band2_sweep.cuh, compiled in band2_m<M>.cu with its own vector stride).
#pragma once

#include <cuda_runtime.h>

#include "strips.h"
#include "types.h"

namespace momg_gpu {
namespace sp {
struct Band2Plan {
  unsigned* ver;   // per-cell sweep counters (zeroed per launch)
  unsigned* next;  // task counter (zeroed per launch)
  int nsweeps;     // <= 16
  int nbands;      // ceil(nx / 16)
  unsigned dirbits;
  int order;       // 1 | 2
  int has_rhs;
  int poll_ns;
  unsigned jitter;  // schedule perturbation seed (race stress tests; 0 = off)
  // strip partition (the k5 BandPlan fields of the same names; no rhs)
  const StripTab* strips;
  unsigned epoch;
  int kb_up, kb_dn, nk;
  int sys;
  const short* korder;          // blocked mode (BandPlan of band_sweep.cuh; 16-column bands)
  const unsigned char* bflags;
};
}  // namespace sp
struct DevCtx;
void band2_launch_m3(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err,
                     const sp::Band2Plan& plan, cudaStream_t st);
void band2_launch_m4(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err,
                     const sp::Band2Plan& plan, cudaStream_t st);
void band2_launch_m5(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err,
                     const sp::Band2Plan& plan, cudaStream_t st);
// the strip-partition variant (plan.strips set, no rhs)
void band2_strips_launch_m3(const DevField& geo, const DevCtx& ctx, DevErr* err, const sp::Band2Plan& plan,
                            cudaStream_t st);
void band2_strips_launch_m4(const DevField& geo, const DevCtx& ctx, DevErr* err, const sp::Band2Plan& plan,
                            cudaStream_t st);
void band2_strips_launch_m5(const DevField& geo, const DevCtx& ctx, DevErr* err, const sp::Band2Plan& plan,
                            cudaStream_t st);
}  // namespace momg_gpu
