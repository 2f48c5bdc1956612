// Second-order / rhs band sweep for moment order M=4 (band2_sweep.cuh),
// compiled with its own vector stride SPV = 21 (16-cell vectors + 4 halo slots).
#define SPV 21
#include "band2_sweep.cuh"

namespace momg_gpu {
void band2_launch_m4(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err,
                     const sp::Band2Plan& plan, cudaStream_t st) {
  band2_launch_impl<4>(f, rhs, ctx, err, plan, st);
}
void band2_strips_launch_m4(const DevField& geo, const DevCtx& ctx, DevErr* err, const sp::Band2Plan& plan,
                            cudaStream_t st) {
  band2_strips_launch_impl<4>(geo, ctx, err, plan, st);
}
}  // namespace momg_gpu
