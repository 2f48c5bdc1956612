// Register-resident second-order / rhs band sweep for moment order M=3
// (reg_band2.cuh), compiled with its own vector stride SPV = 35 (32 columns +
// two halo columns on one side).
#define SPV 35
#include "reg_band2.cuh"

namespace momg_gpu {
void rb2_launch_m3(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err, const sp::BandPlan& plan,
                   cudaStream_t st) {
  rb::rb2_launch_impl<3, 32>(f, rhs, ctx, err, plan, st);
}
}  // namespace momg_gpu
