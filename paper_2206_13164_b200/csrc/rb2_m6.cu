// Register-resident second-order / rhs band sweep for moment order M=6
// (reg_band2.cuh): 84 coefficients per cell, so 16-column bands (vector
// stride SPV = 19: 16 columns + two halo columns) and the half-range flux in
// place in shared memory.  BASELINE C4's NMG levels.
#define SPV 19
#include "reg_band2.cuh"

namespace momg_gpu {
void rb2_launch_m6(const DevField& f, const DevField& rhs, const DevCtx& ctx, DevErr* err, const sp::BandPlan& plan,
                   cudaStream_t st) {
  rb::rb2_launch_impl<6, 16>(f, rhs, ctx, err, plan, st);
}
}  // namespace momg_gpu
