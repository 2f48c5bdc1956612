// Strip partition of a level: the device table shared by the band kernels
// (band_sweep.cuh) and the runtime (runtime.cu).
#pragma once

namespace momg_gpu {
namespace sp {

// Strip partition of one level: the grid's columns
// [i0[r], i0[r+1]) live in strip r's own arrays (its own allocation, on this
// GPU or peer-mapped from another rank's over NVLink).  A cell handle is then
// r << kStripShift | (j * width_r + i - i0[r]); without a table it is the flat
// index j * nx + i.
constexpr int kMaxStrips = 8;
constexpr int kStripShift = 27;
constexpr int kStripMask = (1 << kStripShift) - 1;
struct StripTab {
  int n;
  int i0[kMaxStrips + 1];
  double* c[kMaxStrips];
  double* p[kMaxStrips];
  unsigned* ver[kMaxStrips];
  double* oc[kMaxStrips];  // residual output of the fused residual tasks
  double* op[kMaxStrips];
};

}  // namespace sp
}  // namespace momg_gpu
