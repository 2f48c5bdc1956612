// Internal runtime interface shared by kernels.cu (device ops, C ABI) and
// driver.cu (the host NMG driver).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "../../include/momg_gpu.h"
#include "types.h"

struct momg_field {
  using DevField = momg_gpu::DevField;
  int M, N, NP, nx, ny;
  double Lx, Ly;
  std::vector<double> hdx, hdy, hxc, hyc;
  double* c = nullptr;
  double* p = nullptr;
  double* dgrid = nullptr;  // dx | dy | xc | yc
  uint32_t* sweep_order = nullptr;  // persistent sweep: diagonal order (lazy)
  unsigned* sweep_ver = nullptr;    // persistent sweep: per-cell counters (lazy)
  unsigned* band_next = nullptr;    // band sweep: task counter (lazy)
  int* seg_plan = nullptr;          // thread-granular sweep: diag_lo | seg_start (lazy)
  int* seg_plan32 = nullptr;        // split sweep (32-cell segments)
  cudaEvent_t ev_free = nullptr;        // overlapped transfers: last download of this field done
  // overlapped upload pending on the H2D copy stream: the library stream
  // waits on ev_ready the first time an entry point uses the field
  mutable cudaEvent_t ev_ready = nullptr;
  mutable bool ready_pending = false;
  DevField dev() const {
    DevField d;
    d.nx = nx;
    d.ny = ny;
    d.c = c;
    d.p = p;
    d.dx = dgrid;
    d.dy = dgrid + nx;
    d.xc = dgrid + nx + ny;
    d.yc = dgrid + 2 * nx + ny;
    return d;
  }
};


namespace momg_rt {
int ensure(momg_err* err);
int sync_check(momg_err* err);
int cuda_check(cudaError_t e, momg_err* err, const char* what);
cudaStream_t stream();
momg_gpu::DevErr* err_dev();
void count_launch(long long n);
long long launches();
// launch status of a kernel (cooperative launches return it; <<<>>> launches
// are checked through cudaGetLastError): the first failure is kept and
// reported as MOMG_ERR_CUDA by the next sync_check / fetch_scalar
void note_launch(cudaError_t e);
// make the library stream wait for a pending overlapped upload of f
void acquire(const momg_field* f);
}  // namespace momg_rt

namespace momg_gpu {
// One fused FS + residual launch over a strip-partitioned level (runtime.cu
// momg_strips_*; the table is a device-resident sp::StripTab)
struct StripLaunch {
  DevField geo;       // global nx, ny, dx, dy (c, p unused)
  const void* tab;    // device sp::StripTab
  unsigned* next;     // task counter of this process (zeroed by the caller)
  unsigned epoch;     // counters count from here
  int nbands, kb_up, kb_dn, nk, sys;  // 32-column bands (the k6 strips variant doubles them)
  int order[4];
  int iters;     // consecutive FS iterations (<= 4)
  int with_res;  // append the residual tasks (first order only)
};
// Per-moment-order launchers (kernels_m<M>.cu).
struct Ops {
  void (*residual)(const DevCtx&, const momg_field*, momg_field*);
  void (*sweep)(const DevCtx&, momg_field*, const momg_field*, const int*);
  void (*restrict_sol)(const momg_field*, momg_field*);
  void (*restrict_res)(const momg_field*, const momg_field*, momg_field*);
  void (*fas)(momg_field*, const momg_field*, const momg_field*);
  void (*defect)(const momg_field*, const momg_field*, momg_field*);
  void (*norm_partial)(const momg_field*, const momg_field*, double*, int);
  void (*sweep_n)(const DevCtx&, momg_field*, const momg_field*, const int*, int);
  bool (*sweep_res)(const DevCtx&, momg_field*, const int*, momg_field*, int);
  void (*euler)(const momg_field*, const momg_field*, const momg_field*, const double*);
  bool (*strips_sweep)(const DevCtx&, const StripLaunch&);
};
const Ops* ops_for(int M);
DevCtx make_ctx(const momg_ctx* c);
bool supported(int M);
momg_field* field_new(int M, int nx, int ny, double Lx, double Ly, const double* dx,
                      const double* dy, const double* xc, const double* yc, momg_err* err);
void field_free(momg_field* f);
// Stream-ordered device operations; errors are recorded on the device and
// surface at the next sync_check / fetch_scalar.
void op_residual(const DevCtx& ctx, const momg_field* f, momg_field* out);
void op_sweep(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int order[4]);
void op_sweep_n(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int order[4], int iters);
// fast_sweep_step (no rhs) then residual into out, fused into one launch where possible
void op_sweep_residual(const DevCtx& ctx, momg_field* f, const int order[4], momg_field* out, int iters = 1);
void op_restrict_sol(const momg_field* fine, momg_field* coarse);
void op_restrict_res(const momg_field* arrays, const momg_field* coarse, momg_field* out);
void op_fas(momg_field* fine, const momg_field* before, const momg_field* after);
void op_defect(const momg_field* res, const momg_field* rhs, momg_field* out);
void op_axpy(momg_field* dst, const momg_field* src);
void op_copy(momg_field* dst, const momg_field* src);
void op_mass(const momg_field* f, double target);
void op_scale_by_factor(momg_field* f);
// device-side check of the mass op_mass left (NonphysicalState when <= 0)
void op_mass_guard();
void op_norm(const momg_field* res, const momg_field* field);
void op_rscale(const DevCtx& ctx, const momg_field* f);
// global_dt (single_level.cpp:31-38): min local_dt, result left on the device
void op_global_dt(const DevCtx& ctx, const momg_field* f);
// euler_step (single_level.cpp:74-97) with the dt of the preceding op_global_dt
void op_euler(momg_field* f, const momg_field* residuals, const momg_field* rhs);
int fetch_scalar(double* out, momg_err* err);
}  // namespace momg_gpu
