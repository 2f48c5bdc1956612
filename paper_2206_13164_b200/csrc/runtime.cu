// Runtime, simple kernels (reductions, axpy, scale, fill) and the C ABI of
// include/momg_gpu.h.  The per-cell kernels live in kernels_impl.cuh
// (instantiated per moment order in kernels_m<M>.cu); the host NMG driver in
// driver.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/momg_gpu.h"
#include "momg_cell.cuh"
#include "runtime.h"
#include "sweep_persistent.cuh"
#include "kernels_v3.cuh"

namespace momg_gpu {

__global__ void k_axpy(double* dst, const double* src, size_t n, const DevErr* err) {
  if (err_set(err)) return;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x)
    dst[q] += src[q];
}

// defect without a right-hand side (multigrid.cpp:183-185: defect = -res):
// a flat, coalesced pass over the coefficient records (padding copied) and
// the basis parameters (copied: the defect keeps the residual's basis)
__global__ void k_negate(const double* __restrict__ src_c, const double* __restrict__ src_p, double* dst_c,
                         double* dst_p, size_t ncoef, int N, int NP, size_t nparam, const DevErr* err) {
  if (err_set(err)) return;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < ncoef; q += stride)
    dst_c[q] = (int)(q % NP) < N ? -src_c[q] : src_c[q];
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < nparam; q += stride) dst_p[q] = src_p[q];
}

// mass_correction's check (single_level.cpp:176-183) on the device, so a
// solve iteration needs no host round trip before the rescale: a nonpositive
// or non-finite current mass is recorded as NonphysicalState and every later
// kernel of the iteration early-exits
__global__ void k_mass_guard(const double* current, DevErr* err) {
  const double m = *current;
  if (threadIdx.x == 0 && (!(m > 0.0) || !isfinite(m)) && atomicCAS(&err->code, 0, E_NONPHYSICAL) == 0) {
    err->what = W_MASS;
    err->i = err->j = -1;
    err->value = m;
    __threadfence();
  }
}

__global__ void k_scale_by(double* c, size_t n, double factor) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x)
    c[q] *= factor;
}

__global__ void k_scale(double* c, size_t n, const double* factor_dev, const DevErr* err) {
  if (err_set(err)) return;
  const double f = *factor_dev;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x)
    c[q] *= f;
}

__global__ void k_fill(DevField f, int NP, double rho, double ux, double uy, double uz,
                       double theta) {
  const size_t cells = (size_t)f.nx * f.ny;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < cells * NP; q += (size_t)gridDim.x * blockDim.x)
    f.c[q] = (q % NP) == 0 ? rho : 0.0;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < cells; q += (size_t)gridDim.x * blockDim.x) {
    f.p[q * 4] = ux;
    f.p[q * 4 + 1] = uy;
    f.p[q * 4 + 2] = uz;
    f.p[q * 4 + 3] = theta;
  }
}

// ------------------------------------------------------------ reductions
// Deterministic two-stage reductions: block b reduces the row-major cell
// range [b*chunk, (b+1)*chunk) in a fixed tree order; one block then sums the
// partials in order.  (The reference sums row-major serially; the order
// differs, the result agrees to ~1e-16 relative.)
constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 592;  // 4 x 148 SMs

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(FULL, t, o);
  }
  return t;
}
__device__ __forceinline__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = smax(v, __shfl_down_sync(FULL, v, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = -INFINITY;
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) t = smax(t, __shfl_down_sync(FULL, t, o));
  }
  return t;
}

// total_mass partials: sum rho_ij * dx_i * dy_j
__global__ void k_mass_partial(DevField f, int NP, double* partial) {
  __shared__ double sh[32];
  const int cells = f.nx * f.ny;
  const int chunk = (cells + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * chunk, hi = min(cells, lo + chunk);
  double v = 0.0;
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const int i = k % f.nx, j = k / f.nx;
    v += f.c[(size_t)k * NP] * (f.dx[i] * f.dy[j]);
  }
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// residual_scale partials: max rho (C sqrt(theta)(1/dx + 1/dy) + nu)
__global__ void k_rscale_partial(DevField f, int NP, DevCtx ctx, double* partial) {
  __shared__ double sh[32];
  const int cells = f.nx * f.ny;
  const int chunk = (cells + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * chunk, hi = min(cells, lo + chunk);
  double v = 0.0;
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const int i = k % f.nx, j = k / f.nx;
    const double rho = f.c[(size_t)k * NP];
    const double theta = f.p[(size_t)k * 4 + 3];
    const double nu = ctx.nu_coef * rho * pow(theta, ctx.nu_exp);
    v = smax(v, rho * (ctx.cfl_c_bound * sqrt(theta) * (1.0 / f.dx[i] + 1.0 / f.dy[j]) + nu));
  }
  const double t = block_max(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// global_dt partials (single_level.cpp:31-38): max of -local_dt, so the
// final max stage yields -min; a nonpositive temperature raises
// NonphysicalState like local_dt (:20-21)
__global__ void k_dt_partial(DevField f, DevCtx ctx, double* partial, DevErr* err) {
  __shared__ double sh[32];
  const int cells = f.nx * f.ny;
  const int chunk = (cells + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * chunk, hi = min(cells, lo + chunk);
  double v = -INFINITY;
  for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const int i = k % f.nx, j = k / f.nx;
    const double ux = f.p[(size_t)k * 4], uy = f.p[(size_t)k * 4 + 1], theta = f.p[(size_t)k * 4 + 3];
    if (!(theta > 0.0)) {
      raise_err(err, E_NONPHYSICAL, W_DT_THETA, i, j, theta);
      continue;
    }
    const double c = ctx.cfl_c_bound * sqrt(theta);
    const double dt = ctx.cfl / ((fabs(ux) + c) / f.dx[i] + (fabs(uy) + c) / f.dy[j]);
    v = smax(v, -dt);
  }
  const double t = block_max(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// final stage: out[0] = sum (or max) of partial[0..n); optional
// out[1] = target / out[0] (mass correction factor); mode 0 sum, 1 max,
// 2 sqrt(sum / area)
__global__ void k_final(const double* partial, int n, int mode, double arg, double* out) {
  __shared__ double sh[32];
  // mode 3: max of negated values -> out[0] = -max (a minimum)
  const bool mx = mode == 1 || mode == 3;
  double v = mode == 3 ? -INFINITY : 0.0;
  for (int q = threadIdx.x; q < n; q += blockDim.x) v = mx ? smax(v, partial[q]) : v + partial[q];
  const double t = mx ? block_max(v, sh) : block_sum(v, sh);
  if (threadIdx.x == 0) {
    out[0] = mode == 2 ? sqrt(t / arg) : mode == 3 ? -t : t;
    out[1] = arg / t;
  }
}

}  // namespace momg_gpu

// =====================================================================
//                              runtime + C ABI
// =====================================================================
using namespace momg_gpu;

namespace momg_rt {

static std::mutex g_mu;
static cudaStream_t g_stream = nullptr;
static bool g_own_stream = false;
static int g_device = -1;
static DevErr* g_err_dev = nullptr;
static DevErr* g_err_host = nullptr;  // pinned
static double* g_red = nullptr;       // partials [RED_BLOCKS] + out[4]
static double* g_red_host = nullptr;  // pinned out[4]
static std::atomic<long long> g_launches{0};

static std::atomic<int> g_launch_err{0};  // first failed launch (cudaError_t)
void count_launch(long long n) { g_launches += n; }
void note_launch(cudaError_t e) {
  int expected = 0;
  if (e != cudaSuccess) g_launch_err.compare_exchange_strong(expected, (int)e);
}
void acquire(const momg_field* f) {
  if (f && f->ready_pending) {
    cudaStreamWaitEvent(g_stream, f->ev_ready, 0);
    f->ready_pending = false;
  }
}
long long launches() { return g_launches.load(); }
cudaStream_t stream() { return g_stream; }
DevErr* err_dev() { return g_err_dev; }

static void set(momg_err* err, int code, const char* msg, int i = -1, int j = -1) {
  if (!err) return;
  err->code = code;
  err->i = i;
  err->j = j;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
}

int ensure(momg_err* err) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_err_dev) return MOMG_OK;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    set(err, MOMG_ERR_NO_DEVICE, "momg_gpu: no CUDA device available (no CPU fallback)");
    return MOMG_ERR_NO_DEVICE;
  }
  if (g_device < 0) cudaGetDevice(&g_device);
  cudaSetDevice(g_device);
  if (!g_stream) {
    if (cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking) != cudaSuccess) {
      set(err, MOMG_ERR_CUDA, "momg_gpu: stream creation failed");
      return MOMG_ERR_CUDA;
    }
    g_own_stream = true;
  }
  if (cudaMalloc(&g_err_dev, sizeof(DevErr)) != cudaSuccess ||
      cudaMallocHost(&g_err_host, sizeof(DevErr)) != cudaSuccess ||
      cudaMalloc(&g_red, sizeof(double) * (RED_BLOCKS + 8)) != cudaSuccess ||
      cudaMallocHost(&g_red_host, sizeof(double) * 8) != cudaSuccess) {
    set(err, MOMG_ERR_CUDA, "momg_gpu: runtime allocation failed");
    return MOMG_ERR_CUDA;
  }
  cudaMemset(g_err_dev, 0, sizeof(DevErr));
  cudaDeviceSynchronize();
  return MOMG_OK;
}

int cuda_check(cudaError_t e, momg_err* err, const char* what) {
  if (e == cudaSuccess) return MOMG_OK;
  char buf[256];
  std::snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  set(err, MOMG_ERR_CUDA, buf);
  return MOMG_ERR_CUDA;
}

static const char* what_text(int w) {
  switch (w) {
    case W_GRAD_RHO: return "grad_normalize: nonpositive or non-finite density";
    case W_GRAD_THETA: return "grad_normalize: nonpositive or non-finite temperature";
    case W_GRAD_U: return "grad_normalize: non-finite velocity";
    case W_GRAD_CAP: return "grad_normalize: tolerance not reached within iteration cap";
    case W_PROJ_SPREAD: return "project_coeffs: target spread must be positive";
    case W_MACRO_RHO: return "extract_macro: nonpositive density";
    case W_WALL_DEGEN: return "wall_flux: degenerate incoming wall flux";
    case W_WALL_RHO: return "wall_flux: nonpositive wall density";
    case W_HALF_SPREAD: return "half_flux_coeffs: nonpositive basis spread";
    case W_DT_THETA: return "local_dt: nonpositive temperature";
    case W_DT_HALVING: return "update left cell nonphysical after dt halving";
    case W_FAS: return "coarse-grid correction left cell nonphysical";
    case W_RESTRICT: return "restrict_solution: nonphysical coarse state";
    case W_ES_UNSUPPORTED: return "ES-BGK collision is not available on the device path";
    case W_DEADLOCK: return "persistent sweep: dependency wait timed out (internal error)";
    case W_MASS: return "mass_correction: nonpositive total mass";
    case W_NON_SPD: return "equilibrium_rep: anisotropic-Gaussian tensor not SPD";
    default: return "unknown failure";
  }
}

// Synchronises the stream and converts a device error record into *err
// (then clears it).  Returns the status.
int sync_check(momg_err* err) {
  // a kernel that failed to launch (bad configuration, shared-memory
  // attribute, cooperative grid too large) is an error, not a no-op
  cudaError_t le = cudaGetLastError();
  const int noted = g_launch_err.exchange(0);
  if (le == cudaSuccess && noted) le = (cudaError_t)noted;
  if (le != cudaSuccess) {
    cudaStreamSynchronize(g_stream);
    return cuda_check(le, err, "momg_gpu: kernel launch failed");
  }
  cudaError_t e = cudaMemcpyAsync(g_err_host, g_err_dev, sizeof(DevErr), cudaMemcpyDeviceToHost,
                                  g_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g_stream);
  if (int rc = cuda_check(e, err, "momg_gpu")) return rc;
  if (g_err_host->code == 0) return MOMG_OK;
  char buf[256];
  std::snprintf(buf, sizeof(buf), "%s at cell (%d,%d) [value %g]", what_text(g_err_host->what),
                g_err_host->i, g_err_host->j, g_err_host->value);
  const int code = g_err_host->code;
  set(err, code, buf, g_err_host->i, g_err_host->j);
  cudaMemsetAsync(g_err_dev, 0, sizeof(DevErr), g_stream);
  cudaStreamSynchronize(g_stream);
  return code;
}

double* red_buf() { return g_red; }
double* red_host() { return g_red_host; }

static cudaStream_t g_own = nullptr;  // the library's own stream (kept for a switch back)
// Switch the library stream: work still pending on the old stream is waited
// for first, so nothing enqueued before the switch (field zero-fills, async
// copies) can race with what follows on the new one.  NULL restores the
// library's own stream.
void set_stream(cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_stream) cudaStreamSynchronize(g_stream);
  if (g_own_stream && g_stream && !g_own) g_own = g_stream;
  if (!s) {
    if (!g_own) cudaStreamCreateWithFlags(&g_own, cudaStreamNonBlocking);
    s = g_own;
  }
  g_stream = s;
  g_own_stream = s == g_own;
}

int init_device(int device, momg_err* err) {
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (g_err_dev && device != g_device) {
      set(err, MOMG_ERR_ARG, "momg_init: already initialised on another device");
      return MOMG_ERR_ARG;
    }
    g_device = device;
  }
  return ensure(err);
}

}  // namespace momg_rt

namespace momg_gpu {

DevCtx make_ctx(const momg_ctx* c) {
  DevCtx d;
  d.order = c->space_order;
  d.collision = c->collision;
  d.c_bound = c->c_bound;
  d.cfl = c->cfl;
  d.cfl_c_bound = c->cfl_c_bound;
  const double root_half_pi = std::sqrt(std::atan(1.0) * 2.0);
  const double beta = c->collision == MOMG_ES_BGK ? c->prandtl : 1.0;
  d.nu_coef = beta * root_half_pi / c->knudsen;
  d.nu_exp = 1.0 - c->viscosity_index;
  d.shakhov_w = (1.0 - c->prandtl) / 5.0;
  d.prandtl = c->prandtl;
  d.threads = c->threads;
  for (int w = 0; w < 4; ++w) {
    d.wall_speed[w] = c->wall_speed[w];
    d.wall_theta[w] = c->wall_theta[w];
  }
  return d;
}

const Ops* ops_m3();
const Ops* ops_m4();
const Ops* ops_m5();
const Ops* ops_m6();
const Ops* ops_m7();
const Ops* ops_m8();

const Ops* ops_for(int M) {
  switch (M) {
    case 3: return ops_m3();
    case 4: return ops_m4();
    case 5: return ops_m5();
    case 6: return ops_m6();
    case 7: return ops_m7();
    case 8: return ops_m8();
    default: return nullptr;
  }
}

bool supported(int M) { return M >= 3 && M <= 8; }

static int g_sweep_mode = -1;  // 0 per-diagonal launches, 1 persistent dataflow

bool persistent_sweep_enabled() {
  if (g_sweep_mode < 0) {
    const char* e = std::getenv("MOMG_SWEEP");
    g_sweep_mode = (e && std::string(e) == "diag") ? 0 : 1;
  }
  return g_sweep_mode == 1;
}
void set_sweep_mode(int m) { g_sweep_mode = m; }
void set_band_mode(int m);
void set_rb_mode(int m);
void set_trace(long long cap);
long long read_trace(unsigned long long* host, long long n);

// Segment plan of the thread-granular persistent sweep (kernels_v3.cuh):
// diag_lo[d] and the prefix count of 16-cell segments per anti-diagonal,
// cached per field; counters shared with the warp-granular sweep.
tc::SegPlan tc_seg_plan(momg_field* f, int seg) {
  const int nd = f->nx + f->ny - 1;
  int*& plan_ptr = seg == 32 ? f->seg_plan32 : f->seg_plan;
  if (!plan_ptr) {
    std::vector<int> h(2 * nd + 1);
    int acc = 0;
    for (int d = 0; d < nd; ++d) {
      const int lo = d - (f->ny - 1) > 0 ? d - (f->ny - 1) : 0;
      const int hi = d < f->nx - 1 ? d : f->nx - 1;
      h[d] = lo;
      h[nd + d] = acc;
      acc += (hi - lo + 1 + seg - 1) / seg;
    }
    h[2 * nd] = acc;
    cudaMalloc(&plan_ptr, h.size() * sizeof(int));
    cudaMemcpy(plan_ptr, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice);
  }
  if (!f->sweep_ver) cudaMalloc(&f->sweep_ver, (size_t)f->nx * f->ny * sizeof(unsigned));
  cudaMemsetAsync(f->sweep_ver, 0, (size_t)f->nx * f->ny * sizeof(unsigned), momg_rt::stream());
  tc::SegPlan p;
  p.diag_lo = plan_ptr;
  p.seg_start = plan_ptr + nd;
  p.ver = f->sweep_ver;
  p.nd = nd;
  p.nsweeps = 4;
  for (int s = 0; s < 8; ++s) p.dirs[s] = s & 3;
  return p;
}

}  // namespace momg_gpu

namespace momg_gpu {

static unsigned long long* g_trace = nullptr;
static long long g_trace_cap = 0;
unsigned long long* trace_buffer(long long* cap) {
  *cap = g_trace_cap;
  return g_trace;
}
void set_trace(long long cap) {
  if (g_trace) cudaFree(g_trace);
  g_trace = nullptr;
  g_trace_cap = 0;
  if (cap > 0 && cudaMalloc(&g_trace, cap * 8 * sizeof(unsigned long long)) == cudaSuccess) {
    cudaMemset(g_trace, 0, cap * 8 * sizeof(unsigned long long));
    g_trace_cap = cap;
  }
}
long long read_trace(unsigned long long* host, long long n) {
  if (!g_trace) return 0;
  if (n > g_trace_cap) n = g_trace_cap;
  cudaMemcpy(host, g_trace, n * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return n;
}

// schedule perturbation for the race stress tests (MOMG_JITTER=<seed>, read
// at every launch): the band kernels sleep pseudo-random 0-2 us before task
// claims, publications and polls, so the inter-CTA protocol runs under other
// interleavings; results must stay bitwise identical
unsigned sched_jitter_seed() {
  const char* e = std::getenv("MOMG_JITTER");
  return e ? (unsigned)std::strtoul(e, nullptr, 10) : 0u;
}

// Blocked-parallel sweep plan (BandPlan::korder / bflags) for T workers on
// the nx / band bands (32 columns: k5_band, 16: k6_band): the reference's blocks [nx b / T, nx (b+1) / T)
// (single_level.cpp:137-141) when every boundary is a band boundary, else
// null (the exact order, itself one outcome of the reference's blocked run:
// the workers finishing in block order).  Cached per (T, nx, band).
bool blocked_plan(int T, int nx, int band, const short** korder, const unsigned char** bflags) {
  *korder = nullptr;
  *bflags = nullptr;
  if (T <= 1 || nx % band || T > nx) return false;
  const int nb = nx / band;
  std::vector<int> lo(T + 1);
  for (int b = 0; b <= T; ++b) {
    lo[b] = (int)((long long)nx * b / T);
    if (lo[b] % band) return false;
  }
  struct Entry {
    int T, nx, band;
    short* ko;
    unsigned char* bf;
  };
  static std::vector<Entry> cache;
  for (const Entry& e : cache)
    if (e.T == T && e.nx == nx && e.band == band) {
      *korder = e.ko;
      *bflags = e.bf;
      return true;
    }
  std::vector<short> ko(2 * nb);
  std::vector<unsigned char> bf(2 * nb, 0);
  for (int fr = 0; fr < 2; ++fr) {
    std::vector<int> rb;  // rotated block boundaries in bands, ascending
    for (int b = 0; b <= T; ++b) rb.push_back(fr == 0 ? lo[b] / band : (nx - lo[T - b]) / band);
    int pos = 0;
    for (int t = T - 1; t >= 0; --t) {  // blocks in descending rotated order
      for (int k = rb[t]; k < rb[t + 1]; ++k) ko[fr * nb + pos++] = (short)k;
      if (rb[t + 1] > rb[t]) {
        if (t > 0) bf[fr * nb + rb[t]] |= 1;
        if (t + 1 < T) bf[fr * nb + rb[t + 1] - 1] |= 2;
      }
    }
  }
  Entry e{T, nx, band, nullptr, nullptr};
  cudaMalloc(&e.ko, ko.size() * sizeof(short));
  cudaMalloc(&e.bf, bf.size());
  cudaMemcpy(e.ko, ko.data(), ko.size() * sizeof(short), cudaMemcpyHostToDevice);
  cudaMemcpy(e.bf, bf.data(), bf.size(), cudaMemcpyHostToDevice);
  cache.push_back(e);
  *korder = e.ko;
  *bflags = e.bf;
  return true;
}

void band_scratch(momg_field* f, unsigned** ver, unsigned** next) {
  if (!f->sweep_ver) cudaMalloc(&f->sweep_ver, (size_t)f->nx * f->ny * sizeof(unsigned));
  if (!f->band_next) cudaMalloc(&f->band_next, 64);
  cudaMemsetAsync(f->sweep_ver, 0, (size_t)f->nx * f->ny * sizeof(unsigned), momg_rt::stream());
  cudaMemsetAsync(f->band_next, 0, 64, momg_rt::stream());
  *ver = f->sweep_ver;
  *next = f->band_next;
}

// band kernels for M <= 5 (momg_set_sweep_mode: 1 on, 0 / 2 off)
static int g_band = 1;
bool band_sweep_enabled() { return g_band == 1 && persistent_sweep_enabled(); }
void set_band_mode(int m) { g_band = m; }
// register-resident band kernel (reg_band.cuh) vs the split k5_band
static int g_rb = -1;
bool rb_enabled() {
  if (g_rb < 0) {
    const char* e = getenv("MOMG_RB");
    g_rb = (e && std::string(e) == "0") ? 0 : 1;
  }
  return g_rb == 1;
}
void set_rb_mode(int m) { g_rb = m; }

int rb_grid_cap(int nb, int nk) {
  static const int env = [] {
    const char* e = getenv("MOMG_RB_GRID");
    return e ? atoi(e) : 0;
  }();
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  // 1.5 nk running + waiting tasks, and at most ~2/3 of the SMs: beyond that the
  // second CTA of a TPC costs more than its task gains (4096^2: 290 ms at 96
  // CTAs, 314 ms at 148, 361 ms at 64)
  int cap = (3 * nk + 1) / 2;
  const int tpc = (sms * 13) / 20;
  if (cap > tpc) cap = tpc;
  if (env > 0) cap = env;
  return nb < cap ? nb : (cap < 1 ? 1 : cap);
}
int tc_sweep_blocks(const void* kernel, size_t smem, int threads) {
  int per_sm = 0, dev = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

// Diagonal-major visiting order of direction (i+, j+) (ii | jj << 16) and the
// per-cell counters of the persistent sweep, cached per field.
SweepScratch sweep_scratch(momg_field* f) {
  if (!f->sweep_order) {
    const int nx = f->nx, ny = f->ny;
    std::vector<uint32_t> order;
    order.reserve((size_t)nx * ny);
    for (int d = 0; d <= nx + ny - 2; ++d) {
      const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
      const int hi = d < nx - 1 ? d : nx - 1;
      for (int ii = lo; ii <= hi; ++ii) order.push_back((uint32_t)ii | ((uint32_t)(d - ii) << 16));
    }
    cudaMalloc(&f->sweep_order, order.size() * sizeof(uint32_t));
    cudaMalloc(&f->sweep_ver, order.size() * sizeof(unsigned));
    cudaMemcpy(f->sweep_order, order.data(), order.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  }
  return SweepScratch{f->sweep_order, f->sweep_ver};
}

// ------------------------------------------ internal (deferred-check) ops
void op_residual(const DevCtx& ctx, const momg_field* f, momg_field* out) {
  ops_for(f->M)->residual(ctx, f, out);
}
void op_sweep(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int order[4]) {
  ops_for(f->M)->sweep(ctx, f, rhs, order);
}
void op_sweep_n(const DevCtx& ctx, momg_field* f, const momg_field* rhs, const int order[4], int iters) {
  ops_for(f->M)->sweep_n(ctx, f, rhs, order, iters);
}
void op_restrict_sol(const momg_field* fine, momg_field* coarse) {
  ops_for(fine->M)->restrict_sol(fine, coarse);
}
void op_restrict_res(const momg_field* arrays, const momg_field* coarse, momg_field* out) {
  ops_for(arrays->M)->restrict_res(arrays, coarse, out);
}
void op_fas(momg_field* fine, const momg_field* before, const momg_field* after) {
  ops_for(fine->M)->fas(fine, before, after);
}
void op_sweep_residual(const DevCtx& ctx, momg_field* f, const int order[4], momg_field* out, int iters) {
  if (ops_for(f->M)->sweep_res(ctx, f, order, out, iters)) return;
  op_sweep_n(ctx, f, nullptr, order, iters);
  op_residual(ctx, f, out);
}
void op_defect(const momg_field* res, const momg_field* rhs, momg_field* out) {
  if (!rhs) {
    const size_t cells = (size_t)res->nx * res->ny;
    k_negate<<<148 * 8, 256, 0, momg_rt::stream()>>>(res->c, res->p, out->c, out->p, cells * res->NP, res->N,
                                                     res->NP, cells * 4, momg_rt::err_dev());
    momg_rt::count_launch(1);
    return;
  }
  ops_for(res->M)->defect(res, rhs, out);
}
void op_axpy(momg_field* dst, const momg_field* src) {
  const size_t n = (size_t)dst->nx * dst->ny * dst->NP;
  k_axpy<<<592, 256, 0, momg_rt::stream()>>>(dst->c, src->c, n, momg_rt::err_dev());
  momg_rt::count_launch(1);
}
void op_copy(momg_field* dst, const momg_field* src) {
  const size_t cells = (size_t)dst->nx * dst->ny;
  cudaMemcpyAsync(dst->c, src->c, cells * dst->NP * sizeof(double), cudaMemcpyDeviceToDevice,
                  momg_rt::stream());
  cudaMemcpyAsync(dst->p, src->p, cells * 4 * sizeof(double), cudaMemcpyDeviceToDevice,
                  momg_rt::stream());
}
// Reductions leave their result in red_buf()[RED_BLOCKS + 0..1] on device.
void op_mass(const momg_field* f, double target) {
  k_mass_partial<<<RED_BLOCKS, RED_THREADS, 0, momg_rt::stream()>>>(f->dev(), f->NP,
                                                                     momg_rt::red_buf());
  k_final<<<1, 1024, 0, momg_rt::stream()>>>(momg_rt::red_buf(), RED_BLOCKS, 0, target,
                                             momg_rt::red_buf() + RED_BLOCKS);
  momg_rt::count_launch(2);
}
void op_mass_guard() {
  k_mass_guard<<<1, 32, 0, momg_rt::stream()>>>(momg_rt::red_buf() + RED_BLOCKS, momg_rt::err_dev());
  momg_rt::count_launch(1);
}
void op_scale_by_factor(momg_field* f) {
  const size_t n = (size_t)f->nx * f->ny * f->NP;
  k_scale<<<592, 256, 0, momg_rt::stream()>>>(f->c, n, momg_rt::red_buf() + RED_BLOCKS + 1,
                                              momg_rt::err_dev());
  momg_rt::count_launch(1);
}
void op_norm(const momg_field* res, const momg_field* field) {
  ops_for(res->M)->norm_partial(res, field, momg_rt::red_buf(), RED_BLOCKS);
  k_final<<<1, 1024, 0, momg_rt::stream()>>>(momg_rt::red_buf(), RED_BLOCKS, 2,
                                             field->Lx * field->Ly,
                                             momg_rt::red_buf() + RED_BLOCKS);
  momg_rt::count_launch(1);
}
void op_rscale(const DevCtx& ctx, const momg_field* f) {
  k_rscale_partial<<<RED_BLOCKS, RED_THREADS, 0, momg_rt::stream()>>>(f->dev(), f->NP, ctx,
                                                                       momg_rt::red_buf());
  k_final<<<1, 1024, 0, momg_rt::stream()>>>(momg_rt::red_buf(), RED_BLOCKS, 1, 1.0,
                                             momg_rt::red_buf() + RED_BLOCKS);
  momg_rt::count_launch(2);
}
void op_global_dt(const DevCtx& ctx, const momg_field* f) {
  k_dt_partial<<<RED_BLOCKS, RED_THREADS, 0, momg_rt::stream()>>>(f->dev(), ctx, momg_rt::red_buf(),
                                                                   momg_rt::err_dev());
  k_final<<<1, 1024, 0, momg_rt::stream()>>>(momg_rt::red_buf(), RED_BLOCKS, 3, 1.0,
                                             momg_rt::red_buf() + RED_BLOCKS);
  momg_rt::count_launch(2);
}
void op_euler(momg_field* f, const momg_field* residuals, const momg_field* rhs) {
  ops_for(f->M)->euler(f, residuals, rhs, momg_rt::red_buf() + RED_BLOCKS);
}
// Fetches the reduction result (synchronising); also reports device errors.
int fetch_scalar(double* out, momg_err* err) {
  cudaMemcpyAsync(momg_rt::red_host(), momg_rt::red_buf() + RED_BLOCKS, 2 * sizeof(double),
                  cudaMemcpyDeviceToHost, momg_rt::stream());
  const int rc = momg_rt::sync_check(err);
  if (out) *out = momg_rt::red_host()[0];
  return rc;
}

momg_field* field_new(int M, int nx, int ny, double Lx, double Ly, const double* dx,
                      const double* dy, const double* xc, const double* yc, momg_err* err) {
  momg_field* f = new momg_field();
  f->M = M;
  f->N = tet(M + 1);
  f->NP = (f->N + 3) & ~3;
  f->nx = nx;
  f->ny = ny;
  f->Lx = Lx;
  f->Ly = Ly;
  f->hdx.assign(dx, dx + nx);
  f->hdy.assign(dy, dy + ny);
  f->hxc.assign(xc, xc + nx);
  f->hyc.assign(yc, yc + ny);
  const size_t cells = (size_t)nx * ny;
  cudaError_t e = cudaMalloc(&f->c, cells * f->NP * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&f->p, cells * 4 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&f->dgrid, (2 * nx + 2 * ny) * sizeof(double));
  if (e != cudaSuccess) {
    momg_rt::cuda_check(e, err, "momg_field_create");
    cudaFree(f->c);
    cudaFree(f->p);
    cudaFree(f->dgrid);
    delete f;
    return nullptr;
  }
  std::vector<double> g;
  g.insert(g.end(), f->hdx.begin(), f->hdx.end());
  g.insert(g.end(), f->hdy.begin(), f->hdy.end());
  g.insert(g.end(), f->hxc.begin(), f->hxc.end());
  g.insert(g.end(), f->hyc.begin(), f->hyc.end());
  cudaMemcpy(f->dgrid, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemsetAsync(f->c, 0, cells * f->NP * sizeof(double), momg_rt::stream());
  cudaMemsetAsync(f->p, 0, cells * 4 * sizeof(double), momg_rt::stream());
  return f;
}

void field_free(momg_field* f) {
  if (!f) return;
  cudaStreamSynchronize(momg_rt::stream());
  if (f->ev_free) {
    cudaEventSynchronize(f->ev_free);
    cudaEventDestroy(f->ev_free);
  }
  if (f->ev_ready) {
    cudaEventSynchronize(f->ev_ready);
    cudaEventDestroy(f->ev_ready);
  }
  cudaFree(f->c);
  cudaFree(f->p);
  cudaFree(f->dgrid);
  cudaFree(f->sweep_order);
  cudaFree(f->seg_plan);
  cudaFree(f->seg_plan32);
  cudaFree(f->sweep_ver);
  cudaFree(f->band_next);
  delete f;
}

}  // namespace momg_gpu

// ------------------------------------------------------------------ C ABI
#define ENSURE()                                         \
  do {                                                   \
    if (int rc_ = momg_rt::ensure(err)) return rc_;      \
  } while (0)
#define CLEAR_ERR()          \
  do {                       \
    if (err) {               \
      err->code = 0;         \
      err->i = err->j = -1;  \
      err->msg[0] = 0;       \
    }                        \
  } while (0)

// pending overlapped uploads of the fields an entry point touches
static void ACQ(const momg_field* a, const momg_field* b = nullptr, const momg_field* c = nullptr) {
  momg_rt::acquire(a);
  momg_rt::acquire(b);
  momg_rt::acquire(c);
}

static int arg_error(momg_err* err, const char* msg) {
  if (err) {
    err->code = MOMG_ERR_ARG;
    err->i = err->j = -1;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
  }
  return MOMG_ERR_ARG;
}

extern "C" {

int momg_init(int device, momg_err* err) {
  CLEAR_ERR();
  return momg_rt::init_device(device, err);
}
int momg_set_stream(void* s) {
  momg_rt::set_stream((cudaStream_t)s);
  return MOMG_OK;
}
void* momg_get_stream(void) { return (void*)momg_rt::stream(); }
void copy_streams_sync();
int momg_synchronize(momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  copy_streams_sync();
  return momg_rt::sync_check(err);
}
const char* momg_version(void) { return "momg_gpu 0.1 (sm_100a, FP64)"; }
int momg_supported_order(int M) { return momg_gpu::supported(M) ? 1 : 0; }
long long momg_launch_count(void) { return momg_rt::launches(); }
// Debug instrumentation of the split persistent sweep: per-item %globaltimer
// stamps (start, deps ready, faces done, update done) for the first `cap` items.
int momg_debug_trace(long long cap) {
  momg_gpu::set_trace(cap);
  return MOMG_OK;
}
long long momg_debug_trace_read(unsigned long long* host, long long n) {
  return momg_gpu::read_trace(host, n);
}
int momg_set_sweep_mode(int mode) {
  if (mode < 0 || mode > 2) return MOMG_ERR_ARG;
  momg_gpu::set_sweep_mode(mode == 0 ? 0 : 1);
  momg_gpu::set_band_mode(mode == 1 ? 1 : 0);
  return MOMG_OK;
}

int momg_set_band_kernel(int kind) {
  if (kind < 0 || kind > 1) return MOMG_ERR_ARG;
  momg_gpu::set_rb_mode(kind);
  return MOMG_OK;
}

int momg_field_create(const momg_grid* g, int M, momg_field** out, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  if (!g || !out || g->nx < 1 || g->ny < 1) return arg_error(err, "momg_field_create: bad grid");
  if (!momg_gpu::supported(M)) return arg_error(err, "momg_field_create: moment order not instantiated (3..8)");
  *out = momg_gpu::field_new(M, g->nx, g->ny, g->Lx, g->Ly, g->dx, g->dy, g->xc, g->yc, err);
  return *out ? MOMG_OK : MOMG_ERR_CUDA;
}
void momg_field_destroy(momg_field* f) { momg_gpu::field_free(f); }
int momg_field_shape(const momg_field* f, int* nx, int* ny, int* M, int* N, int* NP) {
  if (!f) return MOMG_ERR_ARG;
  if (nx) *nx = f->nx;
  if (ny) *ny = f->ny;
  if (M) *M = f->M;
  if (N) *N = f->N;
  if (NP) *NP = f->NP;
  return MOMG_OK;
}
int momg_field_device_ptrs(momg_field* f, double** c, double** p) {
  if (!f) return MOMG_ERR_ARG;
  if (c) *c = f->c;
  if (p) *p = f->p;
  return MOMG_OK;
}

static int upload(momg_field* f, const double* coeffs, const double* params, momg_err* err,
                  bool sync) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!f || !coeffs || !params) return arg_error(err, "momg_field_upload: null argument");
  const size_t cells = (size_t)f->nx * f->ny;
  // unpadded records (N % 4 == 0, e.g. M = 5): one linear copy (a pitched copy
  // of millions of short rows runs far below the PCIe rate)
  cudaError_t e = f->NP == f->N
                      ? cudaMemcpyAsync(f->c, coeffs, cells * f->N * sizeof(double), cudaMemcpyHostToDevice,
                                        momg_rt::stream())
                      : cudaMemcpy2DAsync(f->c, f->NP * sizeof(double), coeffs, f->N * sizeof(double),
                                          f->N * sizeof(double), cells, cudaMemcpyHostToDevice,
                                          momg_rt::stream());
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(f->p, params, cells * 4 * sizeof(double), cudaMemcpyHostToDevice,
                        momg_rt::stream());
  if (e == cudaSuccess && sync) e = cudaStreamSynchronize(momg_rt::stream());
  return momg_rt::cuda_check(e, err, "momg_field_upload");
}
static int download(const momg_field* f, double* coeffs, double* params, momg_err* err,
                    bool sync) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!f) return arg_error(err, "momg_field_download: null field");
  const size_t cells = (size_t)f->nx * f->ny;
  cudaError_t e = cudaSuccess;
  if (coeffs)
    e = f->NP == f->N ? cudaMemcpyAsync(coeffs, f->c, cells * f->N * sizeof(double), cudaMemcpyDeviceToHost,
                                        momg_rt::stream())
                      : cudaMemcpy2DAsync(coeffs, f->N * sizeof(double), f->c, f->NP * sizeof(double),
                                          f->N * sizeof(double), cells, cudaMemcpyDeviceToHost,
                                          momg_rt::stream());
  if (e == cudaSuccess && params)
    e = cudaMemcpyAsync(params, f->p, cells * 4 * sizeof(double), cudaMemcpyDeviceToHost,
                        momg_rt::stream());
  if (e == cudaSuccess && sync) e = cudaStreamSynchronize(momg_rt::stream());
  return momg_rt::cuda_check(e, err, "momg_field_download");
}
int momg_field_upload(momg_field* f, const double* c, const double* p, momg_err* err) {
  return upload(f, c, p, err, true);
}
int momg_field_download(const momg_field* f, double* c, double* p, momg_err* err) {
  return download(f, c, p, err, true);
}
int momg_field_upload_async(momg_field* f, const double* c, const double* p, momg_err* err) {
  return upload(f, c, p, err, false);
}
int momg_field_download_async(const momg_field* f, double* c, double* p, momg_err* err) {
  return download(f, c, p, err, false);
}
// ---- overlapped transfers (double-buffered streaming of solves)
static cudaStream_t g_h2d = nullptr, g_d2h = nullptr;
static bool copy_streams() {
  if (!g_h2d && cudaStreamCreateWithFlags(&g_h2d, cudaStreamNonBlocking) != cudaSuccess) return false;
  if (!g_d2h && cudaStreamCreateWithFlags(&g_d2h, cudaStreamNonBlocking) != cudaSuccess) return false;
  return true;
}
void copy_streams_sync() {
  if (g_h2d) cudaStreamSynchronize(g_h2d);
  if (g_d2h) cudaStreamSynchronize(g_d2h);
}
int momg_field_upload_overlapped(momg_field* f, const double* coeffs, const double* params, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  if (!f || !coeffs || !params) return arg_error(err, "momg_field_upload_overlapped: null argument");
  if (!copy_streams()) return momg_rt::cuda_check(cudaErrorUnknown, err, "momg_field_upload_overlapped");
  const size_t cells = (size_t)f->nx * f->ny;
  // the copy must follow (a) the field's previous overlapped download and
  // (b) everything already enqueued on the library stream (the zero-fill of
  // a fresh field, kernels that used it); (b) costs nothing when the
  // caller's compute calls have returned (they synchronise)
  cudaEvent_t ev_lib = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&ev_lib, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev_lib, momg_rt::stream());
  if (e == cudaSuccess) e = cudaStreamWaitEvent(g_h2d, ev_lib, 0);
  if (ev_lib) cudaEventDestroy(ev_lib);
  if (e == cudaSuccess && f->ev_free) e = cudaStreamWaitEvent(g_h2d, f->ev_free, 0);
  if (e == cudaSuccess)
    e = f->NP == f->N ? cudaMemcpyAsync(f->c, coeffs, cells * f->N * sizeof(double), cudaMemcpyHostToDevice, g_h2d)
                      : cudaMemcpy2DAsync(f->c, f->NP * sizeof(double), coeffs, f->N * sizeof(double),
                                          f->N * sizeof(double), cells, cudaMemcpyHostToDevice, g_h2d);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(f->p, params, cells * 4 * sizeof(double), cudaMemcpyHostToDevice, g_h2d);
  // deferred wait: the library stream waits for this copy only when an
  // entry point first uses the field (momg_rt::acquire), so the upload of the
  // next solve overlaps the compute of the current one
  if (e == cudaSuccess && !f->ev_ready) e = cudaEventCreateWithFlags(&f->ev_ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(f->ev_ready, g_h2d);
  if (e == cudaSuccess) f->ready_pending = true;
  return momg_rt::cuda_check(e, err, "momg_field_upload_overlapped");
}
int momg_field_download_overlapped(momg_field* f, double* coeffs, double* params, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!f || !coeffs || !params) return arg_error(err, "momg_field_download_overlapped: null argument");
  if (!copy_streams()) return momg_rt::cuda_check(cudaErrorUnknown, err, "momg_field_download_overlapped");
  const size_t cells = (size_t)f->nx * f->ny;
  cudaEvent_t ev = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, momg_rt::stream());
  if (e == cudaSuccess) e = cudaStreamWaitEvent(g_d2h, ev, 0);
  if (ev) cudaEventDestroy(ev);
  if (e == cudaSuccess)
    e = f->NP == f->N ? cudaMemcpyAsync(coeffs, f->c, cells * f->N * sizeof(double), cudaMemcpyDeviceToHost, g_d2h)
                      : cudaMemcpy2DAsync(coeffs, f->N * sizeof(double), f->c, f->NP * sizeof(double),
                                          f->N * sizeof(double), cells, cudaMemcpyDeviceToHost, g_d2h);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(params, f->p, cells * 4 * sizeof(double), cudaMemcpyDeviceToHost, g_d2h);
  if (e == cudaSuccess && !f->ev_free) e = cudaEventCreateWithFlags(&f->ev_free, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(f->ev_free, g_d2h);
  return momg_rt::cuda_check(e, err, "momg_field_download_overlapped");
}
int momg_copy_barrier(momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  cudaError_t e = cudaSuccess;
  for (cudaStream_t st : {g_h2d, g_d2h}) {
    if (!st || e != cudaSuccess) continue;
    cudaEvent_t ev = nullptr;
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(momg_rt::stream(), ev, 0);
    if (ev) cudaEventDestroy(ev);
  }
  return momg_rt::cuda_check(e, err, "momg_copy_barrier");
}
int momg_field_copy(momg_field* dst, const momg_field* src, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(dst, src);
  if (!dst || !src || dst->nx != src->nx || dst->ny != src->ny || dst->M != src->M)
    return arg_error(err, "momg_field_copy: shape mismatch");
  momg_gpu::op_copy(dst, src);
  return momg_rt::cuda_check(cudaGetLastError(), err, "momg_field_copy");
}
int momg_field_fill_maxwellian(momg_field* f, double rho, const double u[3], double theta,
                               momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!f) return arg_error(err, "momg_field_fill_maxwellian: null field");
  if (!(rho > 0.0) || !(theta > 0.0)) {
    if (err) {
      err->code = MOMG_NONPHYSICAL_STATE;
      std::snprintf(err->msg, sizeof(err->msg), "maxwellian_rep: rho and theta must be positive");
    }
    return MOMG_NONPHYSICAL_STATE;
  }
  momg_gpu::k_fill<<<592, 256, 0, momg_rt::stream()>>>(f->dev(), f->NP, rho, u[0], u[1], u[2],
                                                       theta);
  momg_rt::count_launch(1);
  return momg_rt::sync_check(err);
}

static bool same_shape(const momg_field* a, const momg_field* b) {
  return a && b && a->nx == b->nx && a->ny == b->ny && a->M == b->M;
}
static bool pair_shape(const momg_field* fine, const momg_field* coarse) {
  return fine && coarse && fine->M == coarse->M && fine->nx == 2 * coarse->nx &&
         fine->ny == 2 * coarse->ny;
}
static int config_error(momg_err* err, const char* msg) {
  if (err) {
    err->code = MOMG_CONFIG;
    err->i = err->j = -1;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
  }
  return MOMG_CONFIG;
}

int momg_residual(const momg_ctx* ctx, const momg_field* f, momg_field* out, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f, out);
  if (!ctx || !same_shape(f, out)) return arg_error(err, "momg_residual: shape mismatch");
  if (out == f) return arg_error(err, "momg_residual: out must not alias the field (residual returns a new vector)");
  if (!(ctx->knudsen > 0)) return config_error(err, "collision_frequency: Kn must be positive");
  momg_gpu::op_residual(momg_gpu::make_ctx(ctx), f, out);
  return momg_rt::sync_check(err);
}

int momg_fast_sweep(const momg_ctx* ctx, momg_field* f, const momg_field* rhs,
                    const int* sweep_order, long long* evals, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f, rhs);
  if (!ctx || !f || (rhs && !same_shape(f, rhs))) return arg_error(err, "momg_fast_sweep: shape mismatch");
  if (rhs == f) return arg_error(err, "momg_fast_sweep: rhs must not alias the field");
  if (!(ctx->knudsen > 0)) return config_error(err, "collision_frequency: Kn must be positive");
  static const int canon[4] = {0, 1, 2, 3};
  const int* order = sweep_order ? sweep_order : canon;
  momg_gpu::op_sweep(momg_gpu::make_ctx(ctx), f, rhs, order);
  const int rc = momg_rt::sync_check(err);
  if (rc == MOMG_OK && evals) *evals += 4LL * f->nx * f->ny;
  return rc;
}

int momg_fast_sweep_residual(const momg_ctx* ctx, momg_field* f, const int* sweep_order, momg_field* out,
                             long long* evals, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f, out);
  if (!ctx || !f || !out || !same_shape(f, out)) return arg_error(err, "momg_fast_sweep_residual: shape mismatch");
  if (out == f) return arg_error(err, "momg_fast_sweep_residual: out must not alias the field");
  if (!(ctx->knudsen > 0)) return config_error(err, "collision_frequency: Kn must be positive");
  static const int canon[4] = {0, 1, 2, 3};
  momg_gpu::op_sweep_residual(momg_gpu::make_ctx(ctx), f, sweep_order ? sweep_order : canon, out);
  const int rc = momg_rt::sync_check(err);
  if (rc == MOMG_OK && evals) *evals += 4LL * f->nx * f->ny;
  return rc;
}

int momg_total_mass(const momg_field* f, double* out, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!f) return arg_error(err, "momg_total_mass: null field");
  momg_gpu::op_mass(f, 1.0);
  return momg_gpu::fetch_scalar(out, err);
}

int momg_mass_correction(momg_field* f, double target, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!f) return arg_error(err, "momg_mass_correction: null field");
  double current = 0.0;
  momg_gpu::op_mass(f, target);
  if (int rc = momg_gpu::fetch_scalar(&current, err)) return rc;
  if (!(current > 0.0) || !std::isfinite(current)) {
    if (err) {
      err->code = MOMG_NONPHYSICAL_STATE;
      std::snprintf(err->msg, sizeof(err->msg), "mass_correction: nonpositive total mass %f",
                    current);
    }
    return MOMG_NONPHYSICAL_STATE;
  }
  momg_gpu::op_scale_by_factor(f);
  return momg_rt::sync_check(err);
}

int momg_restrict_solution(const momg_field* fine, momg_field* coarse, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(fine, coarse);
  if (!pair_shape(fine, coarse))
    return config_error(err, "restrict_solution: grids are not a 2x2 refinement pair");
  momg_gpu::op_restrict_sol(fine, coarse);
  return momg_rt::sync_check(err);
}

int momg_restrict_residual(const momg_field* arrays, const momg_field* coarse, momg_field* out,
                           momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(arrays, coarse, out);
  if (!pair_shape(arrays, coarse) || !same_shape(coarse, out))
    return config_error(err, "restrict_residual: grids are not a 2x2 refinement pair");
  momg_gpu::op_restrict_res(arrays, coarse, out);
  return momg_rt::sync_check(err);
}

int momg_fas_correct(momg_field* fine, const momg_field* before, const momg_field* after,
                     momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(fine, before, after);
  if (!pair_shape(fine, before) || !same_shape(before, after))
    return config_error(err, "fas_correct: grids are not a 2x2 refinement pair");
  momg_gpu::op_fas(fine, before, after);
  return momg_rt::sync_check(err);
}

int momg_residual_norm(const momg_field* res, const momg_field* field, double* out, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(res, field);
  if (!same_shape(res, field)) return arg_error(err, "momg_residual_norm: shape mismatch");
  momg_gpu::op_norm(res, field);
  return momg_gpu::fetch_scalar(out, err);
}

int momg_residual_scale(const momg_ctx* ctx, const momg_field* f, double* out, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!ctx || !f) return arg_error(err, "momg_residual_scale: null argument");
  momg_gpu::op_rscale(momg_gpu::make_ctx(ctx), f);
  return momg_gpu::fetch_scalar(out, err);
}

int momg_defect(const momg_field* res, const momg_field* rhs, momg_field* out, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(res, rhs, out);
  if (!same_shape(res, out) || (rhs && !same_shape(res, rhs)))
    return arg_error(err, "momg_defect: shape mismatch");
  momg_gpu::op_defect(res, rhs, out);
  return momg_rt::sync_check(err);
}

// mass_correction's rescale with a factor computed by the caller (a strip of
// a partitioned level: target / the level's total mass, single_level.cpp:176-183)
int momg_field_scale(momg_field* f, double factor, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(f);
  if (!f) return arg_error(err, "momg_field_scale: null field");
  const size_t n = (size_t)f->nx * f->ny * f->NP;
  momg_gpu::k_scale_by<<<592, 256, 0, momg_rt::stream()>>>(f->c, n, factor);
  momg_rt::count_launch(1);
  return momg_rt::sync_check(err);
}

int momg_axpy(momg_field* dst, const momg_field* src, momg_err* err) {
  CLEAR_ERR();
  ENSURE();
  ACQ(dst, src);
  if (!same_shape(dst, src)) return arg_error(err, "momg_axpy: shape mismatch");
  momg_gpu::op_axpy(dst, src);
  return momg_rt::sync_check(err);
}

}  // extern "C"
