// Strip-partitioned levels for multi-GPU (SURVEY.md
// §8(e)): the C ABI momg_strips_* of include/momg_gpu.h.
//
// A level of the global grid is split into n column strips [b[r], b[r+1])
// whose widths are multiples of the 32-column band (so every band task of
// every sweep direction lies in one strip, and 2x2 coarsening stays
// strip-local).  Each strip is an ordinary momg_field on its sub-grid plus a
// per-cell counter array, allocated by the process that owns it; a process
// attaches the strips of other ranks through CUDA IPC handles (peer memory
// over NVLink / NVSwitch).  One momg_strips_fast_sweep_residual launch runs
// the band tasks of this process's strips; tasks read the neighbouring
// strips' halo cells and poll their counters directly in peer memory (the
// single-field dataflow rule of the reference's exact Gauss-Seidel order,
// single_level.cpp:121-166, carried across the strip boundary), so the
// wavefront pipelines across ranks with no collective on the data path.
// Counters are never reset: each launch counts from the partition's epoch
// (advanced by 4 per FS iteration, identically on every rank).
//
// With every strip owned by one process, the same launch is the one-GPU
// emulation of all ranks as ONE kernel over all ranks' data (the GPU tests
// compare it bitwise with the single-field sweep).
#include <cstdio>
#include <cstring>
#include <vector>

#include "runtime.h"
#include "strips.h"

using momg_gpu::sp::kMaxStrips;
using momg_gpu::sp::StripTab;

struct momg_strips {
  int M = 0, n = 0, first = 0, last = -1, nx = 0, ny = 0;
  std::vector<int> b;
  std::vector<momg_field*> field, res;
  std::vector<unsigned*> ver;
  std::vector<int> present;
  std::vector<void*> opened;  // IPC mappings to close
  StripTab tab{};
  StripTab* dtab = nullptr;
  double* dgeo = nullptr;  // global dx | dy
  unsigned* next = nullptr;
  unsigned epoch = 0;
  bool dirty = true;
  bool remote = false;
};

namespace {
int fail(momg_err* err, int code, const char* msg) {
  if (err) {
    err->code = code;
    err->i = err->j = -1;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
  }
  return code;
}
constexpr int kIpcArrays = 5;  // coeffs, params, counters, residual coeffs, residual params
}  // namespace

extern "C" {

int momg_strips_create(const momg_grid* g, int M, int n, const int* bounds, int first, int last,
                       momg_strips** out, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!g || !bounds || !out || n < 1 || n > kMaxStrips || first < 0 || last < first || last >= n)
    return fail(err, MOMG_ERR_ARG, "momg_strips_create: bad arguments (1 <= n <= 8, 0 <= first <= last < n)");
  if (!momg_gpu::supported(M)) return fail(err, MOMG_CONFIG, "momg_strips_create: moment order not supported");
  if (g->nx % 32 || bounds[0] != 0 || bounds[n] != g->nx)
    return fail(err, MOMG_ERR_ARG, "momg_strips_create: nx must be a multiple of 32 and bounds span [0, nx]");
  for (int r = 0; r < n; ++r)
    if (bounds[r + 1] <= bounds[r] || (bounds[r + 1] - bounds[r]) % 32)
      return fail(err, MOMG_ERR_ARG, "momg_strips_create: strip widths must be positive multiples of 32");
  momg_strips* s = new momg_strips();
  s->M = M;
  s->n = n;
  s->first = first;
  s->last = last;
  s->nx = g->nx;
  s->ny = g->ny;
  s->b.assign(bounds, bounds + n + 1);
  s->field.assign(n, nullptr);
  s->res.assign(n, nullptr);
  s->ver.assign(n, nullptr);
  s->present.assign(n, 0);
  s->tab.n = n;
  for (int r = 0; r <= n; ++r) s->tab.i0[r] = bounds[r];
  int rc = MOMG_OK;
  for (int r = first; r <= last && rc == MOMG_OK; ++r) {
    const int i0 = bounds[r], w = bounds[r + 1] - i0;
    double Lx = 0.0;
    for (int i = i0; i < i0 + w; ++i) Lx += g->dx[i];
    for (momg_field** f : {&s->field[r], &s->res[r]}) {
      *f = momg_gpu::field_new(M, w, g->ny, Lx, g->Ly, g->dx + i0, g->dy, g->xc + i0, g->yc, err);
      if (!*f) rc = err ? err->code : MOMG_ERR_CUDA;
    }
    if (rc) break;
    const size_t cells = (size_t)w * g->ny;
    if (cudaMalloc(&s->ver[r], cells * sizeof(unsigned)) != cudaSuccess) {
      rc = fail(err, MOMG_ERR_CUDA, "momg_strips_create: counter allocation failed");
      break;
    }
    cudaMemsetAsync(s->ver[r], 0, cells * sizeof(unsigned), momg_rt::stream());
    s->tab.c[r] = s->field[r]->c;
    s->tab.p[r] = s->field[r]->p;
    s->tab.ver[r] = s->ver[r];
    s->tab.oc[r] = s->res[r]->c;
    s->tab.op[r] = s->res[r]->p;
    s->present[r] = 1;
  }
  if (rc == MOMG_OK) {
    std::vector<double> geo(g->dx, g->dx + g->nx);
    geo.insert(geo.end(), g->dy, g->dy + g->ny);
    if (cudaMalloc(&s->dgeo, geo.size() * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->dtab, sizeof(StripTab)) != cudaSuccess || cudaMalloc(&s->next, 64) != cudaSuccess)
      rc = fail(err, MOMG_ERR_CUDA, "momg_strips_create: allocation failed");
    else
      cudaMemcpy(s->dgeo, geo.data(), geo.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  if (rc == MOMG_OK) rc = momg_rt::sync_check(err);
  if (rc != MOMG_OK) {
    momg_strips_destroy(s);
    return rc;
  }
  *out = s;
  return MOMG_OK;
}

void momg_strips_destroy(momg_strips* s) {
  if (!s) return;
  cudaStreamSynchronize(momg_rt::stream());
  for (void* p : s->opened) cudaIpcCloseMemHandle(p);
  for (int r = 0; r < s->n; ++r) {
    momg_gpu::field_free(s->field[r]);
    momg_gpu::field_free(s->res[r]);
    cudaFree(s->ver[r]);
  }
  cudaFree(s->dtab);
  cudaFree(s->dgeo);
  cudaFree(s->next);
  delete s;
}

int momg_strips_field(momg_strips* s, int r, momg_field** field, momg_field** residual) {
  if (!s || r < 0 || r >= s->n || !s->field[r]) return MOMG_ERR_ARG;
  if (field) *field = s->field[r];
  if (residual) *residual = s->res[r];
  return MOMG_OK;
}

int momg_strips_export(momg_strips* s, int r, void* handle, momg_err* err) {
  if (err) err->code = 0;
  if (!s || !handle || r < 0 || r >= s->n || !s->field[r])
    return fail(err, MOMG_ERR_ARG, "momg_strips_export: not an owned strip");
  cudaIpcMemHandle_t h[kIpcArrays];
  void* ptrs[kIpcArrays] = {s->field[r]->c, s->field[r]->p, s->ver[r], s->res[r]->c, s->res[r]->p};
  for (int k = 0; k < kIpcArrays; ++k)
    if (int rc = momg_rt::cuda_check(cudaIpcGetMemHandle(&h[k], ptrs[k]), err, "momg_strips_export")) return rc;
  std::memcpy(handle, h, sizeof(h));
  return MOMG_OK;
}

int momg_strips_import(momg_strips* s, int r, const void* handle, momg_err* err) {
  if (err) err->code = 0;
  if (!s || !handle || r < 0 || r >= s->n || s->field[r])
    return fail(err, MOMG_ERR_ARG, "momg_strips_import: not a peer strip");
  cudaIpcMemHandle_t h[kIpcArrays];
  std::memcpy(h, handle, sizeof(h));
  void* p[kIpcArrays] = {};
  for (int k = 0; k < kIpcArrays; ++k) {
    if (int rc = momg_rt::cuda_check(cudaIpcOpenMemHandle(&p[k], h[k], cudaIpcMemLazyEnablePeerAccess), err,
                                     "momg_strips_import"))
      return rc;
    s->opened.push_back(p[k]);
  }
  s->tab.c[r] = (double*)p[0];
  s->tab.p[r] = (double*)p[1];
  s->tab.ver[r] = (unsigned*)p[2];
  s->tab.oc[r] = (double*)p[3];
  s->tab.op[r] = (double*)p[4];
  s->present[r] = 1;
  s->remote = true;
  s->dirty = true;
  return MOMG_OK;
}

int momg_strips_fast_sweep_residual(const momg_ctx* ctx, momg_strips* s, const int* sweep_order, long long* evals,
                                    momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!ctx || !s) return fail(err, MOMG_ERR_ARG, "momg_strips_fast_sweep_residual: null argument");
  if (ctx->M != s->M) return fail(err, MOMG_ERR_ARG, "momg_strips_fast_sweep_residual: moment order mismatch");
  if (!(ctx->knudsen > 0)) return fail(err, MOMG_CONFIG, "collision_frequency: Kn must be positive");
  // every strip a task may touch must be attached: the neighbours of the owned range
  const int lo = s->first > 0 ? s->first - 1 : 0, hi = s->last + 1 < s->n ? s->last + 1 : s->n - 1;
  for (int r = lo; r <= hi; ++r)
    if (!s->present[r]) return fail(err, MOMG_ERR_ARG, "momg_strips_fast_sweep_residual: neighbour strip not attached");
  for (int r = s->first; r <= s->last; ++r) momg_rt::acquire(s->field[r]);
  if (s->dirty) {
    cudaMemcpyAsync(s->dtab, &s->tab, sizeof(StripTab), cudaMemcpyHostToDevice, momg_rt::stream());
    s->dirty = false;
  }
  cudaMemsetAsync(s->next, 0, 64, momg_rt::stream());
  momg_gpu::StripLaunch L{};
  L.geo.nx = s->nx;
  L.geo.ny = s->ny;
  L.geo.dx = s->dgeo;
  L.geo.dy = s->dgeo + s->nx;
  L.tab = s->dtab;
  L.next = s->next;
  L.epoch = s->epoch;
  L.nbands = s->nx / 32;
  L.kb_up = s->b[s->first] / 32;
  L.kb_dn = (s->nx - s->b[s->last + 1]) / 32;
  L.nk = (s->b[s->last + 1] - s->b[s->first]) / 32;
  L.sys = s->remote ? 1 : 0;
  static const int canon[4] = {0, 1, 2, 3};
  for (int k = 0; k < 4; ++k) L.order[k] = (sweep_order ? sweep_order : canon)[k];
  s->epoch += 4;  // every rank advances identically, launched or not
  if (!momg_gpu::ops_for(s->M)->strips_sweep_res(momg_gpu::make_ctx(ctx), L))
    return fail(err, MOMG_CONFIG, "momg_strips_fast_sweep_residual: strips run first order, M <= 5, BGK / Shakhov");
  const int rc = momg_rt::sync_check(err);
  if (rc == MOMG_OK && evals) *evals += 4LL * (s->b[s->last + 1] - s->b[s->first]) * s->ny;
  return rc;
}

}  // extern "C"
