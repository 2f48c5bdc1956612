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
#include <algorithm>
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
  double* dgeo = nullptr;  // global dx | dy | xc | yc
  unsigned* next = nullptr;
  unsigned epoch = 0;
  bool dirty = true;
  bool remote = false;
  double Ly = 0.0;
  std::vector<double> hdx, hdy, hxc, hyc;    // global geometry (host)
  std::vector<momg_field*> ext, ext_res;     // owned strips + halo columns (residual)
  std::vector<int> ext_h;                    // their halo width (1 or 2: the stencil radius)
  int strip_of(int i) const {
    int r = 0;
    while (r + 1 < n && i >= b[r + 1]) ++r;
    return r;
  }
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
  s->ext.assign(n, nullptr);
  s->ext_res.assign(n, nullptr);
  s->ext_h.assign(n, 0);
  s->Ly = g->Ly;
  s->hdx.assign(g->dx, g->dx + g->nx);
  s->hdy.assign(g->dy, g->dy + g->ny);
  s->hxc.assign(g->xc, g->xc + g->nx);
  s->hyc.assign(g->yc, g->yc + g->ny);
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
    std::vector<double> geo(g->dx, g->dx + g->nx);  // dx | dy | xc | yc
    geo.insert(geo.end(), g->dy, g->dy + g->ny);
    geo.insert(geo.end(), g->xc, g->xc + g->nx);
    geo.insert(geo.end(), g->yc, g->yc + g->ny);
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
    momg_gpu::field_free(s->ext[r]);
    momg_gpu::field_free(s->ext_res[r]);
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

// one band launch over this process's strips: `iters` FS iterations, plus
// the residual tasks when with_res (first order)
static int strips_launch(const momg_ctx* ctx, momg_strips* s, const int* sweep_order, int iters, int with_res,
                         long long* evals, momg_err* err, const char* who) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!ctx || !s) return fail(err, MOMG_ERR_ARG, "momg_strips: null argument");
  if (ctx->M != s->M) return fail(err, MOMG_ERR_ARG, "momg_strips: moment order mismatch");
  if (!(ctx->knudsen > 0)) return fail(err, MOMG_CONFIG, "collision_frequency: Kn must be positive");
  if (iters < 1 || iters > 4) return fail(err, MOMG_ERR_ARG, "momg_strips: 1 <= iterations per launch <= 4");
  // every strip a task may touch must be attached: the neighbours of the owned range
  const int lo = s->first > 0 ? s->first - 1 : 0, hi = s->last + 1 < s->n ? s->last + 1 : s->n - 1;
  for (int r = lo; r <= hi; ++r)
    if (!s->present[r]) return fail(err, MOMG_ERR_ARG, "momg_strips: neighbour strip not attached");
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
  L.geo.xc = s->dgeo + s->nx + s->ny;
  L.geo.yc = s->dgeo + 2 * s->nx + s->ny;
  L.tab = s->dtab;
  L.next = s->next;
  L.epoch = s->epoch;
  L.nbands = s->nx / 32;
  L.kb_up = s->b[s->first] / 32;
  L.kb_dn = (s->nx - s->b[s->last + 1]) / 32;
  L.nk = (s->b[s->last + 1] - s->b[s->first]) / 32;
  L.sys = s->remote ? 1 : 0;
  L.iters = iters;
  L.with_res = with_res;
  static const int canon[4] = {0, 1, 2, 3};
  for (int k = 0; k < 4; ++k) L.order[k] = (sweep_order ? sweep_order : canon)[k];
  s->epoch += 4u * (unsigned)iters;  // every rank advances identically, launched or not
  if (!momg_gpu::ops_for(s->M)->strips_sweep(momg_gpu::make_ctx(ctx), L))
    return fail(err, MOMG_CONFIG, who);
  const int rc = momg_rt::sync_check(err);
  if (rc == MOMG_OK && evals) *evals += 4LL * iters * (s->b[s->last + 1] - s->b[s->first]) * s->ny;
  return rc;
}

// columns [i0, i1) of the level, from whichever strips hold them (own or
// peer memory), into dst at column x0 (dst: a field of width dnx); which =
// 0: the strips' fields, 1: their residual fields
static void copy_cols(const momg_strips* s, int which, int i0, int i1, momg_field* dst, int x0) {
  const int NP = dst->NP;
  for (int r = 0; r < s->n; ++r) {
    const int a = std::max(i0, s->b[r]), e = std::min(i1, s->b[r + 1]);
    if (a >= e) continue;
    const int w = s->b[r + 1] - s->b[r];
    const double* sc = which ? s->tab.oc[r] : s->tab.c[r];
    const double* sp = which ? s->tab.op[r] : s->tab.p[r];
    const int dx0 = x0 + (a - i0);
    cudaMemcpy2DAsync(dst->c + (size_t)dx0 * NP, (size_t)dst->nx * NP * sizeof(double), sc + (size_t)(a - s->b[r]) * NP,
                      (size_t)w * NP * sizeof(double), (size_t)(e - a) * NP * sizeof(double), s->ny, cudaMemcpyDefault,
                      momg_rt::stream());
    cudaMemcpy2DAsync(dst->p + (size_t)dx0 * 4, (size_t)dst->nx * 4 * sizeof(double), sp + (size_t)(a - s->b[r]) * 4,
                      (size_t)w * 4 * sizeof(double), (size_t)(e - a) * 4 * sizeof(double), s->ny, cudaMemcpyDefault,
                      momg_rt::stream());
  }
}

int momg_strips_fast_sweep_residual(const momg_ctx* ctx, momg_strips* s, const int* sweep_order, long long* evals,
                                    momg_err* err) {
  return strips_launch(ctx, s, sweep_order, 1, 1, evals, err,
                       "momg_strips_fast_sweep_residual: strips run first order, M <= 5, BGK / Shakhov");
}

int momg_strips_fast_sweep(const momg_ctx* ctx, momg_strips* s, const int* sweep_order, int iters, long long* evals,
                           momg_err* err) {
  return strips_launch(ctx, s, sweep_order, iters, 0, evals, err,
                       "momg_strips_fast_sweep: strips run M <= 5, BGK / Shakhov");
}

int momg_strips_residual(const momg_ctx* ctx, momg_strips* s, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!ctx || !s || ctx->M != s->M) return fail(err, MOMG_ERR_ARG, "momg_strips_residual: bad arguments");
  const int h = ctx->space_order == 2 ? 2 : 1;  // stencil radius (spatial.cpp:34-50, 98-124)
  const momg_gpu::DevCtx dctx = momg_gpu::make_ctx(ctx);
  for (int r = s->first; r <= s->last; ++r) {
    const int lo = std::max(0, s->b[r] - h), hi = std::min(s->nx, s->b[r + 1] + h);
    for (int q = lo; q < hi; ++q)
      if (!s->present[s->strip_of(q)]) return fail(err, MOMG_ERR_ARG, "momg_strips_residual: neighbour strip not attached");
    momg_rt::acquire(s->field[r]);
    if (s->ext[r] && s->ext_h[r] != h) {  // the other spatial order: other halo width
      momg_gpu::field_free(s->ext[r]);
      momg_gpu::field_free(s->ext_res[r]);
      s->ext[r] = s->ext_res[r] = nullptr;
    }
    if (!s->ext[r]) {
      s->ext_h[r] = h;
      // the strip plus its neighbours' h columns: the residual of the strip's
      // own cells on this field is the level's (their stencils lie inside it)
      const int w = hi - lo;
      std::vector<double> dx(s->hdx.begin() + lo, s->hdx.begin() + hi), xc(s->hxc.begin() + lo, s->hxc.begin() + hi);
      double Lx = 0.0;
      for (double v : dx) Lx += v;
      for (momg_field** f : {&s->ext[r], &s->ext_res[r]}) {
        *f = momg_gpu::field_new(s->M, w, s->ny, Lx, s->Ly, dx.data(), s->hdy.data(), xc.data(), s->hyc.data(), err);
        if (!*f) return err ? err->code : MOMG_ERR_CUDA;
      }
    }
    copy_cols(s, 0, lo, hi, s->ext[r], 0);
    momg_gpu::op_residual(dctx, s->ext[r], s->ext_res[r]);
    // the strip's own columns of the residual
    const int NP = s->ext_res[r]->NP, w = s->b[r + 1] - s->b[r], off = s->b[r] - lo, W = hi - lo;
    cudaMemcpy2DAsync(s->res[r]->c, (size_t)w * NP * sizeof(double), s->ext_res[r]->c + (size_t)off * NP,
                      (size_t)W * NP * sizeof(double), (size_t)w * NP * sizeof(double), s->ny, cudaMemcpyDeviceToDevice,
                      momg_rt::stream());
    cudaMemcpy2DAsync(s->res[r]->p, (size_t)w * 4 * sizeof(double), s->ext_res[r]->p + (size_t)off * 4,
                      (size_t)W * 4 * sizeof(double), (size_t)w * 4 * sizeof(double), s->ny, cudaMemcpyDeviceToDevice,
                      momg_rt::stream());
  }
  return momg_rt::sync_check(err);
}

int momg_strips_gather(momg_strips* s, int which, momg_field* full, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!s || !full || full->nx != s->nx || full->ny != s->ny || full->M != s->M)
    return fail(err, MOMG_ERR_ARG, "momg_strips_gather: the full field must have the level's shape");
  for (int r = 0; r < s->n; ++r)
    if (!s->present[r]) return fail(err, MOMG_ERR_ARG, "momg_strips_gather: strip not attached");
  for (int r = s->first; r <= s->last; ++r) momg_rt::acquire(which ? s->res[r] : s->field[r]);
  momg_rt::acquire(full);
  copy_cols(s, which, 0, s->nx, full, 0);
  return momg_rt::sync_check(err);
}

int momg_strips_scatter(momg_strips* s, int which, const momg_field* full, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!s || !full || full->nx != s->nx || full->ny != s->ny || full->M != s->M)
    return fail(err, MOMG_ERR_ARG, "momg_strips_scatter: the full field must have the level's shape");
  momg_rt::acquire(full);
  for (int r = s->first; r <= s->last; ++r) {
    momg_field* dst = which ? s->res[r] : s->field[r];
    momg_rt::acquire(dst);
    const int NP = dst->NP, w = s->b[r + 1] - s->b[r];
    cudaMemcpy2DAsync(dst->c, (size_t)w * NP * sizeof(double), full->c + (size_t)s->b[r] * NP,
                      (size_t)s->nx * NP * sizeof(double), (size_t)w * NP * sizeof(double), s->ny,
                      cudaMemcpyDeviceToDevice, momg_rt::stream());
    cudaMemcpy2DAsync(dst->p, (size_t)w * 4 * sizeof(double), full->p + (size_t)s->b[r] * 4,
                      (size_t)s->nx * 4 * sizeof(double), (size_t)w * 4 * sizeof(double), s->ny,
                      cudaMemcpyDeviceToDevice, momg_rt::stream());
  }
  return momg_rt::sync_check(err);
}

}  // extern "C"
