// Host-side NMG driver (kept host C++, as the reference's): GridHierarchy,
// nmg_cycle, solve_steady (multigrid.cpp:12-65, 166-200, 243-320).  Every
// per-cell loop of the reference becomes a stream-ordered device op
// (runtime.h); the host only sees scalars (norms, mass) and error records.
// Data stays device-resident for the whole solve; per-level work buffers are
// allocated once per solve instead of per cycle.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <memory>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "runtime.h"

namespace momg_host {

// Errors inside the driver travel as this exception and are mapped back to
// momg_err at the C boundary (the reference's exception types, types.hpp).
struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

static void check(int rc, const momg_err& e) {
  if (rc != MOMG_OK) throw Fail(rc, e.msg);
}

struct Grid {
  int nx, ny;
  double Lx, Ly;
  std::vector<double> dx, dy, xc, yc;
};

static Grid grid_of(const momg_field* f) {
  return Grid{f->nx, f->ny, f->Lx, f->Ly, f->hdx, f->hdy, f->hxc, f->hyc};
}

// coarsen, multigrid.cpp:12-35
static Grid coarsen(const Grid& fine) {
  Grid g;
  g.nx = fine.nx / 2;
  g.ny = fine.ny / 2;
  g.Lx = fine.Lx;
  g.Ly = fine.Ly;
  g.dx.resize(g.nx);
  g.dy.resize(g.ny);
  g.xc.resize(g.nx);
  g.yc.resize(g.ny);
  double x = 0.0;
  for (int i = 0; i < g.nx; ++i) {
    g.dx[i] = fine.dx[2 * i] + fine.dx[2 * i + 1];
    g.xc[i] = x + 0.5 * g.dx[i];
    x += g.dx[i];
  }
  double y = 0.0;
  for (int j = 0; j < g.ny; ++j) {
    g.dy[j] = fine.dy[2 * j] + fine.dy[2 * j + 1];
    g.yc[j] = y + 0.5 * g.dy[j];
    y += g.dy[j];
  }
  return g;
}

static bool can_coarsen(const Grid& g) {  // multigrid.cpp:37-40, min_coarse_cells = 8
  return g.nx % 2 == 0 && g.ny % 2 == 0 && g.nx / 2 >= 8 && g.ny / 2 >= 8;
}

// GridHierarchy::build, multigrid.cpp:44-65 (coarsest first)
static std::vector<Grid> build_hierarchy(const Grid& finest, int levels) {
  if (levels < 0) throw Fail(MOMG_CONFIG, "hierarchy: level count must be positive");
  std::vector<Grid> grids{finest};
  if (levels == 0) {
    while (can_coarsen(grids.front())) grids.insert(grids.begin(), coarsen(grids.front()));
    return grids;
  }
  for (int k = 1; k < levels; ++k) {
    const Grid& top = grids.front();
    if (top.nx % 2 != 0 || top.ny % 2 != 0)
      throw Fail(MOMG_CONFIG, "hierarchy: " + std::to_string(levels) +
                                  " levels need cell counts divisible by 2 at each split");
    if (!can_coarsen(top))
      throw Fail(MOMG_CONFIG, "hierarchy: " + std::to_string(levels) +
                                  " levels would make the coarsest grid smaller than 8 cells");
    grids.insert(grids.begin(), coarsen(top));
  }
  return grids;
}

struct FieldPtr {
  momg_field* f = nullptr;
  FieldPtr() = default;
  explicit FieldPtr(momg_field* p) : f(p) {}
  FieldPtr(const FieldPtr&) = delete;
  FieldPtr& operator=(const FieldPtr&) = delete;
  FieldPtr(FieldPtr&& o) noexcept : f(o.f) { o.f = nullptr; }
  FieldPtr& operator=(FieldPtr&& o) noexcept {
    std::swap(f, o.f);
    return *this;
  }
  ~FieldPtr() { momg_gpu::field_free(f); }
};

static FieldPtr make_field(const Grid& g, int M) {
  momg_err e{};
  momg_field* f = momg_gpu::field_new(M, g.nx, g.ny, g.Lx, g.Ly, g.dx.data(), g.dy.data(),
                                      g.xc.data(), g.yc.data(), &e);
  if (!f) throw Fail(e.code ? e.code : MOMG_ERR_CUDA, e.msg);
  return FieldPtr(f);
}

// Per-level work buffers of nmg_cycle (multigrid.cpp:176-193), allocated once.
struct LevelWork {
  FieldPtr res, defect;                        // fine-size (this level)
  FieldPtr coarse, before, crhs, cres;         // coarse-size (level - 1)
};

struct Hierarchy {
  std::vector<Grid> grids;        // coarsest first
  std::vector<LevelWork> work;    // indexed by level
};

static Hierarchy prepare(const momg_field* finest, int levels) {
  Hierarchy h;
  h.grids = build_hierarchy(grid_of(finest), levels);
  h.work.resize(h.grids.size());
  for (size_t l = 1; l < h.grids.size(); ++l) {
    LevelWork& w = h.work[l];
    w.res = make_field(h.grids[l], finest->M);
    w.defect = make_field(h.grids[l], finest->M);
    w.coarse = make_field(h.grids[l - 1], finest->M);
    w.before = make_field(h.grids[l - 1], finest->M);
    w.crhs = make_field(h.grids[l - 1], finest->M);
    w.cres = make_field(h.grids[l - 1], finest->M);
  }
  return h;
}

struct Cycle {
  int s1 = 2, s2 = 2, s3 = 4, gamma = 1;
};

static const int kCanon[4] = {0, 1, 2, 3};

static void sweeps(const momg_gpu::DevCtx& ctx, momg_field* field, const momg_field* rhs, int n) {
  while (n > 0) {
    const int k = n < 4 ? n : 4;
    momg_gpu::op_sweep_n(ctx, field, rhs, kCanon, k);
    n -= k;
  }
}

// nmg_cycle, multigrid.cpp:166-200 (Alg. 2 of the paper).  Device errors are
// recorded and every later kernel early-exits, so the check is deferred to
// the caller (solve_steady checks once per outer iteration).
static void nmg_cycle(Hierarchy& h, int level, momg_field* field, const momg_field* rhs,
                      const momg_gpu::DevCtx& ctx, const Cycle& pol, long long* work) {
  const long long cells = (long long)field->nx * field->ny;
  // consecutive fast_sweep_step calls run as one overlapped launch (same
  // results: the per-cell dependency rule is exact across iterations)
  if (level == 0) {
    sweeps(ctx, field, rhs, pol.s3);
    *work += 4 * cells * pol.s3;
    return;
  }
  LevelWork& w = h.work[level];
  if (!rhs && pol.s1 > 0) {
    // finest level: the last pre-smoothing launch and the residual as one
    // band launch (identical results; op_sweep_residual falls back)
    sweeps(ctx, field, nullptr, pol.s1 - 1 - (pol.s1 - 1) % 4);
    momg_gpu::op_sweep_residual(ctx, field, kCanon, w.res.f, (pol.s1 - 1) % 4 + 1);
  } else {
    sweeps(ctx, field, rhs, pol.s1);
    momg_gpu::op_residual(ctx, field, w.res.f);
  }
  *work += 4 * cells * pol.s1;
  momg_gpu::op_defect(w.res.f, rhs, w.defect.f);
  momg_gpu::op_restrict_sol(field, w.coarse.f);
  momg_gpu::op_copy(w.before.f, w.coarse.f);
  momg_gpu::op_restrict_res(w.defect.f, w.coarse.f, w.crhs.f);
  momg_gpu::op_residual(ctx, w.coarse.f, w.cres.f);
  momg_gpu::op_axpy(w.crhs.f, w.cres.f);
  for (int g = 0; g < pol.gamma; ++g) nmg_cycle(h, level - 1, w.coarse.f, w.crhs.f, ctx, pol, work);
  momg_gpu::op_fas(field, w.before.f, w.coarse.f);
  sweeps(ctx, field, rhs, pol.s2);
  *work += 4 * cells * pol.s2;
}

// A solve iteration captured as a CUDA graph (first replay() captures it).
// Capture needs a non-default stream; if the stream cannot be captured the
// iteration simply runs eagerly (same kernels, same results).
static long long g_graph_replays = 0;
struct IterGraph {
  cudaGraphExec_t exec = nullptr;
  long long nodes = 0;
  bool failed = false;
  ~IterGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
  // 0: not run (the caller runs body eagerly), 1: captured and launched
  // (body's host-side effects happened once), 2: replayed
  template <class F>
  int replay(F&& body, cudaStream_t st) {
    if (failed || st == nullptr) return 0;
    if (!exec) {
      cudaGraph_t g = nullptr;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        failed = true;
        cudaGetLastError();
        return 0;
      }
      const long long l0 = momg_rt::launches();
      try {
        body();
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      const cudaError_t ec = cudaStreamEndCapture(st, &g);
      nodes = momg_rt::launches() - l0;
      momg_rt::count_launch(-nodes);  // counted per replay below
      if (ec != cudaSuccess || !g || cudaGraphInstantiate(&exec, g, 0) != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        exec = nullptr;
        failed = true;
        cudaGetLastError();
        return 0;
      }
      cudaGraphDestroy(g);
      momg_rt::note_launch(cudaGraphLaunch(exec, st));
      momg_rt::count_launch(nodes);
      return 1;
    }
    momg_rt::note_launch(cudaGraphLaunch(exec, st));
    momg_rt::count_launch(nodes);
    ++g_graph_replays;
    return 2;
  }
};

static double scalar(momg_err& e) {
  double v = 0.0;
  check(momg_gpu::fetch_scalar(&v, &e), e);
  return v;
}

}  // namespace momg_host

using namespace momg_host;

static int map_fail(const Fail& f, momg_err* err) {
  if (err) {
    err->code = f.code;
    err->i = err->j = -1;
    std::snprintf(err->msg, sizeof(err->msg), "%s", f.what());
  }
  return f.code;
}

extern "C" {

long long momg_graph_replays(void) { return g_graph_replays; }

int momg_nmg_cycle(const momg_ctx* ctx, momg_field* field, int levels, int s1, int s2, int s3,
                   int gamma, long long* work, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!ctx || !field) {
    if (err) err->code = MOMG_ERR_ARG;
    return MOMG_ERR_ARG;
  }
  momg_rt::acquire(field);
  try {
    Hierarchy h = prepare(field, levels);
    Cycle pol{s1, s2, s3, gamma};
    long long w = 0;
    nmg_cycle(h, (int)h.grids.size() - 1, field, nullptr, momg_gpu::make_ctx(ctx), pol, &w);
    momg_err e{};
    check(momg_rt::sync_check(&e), e);
    if (work) *work = w;
    return MOMG_OK;
  } catch (const Fail& f) {
    return map_fail(f, err);
  }
}

// nmg_cycle with a right-hand side (the coarse problem of an outer cycle run
// elsewhere, e.g. the strip-partitioned finest level of strips.py)
int momg_nmg_cycle_rhs(const momg_ctx* ctx, momg_field* field, const momg_field* rhs, int levels, int s1, int s2,
                       int s3, int gamma, long long* work, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!ctx || !field || (rhs && (rhs->nx != field->nx || rhs->ny != field->ny || rhs->M != field->M))) {
    if (err) err->code = MOMG_ERR_ARG;
    return MOMG_ERR_ARG;
  }
  momg_rt::acquire(field);
  momg_rt::acquire(rhs);
  try {
    Hierarchy h = prepare(field, levels);
    Cycle pol{s1, s2, s3, gamma};
    long long w = 0;
    nmg_cycle(h, (int)h.grids.size() - 1, field, rhs, momg_gpu::make_ctx(ctx), pol, &w);
    momg_err e{};
    check(momg_rt::sync_check(&e), e);
    if (work) *work = w;
    return MOMG_OK;
  } catch (const Fail& f) {
    return map_fail(f, err);
  }
}

// solve_steady, multigrid.cpp:243-320
int momg_solve_steady(const momg_ctx* ctx, momg_field* field, const momg_solver_opts* opts,
                      momg_report* report, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!ctx || !field || !opts) {
    if (err) err->code = MOMG_ERR_ARG;
    return MOMG_ERR_ARG;
  }
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  momg_report local{};
  momg_report& rep = report ? *report : local;
  rep.converged = 0;
  rep.iterations = 0;
  rep.r0_norm = rep.final_norm = rep.final_ratio = 0.0;
  rep.work = 0;
  rep.seconds = 0.0;
  rep.history_len = 0;
  const int cap = opts->max_iterations > 0 ? opts->max_iterations : (opts->kind == 2 ? 200 : 100000);
  const momg_gpu::DevCtx dctx = momg_gpu::make_ctx(ctx);
  long long work = 0;
  momg_rt::acquire(field);
  try {
    if (!(ctx->knudsen > 0)) throw Fail(MOMG_CONFIG, "collision_frequency: Kn must be positive");
    momg_err e{};
    FieldPtr res = make_field(grid_of(field), field->M);
    momg_gpu::op_residual(dctx, field, res.f);
    momg_gpu::op_norm(res.f, field);
    rep.r0_norm = scalar(e);
    momg_gpu::op_rscale(dctx, field);
    const double scale = scalar(e);
    if (rep.r0_norm <= 1e-12 * scale) {
      rep.converged = 1;
      rep.final_norm = rep.r0_norm;
      rep.final_ratio = 0.0;
      rep.seconds = elapsed();
      return MOMG_OK;
    }
    Hierarchy h;
    if (opts->kind == 2) h = prepare(field, opts->levels);
    momg_gpu::op_mass(field, 1.0);
    const double target = scalar(e);
    Cycle pol{opts->s1, opts->s2, opts->s3, opts->gamma};
    // One iteration of the solve loop (multigrid.cpp:272-283): the smoother /
    // cycle, mass_correction (its positivity check on the device), the
    // residual and its norm -- all stream-ordered, one host read at the end.
    // After the first (eager) iteration, which initialises every lazily
    // allocated buffer and kernel attribute, the iteration is captured once
    // as a CUDA graph and replayed: one launch per iteration instead of one
    // per kernel.
    long long iter_work = 0;
    auto body = [&]() {
      long long w0 = work;
      if (opts->kind == 0) {
        // euler_step(field, res, {}, ctx) with res = R(field) of the previous iteration
        momg_gpu::op_global_dt(dctx, field);
        momg_gpu::op_euler(field, res.f, nullptr);
      } else if (opts->kind == 1) {
        momg_gpu::op_sweep(dctx, field, nullptr, kCanon);
        work += 4LL * field->nx * field->ny;
      } else {
        nmg_cycle(h, (int)h.grids.size() - 1, field, nullptr, dctx, pol, &work);
      }
      // mass_correction (single_level.cpp:176-183)
      momg_gpu::op_mass(field, target);
      momg_gpu::op_mass_guard();
      momg_gpu::op_scale_by_factor(field);
      momg_gpu::op_residual(dctx, field, res.f);
      momg_gpu::op_norm(res.f, field);
      iter_work = work - w0;
    };
    IterGraph graph;
    for (int n = 1; n <= cap; ++n) {
      int step_rc = MOMG_OK;
      std::string step_msg;
      try {
        const long long w_before = work;
        const int how = n == 1 ? 0 : graph.replay(body, momg_rt::stream());
        if (how == 0) {
          work = w_before;  // (a failed capture ran body's host side only)
          body();
        } else if (how == 2) {
          work += iter_work;
        }
        rep.final_norm = scalar(e);
      } catch (const Fail& f) {
        step_rc = f.code;
        step_msg = f.what();
      }
      if (step_rc == MOMG_SOLVER_ERROR || step_rc == MOMG_NONPHYSICAL_STATE) {
        rep.work = work;
        rep.seconds = elapsed();
        throw Fail(MOMG_NONCONVERGENCE,
                   std::string(step_rc == MOMG_SOLVER_ERROR ? "iteration step failed: "
                                                            : "iteration left the field nonphysical: ") +
                       step_msg);
      }
      if (step_rc != MOMG_OK) throw Fail(step_rc, step_msg);
      rep.iterations = n;
      rep.final_ratio = rep.final_norm / rep.r0_norm;
      if (rep.history && rep.history_len < rep.history_cap) rep.history[rep.history_len] = rep.final_ratio;
      if (rep.history_seconds && rep.history_len < rep.history_cap) rep.history_seconds[rep.history_len] = elapsed();
      rep.history_len++;
      rep.work = work;
      rep.seconds = elapsed();
      if (!std::isfinite(rep.final_ratio) || rep.final_ratio > 1e6)
        throw Fail(MOMG_NONCONVERGENCE, "residual diverged: ratio " +
                                            std::to_string(rep.final_ratio) + " at iteration " +
                                            std::to_string(n));
      if (rep.final_ratio <= opts->tol) {
        rep.converged = 1;
        return MOMG_OK;
      }
    }
    throw Fail(MOMG_NONCONVERGENCE, "iteration cap " + std::to_string(cap) + " reached at ratio " +
                                        std::to_string(rep.final_ratio));
  } catch (const Fail& f) {
    rep.work = work;
    rep.seconds = elapsed();
    return map_fail(f, err);
  }
}

// euler_step (single_level.cpp:74-97): global_dt reduction, then the
// per-cell forward-Euler update with the dt/2 retry; residuals nullable
// (R(field) is evaluated first, as solve_steady passes it)
int momg_euler_step(const momg_ctx* ctx, momg_field* field, const momg_field* residuals,
                    const momg_field* rhs, momg_err* err) {
  if (err) err->code = 0;
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!ctx || !field || (residuals && (residuals->nx != field->nx || residuals->ny != field->ny ||
                                        residuals->M != field->M)) ||
      (rhs && (rhs->nx != field->nx || rhs->ny != field->ny || rhs->M != field->M)) || residuals == field ||
      rhs == field) {
    if (err) {
      err->code = MOMG_ERR_ARG;
      std::snprintf(err->msg, sizeof(err->msg), "momg_euler_step: shape mismatch or aliased arguments");
    }
    return MOMG_ERR_ARG;
  }
  momg_rt::acquire(field);
  momg_rt::acquire(residuals);
  momg_rt::acquire(rhs);
  try {
    if (!(ctx->knudsen > 0)) throw Fail(MOMG_CONFIG, "collision_frequency: Kn must be positive");
    const momg_gpu::DevCtx dctx = momg_gpu::make_ctx(ctx);
    FieldPtr own;
    if (!residuals) {
      own = make_field(grid_of(field), field->M);
      momg_gpu::op_residual(dctx, field, own.f);
      residuals = own.f;
    }
    momg_gpu::op_global_dt(dctx, field);
    momg_gpu::op_euler(field, residuals, rhs);
    momg_err e{};
    check(momg_rt::sync_check(&e), e);
    return MOMG_OK;
  } catch (const Fail& f) {
    return map_fail(f, err);
  }
}

double momg_max_hermite_root(int degree) {
  // Largest zero of He_degree (tables.cpp:22-41): Newton from the upper bound
  // 2 sqrt(degree) + 1 (monotone from above), polished to a fixed point.
  if (degree < 1) return NAN;
  if (degree == 1) return 0.0;
  double x = 2.0 * std::sqrt((double)degree) + 1.0;
  for (int it = 0; it < 200; ++it) {
    double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0;
    for (int k = 1; k < degree; ++k) {
      const double p2 = x * p1 - k * p0;
      const double d2 = p1 + x * d1 - k * d0;
      p0 = p1;
      p1 = p2;
      d0 = d1;
      d1 = d2;
    }
    const double nx = x - p1 / d1;
    if (nx == x || std::fabs(nx - x) <= 1e-16 * std::fabs(x)) {
      x = nx;
      break;
    }
    x = nx;
  }
  return x;
}

}  // extern "C"
