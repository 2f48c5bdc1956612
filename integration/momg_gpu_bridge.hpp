// Drop-in bridge for the reference's own C++ (namespace momg, /root/reference/proj):
// the same signatures as the reference functions, executed on the B200 through
// the C ABI of include/momg_gpu.h.  Two ways to switch the reference's hot path:
//
//  (1) call momg::gpu::X where the reference calls momg::X (this header), or
//  (2) link / preload integration/momg_gpu_interpose.cpp (built into
//      integration/_build/libmomg_gpu_interpose.so): it DEFINES momg::X with
//      the reference's own signatures, so the reference's unmodified
//      multigrid.cpp (nmg_cycle, solve_steady) resolves its calls to the GPU
//      (ELF symbol interposition).
//
//   momg::gpu::residual           <- spatial.hpp:52-56 (both signatures)
//   momg::gpu::fast_sweep_step    <- single_level.hpp:63-65
//   momg::gpu::euler_step         <- single_level.hpp:52-53
//   momg::gpu::total_mass         <- single_level.hpp:68
//   momg::gpu::mass_correction    <- single_level.hpp:73
//   momg::gpu::restrict_solution  <- multigrid.hpp:41
//   momg::gpu::restrict_residual  <- multigrid.hpp:45-47
//   momg::gpu::fas_correct        <- multigrid.hpp:52-53
//   momg::gpu::nmg_cycle          <- multigrid.hpp:58-60 (device-resident V-cycle)
//   momg::gpu::residual_norm      <- multigrid.hpp:67-68
//   momg::gpu::solve_steady       <- multigrid.hpp:114-116 (whole solve device-resident)
//   momg::gpu::DeviceCellField    <- CellField (grid.hpp:54-85) kept in HBM: the
//                                    per-call functions have overloads on it, so
//                                    a caller that owns its levels keeps them on
//                                    the device between calls
//
// The CellField overloads upload / download the field per call (the
// reference keeps host AoS fields); nmg_cycle / solve_steady and every
// DeviceCellField overload keep the data in HBM.  Errors are rethrown as the
// reference's exception types (types.hpp:20-57, NonConvergence
// multigrid.hpp:89-97).
#pragma once

#include <array>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "momg/multigrid.hpp"
#include "momg_gpu.h"

namespace momg {
namespace gpu {

[[noreturn]] inline void rethrow(int rc, const momg_err& e, const SolveReport* report = nullptr) {
  const std::string what = e.msg;
  switch (rc) {
    case MOMG_NONPHYSICAL_STATE: throw NonphysicalState(what);
    case MOMG_SOLVER_ERROR: throw SolverError(what);
    case MOMG_NON_SPD: throw NonSpdTensor(what, 0.0);
    case MOMG_CONFIG: throw ConfigError(what);
    case MOMG_NONCONVERGENCE: throw NonConvergence(what, report ? *report : SolveReport{});
    default: throw Error("momg_gpu: " + what);
  }
}

inline void check(int rc, const momg_err& e) {
  if (rc != MOMG_OK) rethrow(rc, e);
}

inline momg_ctx context(const SolveContext& c, int M) {
  momg_ctx x{};
  x.M = M;
  x.space_order = c.scheme.order;
  x.c_bound = c.scheme.c_bound;
  x.cfl = c.cfl.cfl;
  x.cfl_c_bound = c.cfl.c_bound;
  x.collision = c.model.kind == CollisionKind::bgk ? MOMG_BGK
                : c.model.kind == CollisionKind::shakhov ? MOMG_SHAKHOV : MOMG_ES_BGK;
  x.prandtl = c.model.prandtl;
  x.knudsen = c.gas.knudsen;
  x.viscosity_index = c.gas.viscosity_index;
  const WallSpec* w[4] = {&c.walls.left, &c.walls.right, &c.walls.bottom, &c.walls.top};
  for (int k = 0; k < 4; ++k) {
    x.wall_speed[k] = w[k]->speed;
    x.wall_theta[k] = w[k]->theta;
  }
  x.threads = c.threads;
  return x;
}

struct FieldDeleter {
  void operator()(momg_field* f) const { momg_field_destroy(f); }
};
using DeviceField = std::unique_ptr<momg_field, FieldDeleter>;

// CellField (grid.hpp:54-76) -> device level
inline DeviceField upload(const CellField& f) {
  const Grid2D& g = f.grid();
  momg_grid mg{g.nx, g.ny, g.Lx, g.Ly, g.dx.data(), g.dy.data(), g.xc.data(), g.yc.data()};
  momg_err e{};
  momg_field* h = nullptr;
  check(momg_field_create(&mg, f.order(), &h, &e), e);
  DeviceField d(h);
  const int n = IndexSet::count(f.order());
  std::vector<double> c((size_t)f.size() * n), p((size_t)f.size() * 4);
  for (int k = 0; k < f.size(); ++k) {
    for (int q = 0; q < n; ++q) c[(size_t)k * n + q] = f[k].coeffs[q];
    for (int q = 0; q < 3; ++q) p[(size_t)k * 4 + q] = f[k].params.mean[q];
    p[(size_t)k * 4 + 3] = f[k].params.spread;
  }
  check(momg_field_upload(d.get(), c.data(), p.data(), &e), e);
  return d;
}

inline void download(momg_field* d, CellField& f) {
  const int n = IndexSet::count(f.order());
  std::vector<double> c((size_t)f.size() * n), p((size_t)f.size() * 4);
  momg_err e{};
  check(momg_field_download(d, c.data(), p.data(), &e), e);
  for (int k = 0; k < f.size(); ++k) {
    for (int q = 0; q < n; ++q) f[k].coeffs[q] = c[(size_t)k * n + q];
    for (int q = 0; q < 3; ++q) f[k].params.mean[q] = p[(size_t)k * 4 + q];
    f[k].params.spread = p[(size_t)k * 4 + 3];
  }
}

inline DeviceField empty_like(const Grid2D& g, int order) {
  momg_grid mg{g.nx, g.ny, g.Lx, g.Ly, g.dx.data(), g.dy.data(), g.xc.data(), g.yc.data()};
  momg_err e{};
  momg_field* h = nullptr;
  check(momg_field_create(&mg, order, &h, &e), e);
  return DeviceField(h);
}

// per-cell arrays carrying their own bases (RhsField, residual vectors) -> device level
inline DeviceField upload(const std::vector<MomentRep<double>>& v, const Grid2D& g, int order) {
  if ((int)v.size() != g.nx * g.ny) throw Error("momg_gpu: array size does not match the grid");
  DeviceField d = empty_like(g, order);
  const int n = IndexSet::count(order);
  std::vector<double> c(v.size() * n), p(v.size() * 4);
  for (size_t k = 0; k < v.size(); ++k) {
    if ((int)v[k].coeffs.size() != n) throw Error("momg_gpu: array order does not match the field");
    for (int q = 0; q < n; ++q) c[k * n + q] = v[k].coeffs[q];
    for (int q = 0; q < 3; ++q) p[k * 4 + q] = v[k].params.mean[q];
    p[k * 4 + 3] = v[k].params.spread;
  }
  momg_err e{};
  check(momg_field_upload(d.get(), c.data(), p.data(), &e), e);
  return d;
}

inline std::vector<MomentRep<double>> download_reps(const momg_field* d, int cells, int order) {
  const int n = IndexSet::count(order);
  std::vector<double> c((size_t)cells * n), p((size_t)cells * 4);
  momg_err e{};
  check(momg_field_download(d, c.data(), p.data(), &e), e);
  std::vector<MomentRep<double>> v(cells);
  for (int k = 0; k < cells; ++k) {
    v[k].order = order;
    v[k].coeffs = VecX<double>::Zero(n);
    for (int q = 0; q < n; ++q) v[k].coeffs[q] = c[(size_t)k * n + q];
    for (int q = 0; q < 3; ++q) v[k].params.mean[q] = p[(size_t)k * 4 + q];
    v[k].params.spread = p[(size_t)k * 4 + 3];
  }
  return v;
}

inline SolveContext context_of(const Walls& walls, const CollisionModel& model, const GasParams& gas,
                               const SpatialScheme& scheme, int threads) {
  SolveContext ctx;
  ctx.walls = walls;
  ctx.model = model;
  ctx.gas = gas;
  ctx.scheme = scheme;
  ctx.threads = threads;
  return ctx;
}

// A CellField level resident in HBM (grid.hpp:54-85 layout on the device:
// coefficients [cells][NP], params [cells][4]).  Owns the device level.
class DeviceCellField {
 public:
  DeviceCellField(const Grid2D& g, int order) : grid_(g), order_(order), d_(empty_like(g, order)) {}
  explicit DeviceCellField(const CellField& f) : grid_(f.grid()), order_(f.order()), d_(upload(f)) {}
  const Grid2D& grid() const { return grid_; }
  int order() const { return order_; }
  int size() const { return grid_.nx * grid_.ny; }
  momg_field* handle() const { return d_.get(); }
  void assign(const CellField& f) {
    momg_err e{};
    DeviceField t = upload(f);
    check(momg_field_copy(d_.get(), t.get(), &e), e);
  }
  void copy_to(CellField& f) const { download(d_.get(), f); }
  CellField to_host() const {
    CellField f(grid_, order_);
    download(d_.get(), f);
    return f;
  }

 private:
  Grid2D grid_;
  int order_;
  DeviceField d_;
};

// ---- device-resident overloads (no host copies) ----------------------------
inline void residual(const DeviceCellField& field, const SolveContext& ctx, DeviceCellField& out) {
  const momg_ctx c = context(ctx, field.order());
  momg_err e{};
  check(momg_residual(&c, field.handle(), out.handle(), &e), e);
}
inline void fast_sweep_step(DeviceCellField& field, const DeviceCellField* rhs, const SolveContext& ctx,
                            WorkStats* work = nullptr, const std::array<int, 4>& sweep_order = {0, 1, 2, 3}) {
  const momg_ctx c = context(ctx, field.order());
  long long evals = 0;
  momg_err e{};
  const int rc = momg_fast_sweep(&c, field.handle(), rhs ? rhs->handle() : nullptr, sweep_order.data(), &evals, &e);
  if (work) work->cell_evals += evals;
  check(rc, e);
}
inline double total_mass(const DeviceCellField& field) {
  double m = 0.0;
  momg_err e{};
  check(momg_total_mass(field.handle(), &m, &e), e);
  return m;
}
inline void mass_correction(DeviceCellField& field, double target_mass) {
  momg_err e{};
  check(momg_mass_correction(field.handle(), target_mass, &e), e);
}
inline void restrict_solution(const DeviceCellField& fine, DeviceCellField& coarse) {
  momg_err e{};
  check(momg_restrict_solution(fine.handle(), coarse.handle(), &e), e);
}
inline void fas_correct(DeviceCellField& fine, const DeviceCellField& before, const DeviceCellField& after) {
  momg_err e{};
  check(momg_fas_correct(fine.handle(), before.handle(), after.handle(), &e), e);
}
inline double residual_norm(const DeviceCellField& res, const DeviceCellField& field) {
  double v = 0.0;
  momg_err e{};
  check(momg_residual_norm(res.handle(), field.handle(), &v, &e), e);
  return v;
}

// ---- the reference's signatures (host CellField in, host results out) -------
// residual (spatial.cpp:135-159; spatial.hpp:52-56)
inline std::vector<MomentRep<double>> residual(const CellField& field, const Walls& walls,
                                               const CollisionModel& model, const GasParams& gas,
                                               const SpatialScheme& scheme, int threads = 1) {
  const SolveContext ctx = context_of(walls, model, gas, scheme, threads);
  DeviceField d = upload(field), out = empty_like(field.grid(), field.order());
  const momg_ctx c = context(ctx, field.order());
  momg_err e{};
  check(momg_residual(&c, d.get(), out.get(), &e), e);
  return download_reps(out.get(), field.size(), field.order());
}
inline std::vector<MomentRep<double>> residual(const CellField& field, const SolveContext& ctx) {
  return gpu::residual(field, ctx.walls, ctx.model, ctx.gas, ctx.scheme, ctx.threads);
}

// fast_sweep_step (single_level.cpp:121-166)
inline void fast_sweep_step(CellField& field, const RhsField& rhs, const SolveContext& ctx,
                            WorkStats* work = nullptr,
                            const std::array<int, 4>& sweep_order = {0, 1, 2, 3}) {
  DeviceField d = upload(field);
  DeviceField r;
  if (!rhs.empty()) r = upload(rhs, field.grid(), field.order());
  const momg_ctx c = context(ctx, field.order());
  long long evals = 0;
  momg_err e{};
  const int rc = momg_fast_sweep(&c, d.get(), r.get(), sweep_order.data(), &evals, &e);
  if (work) work->cell_evals += evals;
  if (rc == MOMG_OK) download(d.get(), field);
  check(rc, e);
}

// euler_step (single_level.cpp:74-97)
inline void euler_step(CellField& field, const std::vector<MomentRep<double>>& residuals, const RhsField& rhs,
                       const SolveContext& ctx) {
  DeviceField d = upload(field), res = upload(residuals, field.grid(), field.order());
  DeviceField r;
  if (!rhs.empty()) r = upload(rhs, field.grid(), field.order());
  const momg_ctx c = context(ctx, field.order());
  momg_err e{};
  const int rc = momg_euler_step(&c, d.get(), res.get(), r.get(), &e);
  if (rc == MOMG_OK) download(d.get(), field);
  check(rc, e);
}

// total_mass / mass_correction (single_level.cpp:168-183)
inline double total_mass(const CellField& field) {
  DeviceField d = upload(field);
  double m = 0.0;
  momg_err e{};
  check(momg_total_mass(d.get(), &m, &e), e);
  return m;
}
inline void mass_correction(CellField& field, double target_mass) {
  DeviceField d = upload(field);
  momg_err e{};
  check(momg_mass_correction(d.get(), target_mass, &e), e);
  download(d.get(), field);
}

// restrict_solution (multigrid.cpp:67-112)
inline CellField restrict_solution(const CellField& fine, const Grid2D& coarse) {
  DeviceField d = upload(fine);
  CellField out(coarse, fine.order());
  DeviceField o = empty_like(coarse, fine.order());
  momg_err e{};
  check(momg_restrict_solution(d.get(), o.get(), &e), e);
  download(o.get(), out);
  return out;
}

// restrict_residual (multigrid.cpp:114-142): the fine arrays carry their own
// bases; `fine` fixes the grid (areas), `coarse` the target bases
inline std::vector<MomentRep<double>> restrict_residual(const std::vector<MomentRep<double>>& fine_arrays,
                                                        const CellField& fine, const CellField& coarse) {
  DeviceField a = upload(fine_arrays, fine.grid(), fine.order());
  DeviceField c = upload(coarse);
  DeviceField o = empty_like(coarse.grid(), coarse.order());
  momg_err e{};
  check(momg_restrict_residual(a.get(), c.get(), o.get(), &e), e);
  return download_reps(o.get(), coarse.size(), coarse.order());
}

// fas_correct (multigrid.cpp:144-164)
inline void fas_correct(CellField& fine, const CellField& before, const CellField& after) {
  DeviceField d = upload(fine), b = upload(before), a = upload(after);
  momg_err e{};
  const int rc = momg_fas_correct(d.get(), b.get(), a.get(), &e);
  if (rc == MOMG_OK) download(d.get(), fine);
  check(rc, e);
}

// residual_norm (multigrid.cpp:202-218)
inline double residual_norm(const std::vector<MomentRep<double>>& residuals, const CellField& field) {
  DeviceField r = upload(residuals, field.grid(), field.order()), f = upload(field);
  double v = 0.0;
  momg_err e{};
  check(momg_residual_norm(r.get(), f.get(), &v, &e), e);
  return v;
}

// nmg_cycle (multigrid.cpp:166-200) on the finest level of a hierarchy built
// by GridHierarchy::build(field.grid(), levels), no rhs (the call
// solve_steady makes): the whole V-cycle device-resident, one upload and one
// download.  Other (level, rhs) combinations are the reference's recursion
// itself, which the interposer (2) runs with the GPU per-call functions.
inline void nmg_cycle(const GridHierarchy& hierarchy, int level, CellField& field, const RhsField& rhs,
                      const SolveContext& ctx, const CyclePolicy& policy, WorkStats* work = nullptr) {
  if (!rhs.empty() || level != hierarchy.finest_level() || field.grid().nx != hierarchy.grids.back().nx ||
      field.grid().ny != hierarchy.grids.back().ny)
    throw ConfigError("momg::gpu::nmg_cycle: device V-cycle runs the finest level without rhs");
  DeviceField d = upload(field);
  const momg_ctx c = context(ctx, field.order());
  long long w = 0;
  momg_err e{};
  const int rc = momg_nmg_cycle(&c, d.get(), (int)hierarchy.grids.size(), policy.s1, policy.s2, policy.s3,
                                policy.gamma, &w, &e);
  if (work) work->cell_evals += w;
  if (rc == MOMG_OK) download(d.get(), field);
  check(rc, e);
}

// solve_steady (multigrid.cpp:243-320), device-resident from start to end
inline SolveReport solve_steady(CellField& field, const SolveContext& ctx,
                                const SolverOptions& options) {
  DeviceField d = upload(field);
  const momg_ctx c = context(ctx, field.order());
  momg_solver_opts o{};
  o.kind = options.kind == SolverKind::euler ? 0 : options.kind == SolverKind::fs ? 1 : 2;
  o.tol = options.tol;
  o.max_iterations = options.max_iterations;
  o.levels = options.levels;
  o.s1 = options.cycle.s1;
  o.s2 = options.cycle.s2;
  o.s3 = options.cycle.s3;
  o.gamma = options.cycle.gamma;
  std::vector<double> hist(100000), secs(100000);
  momg_report r{};
  r.history = hist.data();
  r.history_cap = (int)hist.size();
  r.history_seconds = secs.data();
  momg_err e{};
  const int rc = momg_solve_steady(&c, d.get(), &o, &r, &e);
  SolveReport rep;
  rep.converged = r.converged;
  rep.iterations = r.iterations;
  rep.r0_norm = r.r0_norm;
  rep.final_norm = r.final_norm;
  rep.final_ratio = r.final_ratio;
  rep.work = r.work;
  rep.seconds = r.seconds;
  for (int k = 0; k < r.history_len && k < r.history_cap; ++k)
    rep.history.push_back({k + 1, hist[k], secs[k]});
  download(d.get(), field);
  if (rc != MOMG_OK) rethrow(rc, e, &rep);
  return rep;
}

}  // namespace gpu
}  // namespace momg
