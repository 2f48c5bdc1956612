// Drop-in bridge for the reference's own C++ (namespace momg, /root/reference/proj):
// the same signatures as the reference functions, executed on the B200 through
// the C ABI of include/momg_gpu.h.  A maintainer of the reference switches the
// hot path by including this header and calling momg::gpu::X where the driver
// called momg::X (or replacing the calls at multigrid.cpp:170-199, 257-288).
//
//   momg::gpu::residual          <- spatial.hpp:52-56
//   momg::gpu::fast_sweep_step   <- single_level.hpp:63-65
//   momg::gpu::restrict_solution <- multigrid.hpp:41
//   momg::gpu::fas_correct       <- multigrid.hpp:52-53
//   momg::gpu::solve_steady      <- multigrid.hpp:114-116 (whole solve device-resident)
//
// Per-call functions upload / download the CellField (the reference keeps
// host AoS fields); solve_steady keeps everything in HBM and only copies the
// converged field back.  Errors are rethrown as the reference's exception
// types (types.hpp:20-57, NonConvergence multigrid.hpp:89-97).
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

// residual (spatial.cpp:135-159)
inline std::vector<MomentRep<double>> residual(const CellField& field, const SolveContext& ctx) {
  DeviceField d = upload(field), out = upload(field);
  const momg_ctx c = context(ctx, field.order());
  momg_err e{};
  check(momg_residual(&c, d.get(), out.get(), &e), e);
  CellField r = field;
  download(out.get(), r);
  std::vector<MomentRep<double>> v(r.size());
  for (int k = 0; k < r.size(); ++k) v[k] = r[k];
  return v;
}

// fast_sweep_step (single_level.cpp:121-166)
inline void fast_sweep_step(CellField& field, const RhsField& rhs, const SolveContext& ctx,
                            WorkStats* work = nullptr,
                            const std::array<int, 4>& sweep_order = {0, 1, 2, 3}) {
  DeviceField d = upload(field);
  DeviceField r;
  if (!rhs.empty()) {
    CellField rf = field;
    for (int k = 0; k < rf.size(); ++k) rf[k] = rhs[k];
    r = upload(rf);
  }
  const momg_ctx c = context(ctx, field.order());
  long long evals = 0;
  momg_err e{};
  const int rc = momg_fast_sweep(&c, d.get(), r.get(), sweep_order.data(), &evals, &e);
  if (work) work->cell_evals += evals;
  download(d.get(), field);
  check(rc, e);
}

// restrict_solution (multigrid.cpp:67-112)
inline CellField restrict_solution(const CellField& fine, const Grid2D& coarse) {
  DeviceField d = upload(fine);
  CellField out(coarse, fine.order());
  DeviceField o = upload(out);
  momg_err e{};
  check(momg_restrict_solution(d.get(), o.get(), &e), e);
  download(o.get(), out);
  return out;
}

// fas_correct (multigrid.cpp:144-164)
inline void fas_correct(CellField& fine, const CellField& before, const CellField& after) {
  DeviceField d = upload(fine), b = upload(before), a = upload(after);
  momg_err e{};
  const int rc = momg_fas_correct(d.get(), b.get(), a.get(), &e);
  download(d.get(), fine);
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
  std::vector<double> hist(100000);
  momg_report r{};
  r.history = hist.data();
  r.history_cap = (int)hist.size();
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
    rep.history.push_back({k + 1, hist[k], 0.0});
  download(d.get(), field);
  if (rc != MOMG_OK) rethrow(rc, e, &rep);
  return rep;
}

}  // namespace gpu
}  // namespace momg
