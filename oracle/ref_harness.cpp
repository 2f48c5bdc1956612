// extern "C" harness over the REFERENCE library -- TEST INFRASTRUCTURE ONLY.
//
// Linked with the reference's own translation units (oracle/Makefile) into
// oracle/_ref/libmomg_ref.so.  Each entry point converts flat arrays to the
// reference's types (CellField / MomentRep / Grid2D, grid.hpp:12-85), calls the
// reference function named in its comment, and maps its exceptions onto
// mo_err codes.  No arithmetic of the path happens here.
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "momg/collision.hpp"
#include "momg/flux.hpp"
#include "momg/halfspace.hpp"
#include "momg/hermite.hpp"
#include "momg/multigrid.hpp"
#include "momg/projection.hpp"
#include "momg/scenario.hpp"
#include "momg/single_level.hpp"
#include "momg/spatial.hpp"
#include "momg_oracle.h"

using namespace momg;

namespace {

void set_err(mo_err* err, int code, const char* what) {
  if (!err) return;
  err->code = code;
  std::strncpy(err->msg, what, sizeof(err->msg) - 1);
  err->msg[sizeof(err->msg) - 1] = 0;
}

template <typename F>
int guarded(mo_err* err, F&& f) {
  if (err) {
    err->code = MO_OK;
    err->msg[0] = 0;
  }
  try {
    f();
    return MO_OK;
  } catch (const NonConvergence& e) {
    set_err(err, MO_NONCONVERGENCE, e.what());
    return MO_NONCONVERGENCE;
  } catch (const NonphysicalState& e) {
    set_err(err, MO_NONPHYSICAL_STATE, e.what());
    return MO_NONPHYSICAL_STATE;
  } catch (const SolverError& e) {
    set_err(err, MO_SOLVER_ERROR, e.what());
    return MO_SOLVER_ERROR;
  } catch (const NonSpdTensor& e) {
    set_err(err, MO_NON_SPD, e.what());
    return MO_NON_SPD;
  } catch (const ConfigError& e) {
    set_err(err, MO_CONFIG, e.what());
    return MO_CONFIG;
  } catch (const std::exception& e) {
    set_err(err, MO_ERROR, e.what());
    return MO_ERROR;
  }
}

BasisParams<double> bp(const double* p) {
  BasisParams<double> b;
  b.mean = Vec3<double>(p[0], p[1], p[2]);
  b.spread = p[3];
  return b;
}
void put_bp(const BasisParams<double>& b, double* p) {
  p[0] = b.mean[0];
  p[1] = b.mean[1];
  p[2] = b.mean[2];
  p[3] = b.spread;
}
MomentRep<double> rep(int M, const double* c, const double* p) {
  MomentRep<double> r;
  r.order = M;
  r.params = bp(p);
  const int n = IndexSet::count(M);
  r.coeffs = VecX<double>(n);
  for (int k = 0; k < n; ++k) r.coeffs[k] = c[k];
  return r;
}
void put_coeffs(const VecX<double>& v, double* out) {
  for (int k = 0; k < v.size(); ++k) out[k] = v[k];
}

Grid2D grid(const mo_grid* g) {
  Grid2D out;
  out.nx = g->nx;
  out.ny = g->ny;
  out.Lx = g->Lx;
  out.Ly = g->Ly;
  out.dx.assign(g->dx, g->dx + g->nx);
  out.dy.assign(g->dy, g->dy + g->ny);
  out.xc.assign(g->xc, g->xc + g->nx);
  out.yc.assign(g->yc, g->yc + g->ny);
  return out;
}

CellField field(const Grid2D& g, int M, const double* c, const double* p) {
  CellField f(g, M);
  const int n = IndexSet::count(M);
  for (int k = 0; k < f.size(); ++k) f[k] = rep(M, c + (size_t)k * n, p + (size_t)k * 4);
  return f;
}
void put_field(const CellField& f, double* c, double* p) {
  const int n = IndexSet::count(f.order());
  for (int k = 0; k < f.size(); ++k) {
    put_coeffs(f[k].coeffs, c + (size_t)k * n);
    if (p) put_bp(f[k].params, p + (size_t)k * 4);
  }
}
std::vector<MomentRep<double>> arrays(int M, int cells, const double* c, const double* p) {
  const int n = IndexSet::count(M);
  std::vector<MomentRep<double>> v(cells);
  for (int k = 0; k < cells; ++k) v[k] = rep(M, c + (size_t)k * n, p + (size_t)k * 4);
  return v;
}

SolveContext context(const mo_ctx* c) {
  SolveContext ctx;
  auto wall = [&](int w) {
    WallSpec s;
    s.speed = c->wall_speed[w];
    s.theta = c->wall_theta[w];
    return s;
  };
  ctx.walls.left = wall(MO_WALL_LEFT);
  ctx.walls.right = wall(MO_WALL_RIGHT);
  ctx.walls.bottom = wall(MO_WALL_BOTTOM);
  ctx.walls.top = wall(MO_WALL_TOP);
  ctx.model.kind = c->collision == MO_BGK ? CollisionKind::bgk
                   : c->collision == MO_ES_BGK ? CollisionKind::es_bgk
                                               : CollisionKind::shakhov;
  ctx.model.prandtl = c->prandtl;
  ctx.gas.knudsen = c->knudsen;
  ctx.gas.viscosity_index = c->viscosity_index;
  ctx.scheme.order = c->space_order;
  ctx.scheme.c_bound = c->c_bound;
  ctx.cfl.cfl = c->cfl;
  ctx.cfl.c_bound = c->cfl_c_bound;
  ctx.threads = c->threads > 0 ? c->threads : 1;
  return ctx;
}

}  // namespace

extern "C" {

int mo_index_count(int M) { return IndexSet::count(M); }

// multi_index.hpp:25-103 / tables.cpp:12-20
void mo_index_tables(int M, int* a, int* down, int* up, int* degree, double* factorial) {
  const IndexSet& s = index_set(M);
  const int n = s.size();
  for (int k = 0; k < n; ++k) {
    a[3 * k] = s[k].a1;
    a[3 * k + 1] = s[k].a2;
    a[3 * k + 2] = s[k].a3;
    for (int d = 0; d < 3; ++d) {
      down[d * n + k] = s.down(k, d);
      up[d * n + k] = s.up(k, d);
    }
    degree[k] = s.degree(k);
    factorial[k] = s.factorial(k);
  }
}

// tables.cpp:22-41
double mo_max_hermite_root(int degree) { return max_hermite_root(degree); }

// projection.hpp:83-89
int mo_project(int M, const double* coeffs, const double* from, const double* to,
               double* out, mo_err* err) {
  return guarded(err, [&] { put_coeffs(project(rep(M, coeffs, from), bp(to)).coeffs, out); });
}

// projection.hpp:96-121
int mo_grad_normalize(int M, double* coeffs, double* params, mo_err* err) {
  return guarded(err, [&] {
    MomentRep<double> r = rep(M, coeffs, params);
    try {
      grad_normalize(r);
    } catch (...) {
      put_coeffs(r.coeffs, coeffs);
      put_bp(r.params, params);
      throw;
    }
    put_coeffs(r.coeffs, coeffs);
    put_bp(r.params, params);
  });
}

// moment_rep.hpp:97-110
double mo_grad_defect(int M, const double* coeffs) {
  const double zero[4] = {0, 0, 0, 1};
  return grad_defect(rep(M, coeffs, zero));
}

// halfspace.hpp:18-57
void mo_half_range_table(int pmax, double a, double* upper, double* lower) {
  HalfRangeTable<double> t(pmax, a);
  for (int m = 0; m <= pmax; ++m)
    for (int p = 0; p <= pmax; ++p) {
      upper[m * (pmax + 1) + p] = t.upper(m, p);
      lower[m * (pmax + 1) + p] = t.lower(m, p);
    }
}

// flux.cpp:29-75
int mo_half_flux(int M, const double* coeffs, const double* params, int axis,
                 int positive_side, double* out, mo_err* err) {
  return guarded(err, [&] {
    put_coeffs(half_flux_coeffs(rep(M, coeffs, params), axis, positive_side != 0).coeffs, out);
  });
}

// flux.cpp:10-27
void mo_full_flux(int M, const double* coeffs, const double* params, int axis, double* out) {
  put_coeffs(full_flux_coeffs(rep(M, coeffs, params), axis).coeffs, out);
}

// flux.cpp:77-97
int mo_face_flux(int M, const double* lc, const double* lp, const double* rc,
                 const double* rp, int axis, double c_bound, double* out,
                 double* out_params, mo_err* err) {
  return guarded(err, [&] {
    MomentRep<double> f = face_flux(rep(M, lc, lp), rep(M, rc, rp), axis, c_bound);
    put_coeffs(f.coeffs, out);
    put_bp(f.params, out_params);
  });
}

// flux.cpp:105-130
int mo_wall_flux(int M, const double* c, const double* p, int axis, int high_side,
                 double speed, double theta, double* out, double* out_params,
                 mo_err* err) {
  return guarded(err, [&] {
    WallSpec w;
    w.speed = speed;
    w.theta = theta;
    MomentRep<double> f = wall_flux(rep(M, c, p), axis, high_side != 0, w);
    put_coeffs(f.coeffs, out);
    put_bp(f.params, out_params);
  });
}

// collision.hpp:120-127
int mo_collision(const mo_ctx* ctx, const double* coeffs, const double* params,
                 double* out, mo_err* err) {
  return guarded(err, [&] {
    const SolveContext c = context(ctx);
    put_coeffs(collision_coeffs(rep(ctx->M, coeffs, params), c.model, c.gas), out);
  });
}

// spatial.cpp:135-159
int mo_residual(const mo_ctx* ctx, const mo_grid* g, const double* coeffs,
                const double* params, double* res_out, mo_err* err) {
  return guarded(err, [&] {
    const SolveContext c = context(ctx);
    const CellField f = field(grid(g), ctx->M, coeffs, params);
    const auto r = residual(f, c.walls, c.model, c.gas, c.scheme, c.threads);
    const int n = IndexSet::count(ctx->M);
    for (size_t k = 0; k < r.size(); ++k) put_coeffs(r[k].coeffs, res_out + k * n);
  });
}

// single_level.cpp:121-166
int mo_fast_sweep(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                  const double* rhs_coeffs, const double* rhs_params,
                  const int* sweep_order, long long* evals, mo_err* err) {
  const SolveContext c = context(ctx);
  CellField f = field(grid(g), ctx->M, coeffs, params);
  RhsField rhs;
  if (rhs_coeffs) rhs = arrays(ctx->M, f.size(), rhs_coeffs, rhs_params);
  std::array<int, 4> order = {0, 1, 2, 3};
  if (sweep_order)
    for (int s = 0; s < 4; ++s) order[s] = sweep_order[s];
  WorkStats work;
  const int rc = guarded(err, [&] { fast_sweep_step(f, rhs, c, &work, order); });
  put_field(f, coeffs, params);
  if (evals) *evals = work.cell_evals;
  return rc;
}

// single_level.cpp:168-174
double mo_total_mass(const mo_grid* g, int M, const double* coeffs) {
  std::vector<double> p(4 * (size_t)g->nx * g->ny, 0.0);
  for (size_t k = 0; k < p.size(); k += 4) p[k + 3] = 1.0;
  return total_mass(field(grid(g), M, coeffs, p.data()));
}

// single_level.cpp:176-183
int mo_mass_correction(const mo_grid* g, int M, double* coeffs, double target, mo_err* err) {
  std::vector<double> p(4 * (size_t)g->nx * g->ny, 0.0);
  for (size_t k = 0; k < p.size(); k += 4) p[k + 3] = 1.0;
  CellField f = field(grid(g), M, coeffs, p.data());
  const int rc = guarded(err, [&] { mass_correction(f, target); });
  put_field(f, coeffs, nullptr);
  return rc;
}

// multigrid.cpp:67-112
int mo_restrict_solution(int M, const mo_grid* fine, const double* fc, const double* fp,
                         const mo_grid* coarse, double* cc, double* cp, mo_err* err) {
  return guarded(err, [&] {
    const CellField f = field(grid(fine), M, fc, fp);
    const CellField out = restrict_solution(f, grid(coarse));
    put_field(out, cc, cp);
  });
}

// multigrid.cpp:114-142
int mo_restrict_residual(int M, const mo_grid* fine, const double* arr_c,
                         const double* arr_p, const double* fine_params,
                         const mo_grid* coarse, const double* coarse_params,
                         double* out, mo_err* err) {
  return guarded(err, [&] {
    const Grid2D fg = grid(fine), cg = grid(coarse);
    const int n = IndexSet::count(M);
    std::vector<double> zc((size_t)fg.cells() * n, 0.0), zcc((size_t)cg.cells() * n, 0.0);
    const CellField f = field(fg, M, zc.data(), fine_params);
    const CellField c = field(cg, M, zcc.data(), coarse_params);
    const auto r = restrict_residual(arrays(M, fg.cells(), arr_c, arr_p), f, c);
    for (size_t k = 0; k < r.size(); ++k) put_coeffs(r[k].coeffs, out + k * n);
  });
}

// multigrid.cpp:144-164
int mo_fas_correct(int M, const mo_grid* fine, double* fc, double* fp,
                   const mo_grid* coarse, const double* bc, const double* bp_,
                   const double* ac, const double* ap, mo_err* err) {
  CellField f = field(grid(fine), M, fc, fp);
  const Grid2D cg = grid(coarse);
  const CellField before = field(cg, M, bc, bp_);
  const CellField after = field(cg, M, ac, ap);
  const int rc = guarded(err, [&] { fas_correct(f, before, after); });
  put_field(f, fc, fp);
  return rc;
}

// multigrid.cpp:202-218
double mo_residual_norm(int M, const mo_grid* g, const double* res, const double* field_params) {
  const Grid2D gg = grid(g);
  const int n = IndexSet::count(M);
  std::vector<double> z((size_t)gg.cells() * n, 0.0);
  const CellField f = field(gg, M, z.data(), field_params);
  return residual_norm(arrays(M, gg.cells(), res, field_params), f);
}

// multigrid.cpp:243-320
int mo_solve_steady(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                    int solver, double tol, int max_iterations, int levels, int s1,
                    int s2, int s3, int gamma, mo_report* report, mo_err* err) {
  const SolveContext c = context(ctx);
  CellField f = field(grid(g), ctx->M, coeffs, params);
  SolverOptions opt;
  opt.kind = solver == 0 ? SolverKind::euler : solver == 1 ? SolverKind::fs : SolverKind::nmg;
  opt.tol = tol;
  opt.max_iterations = max_iterations;
  opt.levels = levels;
  opt.cycle.s1 = s1;
  opt.cycle.s2 = s2;
  opt.cycle.s3 = s3;
  opt.cycle.gamma = gamma;
  SolveReport rep_out;
  const int rc = guarded(err, [&] {
    try {
      rep_out = solve_steady(f, c, opt);
    } catch (const NonConvergence& e) {
      rep_out = e.report();
      throw;
    }
  });
  put_field(f, coeffs, params);
  if (report) {
    report->converged = rep_out.converged;
    report->iterations = rep_out.iterations;
    report->r0_norm = rep_out.r0_norm;
    report->final_norm = rep_out.final_norm;
    report->final_ratio = rep_out.final_ratio;
    report->work = rep_out.work;
    report->seconds = rep_out.seconds;
    report->history_len = 0;
    for (const HistoryEntry& h : rep_out.history) {
      if (report->history && report->history_len < report->history_cap)
        report->history[report->history_len] = h.rel_residual;
      ++report->history_len;
    }
  }
  return rc;
}

// multigrid.cpp:166-200 on a hierarchy from GridHierarchy::build (multigrid.cpp:44-65)
int mo_nmg_cycle(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                 int levels, int s1, int s2, int s3, int gamma, long long* work,
                 mo_err* err) {
  const SolveContext c = context(ctx);
  CellField f = field(grid(g), ctx->M, coeffs, params);
  WorkStats ws;
  const int rc = guarded(err, [&] {
    const GridHierarchy h = GridHierarchy::build(f.grid(), levels);
    CyclePolicy pol;
    pol.s1 = s1;
    pol.s2 = s2;
    pol.s3 = s3;
    pol.gamma = gamma;
    nmg_cycle(h, h.finest_level(), f, {}, c, pol, &ws);
  });
  put_field(f, coeffs, params);
  if (work) *work = ws.cell_evals;
  return rc;
}

// single_level.cpp:74-97 (residual + euler_step as solve_steady does, multigrid.cpp:257,277)
int mo_euler_step(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                  mo_err* err) {
  const SolveContext c = context(ctx);
  CellField f = field(grid(g), ctx->M, coeffs, params);
  const int rc = guarded(err, [&] {
    const auto r = residual(f, c.walls, c.model, c.gas, c.scheme, c.threads);
    euler_step(f, r, {}, c);
  });
  put_field(f, coeffs, params);
  return rc;
}

int mo_euler_step_rhs(const mo_ctx* ctx, const mo_grid* g, double* coeffs, double* params,
                      const double* rhs_coeffs, const double* rhs_params, mo_err* err) {
  const SolveContext c = context(ctx);
  CellField f = field(grid(g), ctx->M, coeffs, params);
  RhsField rhs;
  if (rhs_coeffs) rhs = arrays(ctx->M, f.size(), rhs_coeffs, rhs_params);
  const int rc = guarded(err, [&] {
    const auto r = residual(f, c.walls, c.model, c.gas, c.scheme, c.threads);
    euler_step(f, r, rhs, c);
  });
  put_field(f, coeffs, params);
  return rc;
}


// ---- front end (scenario.cpp), reference only: golden fixtures of the wire formats
// parse_config (scenario.cpp:219-311) + config_echo (:321-352) of a JSON document
int mo_ref_config_echo(const char* json_text, char* out, int cap, mo_err* err) {
  return guarded(err, [&] {
    const std::string e = config_echo(parse_config(json_text));
    std::snprintf(out, (size_t)cap, "%s", e.c_str());
    if ((int)e.size() >= cap) throw Error("mo_ref_config_echo: buffer too small");
  });
}

// run_scenario (scenario.cpp:401-459) of a JSON document: writes history.tsv,
// field.tsv and report.txt under its output_dir
int mo_ref_run_scenario(const char* json_text, mo_err* err) {
  return guarded(err, [&] { run_scenario(parse_config(json_text)); });
}

// export_field (scenario.cpp:372-399) of a given field with the unit scales of a
// JSON document's configuration
int mo_ref_export_field(const char* json_text, const mo_grid* g, int M, const double* coeffs,
                        const double* params, const char* path, mo_err* err) {
  return guarded(err, [&] {
    const ScenarioConfig c = parse_config(json_text);
    export_field(field(grid(g), M, coeffs, params), c, unit_scales(c), path);
  });
}

}  // extern "C"
