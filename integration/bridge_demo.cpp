// The reference's own program, switched to the B200 by one include: runs C1
// (BASELINE configs[0]: 32^2 lid cavity, M = 3, FS to 1e-8) with the
// reference's CPU solve_steady and with momg::gpu::solve_steady, and prints a
// JSON line comparing iterations and fields.  Built by `make -C oracle
// bridge` against the reference sources; without a GPU it reports the
// DeviceUnavailable status (no CPU fallback).
#include <chrono>
#include <cmath>
#include <cstdio>

#include "momg_gpu_bridge.hpp"

int main(int argc, char** argv) {
  using namespace momg;
  const int n = argc > 1 ? std::atoi(argv[1]) : 32;
  const Grid2D g = Grid2D::uniform(n, n, 1.0, 1.0);
  SolveContext ctx;
  ctx.walls.top.speed = 0.1;
  ctx.model.kind = CollisionKind::bgk;
  ctx.gas.knudsen = 0.1;
  ctx.scheme = SpatialScheme::for_moment_order(3, 1);
  ctx.cfl.c_bound = ctx.scheme.c_bound;
  SolverOptions opt;
  opt.kind = SolverKind::fs;
  opt.tol = 1e-8;
  CellField cpu = uniform_field(g, 3, 1.0, zero3(), 1.0);
  CellField gpu = cpu;
  auto t0 = std::chrono::steady_clock::now();
  const SolveReport rc = solve_steady(cpu, ctx, opt);
  auto t1 = std::chrono::steady_clock::now();
  SolveReport rg;
  try {
    rg = gpu::solve_steady(gpu, ctx, opt);
  } catch (const Error& e) {
    std::printf("{\"cpu_iterations\": %d, \"gpu\": \"%s\"}\n", rc.iterations, e.what());
    return 0;
  }
  auto t2 = std::chrono::steady_clock::now();
  double maxdiff = 0.0;
  for (int k = 0; k < cpu.size(); ++k) {
    maxdiff = std::max(maxdiff, std::fabs(cpu[k].coeffs[0] - gpu[k].coeffs[0]));
    for (int d = 0; d < 3; ++d)
      maxdiff = std::max(maxdiff, std::fabs(cpu[k].params.mean[d] - gpu[k].params.mean[d]));
    maxdiff = std::max(maxdiff, std::fabs(cpu[k].params.spread - gpu[k].params.spread));
  }
  std::printf("{\"n\": %d, \"cpu_iterations\": %d, \"gpu_iterations\": %d, \"max_macro_diff\": %.3e, "
              "\"cpu_s\": %.3f, \"gpu_s\": %.3f}\n",
              n, rc.iterations, rg.iterations, maxdiff,
              std::chrono::duration<double>(t1 - t0).count(),
              std::chrono::duration<double>(t2 - t1).count());
  return (std::abs(rc.iterations - rg.iterations) <= 1 && maxdiff < 1e-8) ? 0 : 1;
}
