"""Checkpointed CPU-oracle NMG solve of a BASELINE cavity config (C3 / C4 are
hours long on one core) -- TEST INFRASTRUCTURE ONLY.

Restates the iteration loop of solve_steady (multigrid.cpp:243-320) on top of
the oracle's own nmg_cycle / mass_correction / residual / residual_norm, so
the result is the oracle's solve_steady, but the state is written after
every V-cycle:

  oracle_runs/<name>_<kind>_hist.json   iteration, ratio, wall time (every cycle)
  oracle_runs/<name>_<kind>_it<k>.npz   full field after cycle k (k = 1, 2, final)
  tests/golden/<name>_it<k>.npz         compact fixture (see compact()), committed

Usage: python tools/oracle_solve_ckpt.py C3 [--ref] [--max N]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle.api import Grid, Oracle, uniform_field  # noqa: E402
from tools.run_oracle_configs import CONFIGS  # noqa: E402
from oracle.api import Ctx  # noqa: E402


def compact(c, p, nx, ny):
    """Size-independent summary of a field: per-row and per-column coefficient
    sums (ny x N, nx x N), the params and rho on every 4th cell."""
    n = c.shape[1]
    c3 = c.reshape(ny, nx, n)
    p3 = p.reshape(ny, nx, 4)
    return dict(row_sums=c3.sum(axis=1), col_sums=c3.sum(axis=0),
                params_sub=p3[::4, ::4].copy(), rho_sub=c3[::4, ::4, 0].copy())


def main():
    name = sys.argv[1]
    kind = "reference" if "--ref" in sys.argv else "port"
    cap = int(sys.argv[sys.argv.index("--max") + 1]) if "--max" in sys.argv else 200
    n, M, order, model, kn, pr, lid, bt, solver, levels = CONFIGS[name]
    o = Oracle(kind)
    g = Grid.uniform(n, n)
    cb = o.max_hermite_root(M + 1)
    ctx = Ctx(M=M, space_order=order, c_bound=cb, cfl=0.9, cfl_c_bound=cb, collision=model,
              prandtl=pr, knudsen=kn, wall_speed=(0, 0, 0, lid), wall_theta=(1, 1, bt, 1))
    c, p = uniform_field(g, M)
    run_dir = os.path.join(ROOT, "oracle_runs")
    os.makedirs(run_dir, exist_ok=True)
    hist_path = os.path.join(run_dir, f"{name}_{kind}_hist.json")
    t0 = time.time()
    res = o.residual(ctx, g, c, p)
    r0 = o.residual_norm(M, g, res, p)
    target = o.total_mass(g, M, c)
    hist = dict(config=dict(n=n, M=M, order=order, model=model, Kn=kn, Pr=pr, lid=lid,
                            bottom_theta=bt, levels=levels, c_bound=cb, kind=kind),
                r0_norm=r0, target_mass=target, history=[], converged=False)
    for it in range(1, cap + 1):
        try:
            c, p, w = o.nmg_cycle(ctx, g, c, p, levels=levels)
            c = o.mass_correction(g, M, c, target)
            res = o.residual(ctx, g, c, p)
        except Exception as e:  # NonConvergence mapping of solve_steady
            hist["error"] = str(e)
            json.dump(hist, open(hist_path, "w"), indent=1)
            raise
        nrm = o.residual_norm(M, g, res, p)
        ratio = nrm / r0
        hist["history"].append(dict(it=it, ratio=ratio, norm=nrm, wall_s=time.time() - t0))
        hist["iterations"] = it
        print(f"{name} it {it} ratio {ratio:.6e} t {time.time() - t0:.0f}s", flush=True)
        last = ratio <= 1e-8 or not np.isfinite(ratio) or ratio > 1e6
        if it in (1, 2) or last:
            tag = f"it{it}" if it <= 2 else "final"
            np.savez_compressed(os.path.join(run_dir, f"{name}_{kind}_{tag}.npz"), coeffs=c, params=p)
            np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"{name}_{tag}.npz"),
                                iteration=it, ratio=ratio, norm=nrm, r0_norm=r0,
                                mass=o.total_mass(g, M, c), **compact(c, p, n, n))
        if ratio <= 1e-8:
            hist["converged"] = True
        json.dump(hist, open(hist_path, "w"), indent=1)
        if last:
            break


if __name__ == "__main__":
    main()
