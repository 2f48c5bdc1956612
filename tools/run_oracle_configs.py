"""Runs the CPU oracle (C restatement; optionally the reference itself) on the
BASELINE.json cavity configs and records iteration counts, timings and the
final residual history to tests/golden/configs_<name>.json (test fixtures for
the GPU solve parity).  Usage: python tools/run_oracle_configs.py C1 [C2 ...] [--ref]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.api import BGK, SHAKHOV, Ctx, Grid, Oracle, uniform_field  # noqa: E402

CONFIGS = {
    # name: (n, M, order, model, Kn, Pr, lid, bottom_theta, solver, levels)
    "C1": (32, 3, 1, BGK, 0.1, 1.0, 0.1, 1.0, 1, 0),
    "C2": (128, 5, 2, BGK, 0.1, 1.0, 0.1, 1.0, 2, 4),
    "C3": (256, 8, 2, SHAKHOV, 0.01, 2.0 / 3.0, 0.1, 1.0, 2, 5),
    "C4": (512, 6, 2, BGK, 0.1, 1.0, 0.0, 2.0, 2, 6),
    "C2o1": (128, 5, 1, BGK, 0.1, 1.0, 0.1, 1.0, 2, 4),
}


def run(name, kind="port", max_iterations=0):
    n, M, order, model, kn, pr, lid, bt, solver, levels = CONFIGS[name]
    o = Oracle(kind)
    g = Grid.uniform(n, n)
    cb = o.max_hermite_root(M + 1)
    ctx = Ctx(M=M, space_order=order, c_bound=cb, cfl=0.9, cfl_c_bound=cb, collision=model,
              prandtl=pr, knudsen=kn, wall_speed=(0, 0, 0, lid), wall_theta=(1, 1, bt, 1))
    c, p = uniform_field(g, M)
    t = time.time()
    c, p, rep = o.solve_steady(ctx, g, c, p, solver=solver, tol=1e-8, levels=levels,
                               max_iterations=max_iterations)
    rep["wall_s"] = time.time() - t
    rep["history"] = [float(x) for x in rep["history"]]
    rep["config"] = dict(n=n, M=M, order=order, model=model, Kn=kn, Pr=pr, lid=lid,
                         bottom_theta=bt, solver=solver, levels=levels, c_bound=cb, kind=kind)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                       "golden", f"configs_{name}_{kind}.json")
    json.dump(rep, open(out, "w"), indent=1)
    np.savez_compressed(out.replace(".json", "_field.npz"), coeffs=c, params=p)
    print(name, kind, {k: rep[k] for k in ("rc", "converged", "iterations", "final_ratio", "wall_s")})


if __name__ == "__main__":
    kind = "reference" if "--ref" in sys.argv else "port"
    for a in sys.argv[1:]:
        if not a.startswith("--"):
            run(a, kind)
