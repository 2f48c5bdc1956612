"""Device NMG solves of the BASELINE cavity configs to ||R||/||R0|| <= 1e-8
(solve_steady, multigrid.cpp:243-320, device-resident, CUDA-graph iterations):
iterations, wall time, per-V-cycle time and the residual history, plus the
compact field summary of tools/make_config_fixtures.py for comparison with
the oracle's run when it finishes.  Usage: python tools/solve_configs_device.py C3 C4 [--max N]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2206_13164_b200 import momg  # noqa: E402
from tools.make_config_fixtures import compact  # noqa: E402

CONFIGS = {  # name: (n, M, order, model, Kn, Pr, lid, bottom theta, levels)
    "C2": (128, 5, 2, momg.CollisionKind.bgk, 0.1, 1.0, 0.1, 1.0, 4),
    "C3": (256, 8, 2, momg.CollisionKind.shakhov, 0.01, 2.0 / 3.0, 0.1, 1.0, 5),
    "C4": (512, 6, 2, momg.CollisionKind.bgk, 0.1, 1.0, 0.0, 2.0, 6),
}


def main():
    names = [a for a in sys.argv[1:] if a in CONFIGS]
    cap = int(sys.argv[sys.argv.index("--max") + 1]) if "--max" in sys.argv else 0
    out = {}
    for name in names:
        n, M, order, model, kn, pr, lid, bt, levels = CONFIGS[name]
        ctx = momg.cavity_context(M, order, model, knudsen=kn, lid=lid, prandtl=pr, bottom_theta=bt)
        g = momg.Grid2D.uniform(n, n)
        f = momg.uniform_field(g, M, 1.0, (0.0, 0.0, 0.0), 1.0)
        momg.synchronize()
        t = time.perf_counter()
        try:
            rep = momg.solve_steady(f, ctx, momg.SolverOptions(momg.SolverKind.nmg, 1e-8, cap, levels))
            status = "converged" if rep.converged else "not converged"
        except momg.NonConvergence as e:
            rep, status = e.report, f"NonConvergence: {e}"
        wall = time.perf_counter() - t
        c, p = f.download()
        out[name] = dict(status=status, iterations=rep.iterations, seconds=wall,
                         ms_per_vcycle=1e3 * wall / max(1, rep.iterations), final_ratio=rep.final_ratio,
                         history=rep.history, work=rep.work, graph_replays=momg.graph_replays())
        np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"{name}_device_final.npz"), **compact(c, p, n))
        print(name, status, rep.iterations, f"{wall:.1f} s", flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "configs_device.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
