"""Probe of the register-resident band kernel against the split kernel on
small fields (one configuration per process: a device fault ends only that
case).  Usage: python tools/rb_probe.py [case ...]  (case = M,nx,ny,op)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_case(M, nx, ny, op):
    from paper_2206_13164_b200 import momg
    from paper_2206_13164_b200.synthetic import c5_field
    g = momg.Grid2D.uniform(nx, ny)
    ctx = momg.cavity_context(M, 1, knudsen=0.1, lid=0.1)
    c, p = c5_field(nx, ny, M, seed=3)
    out = {}
    for kind in ("split", "register"):
        momg.set_band_kernel(kind)
        f = momg.CellField.from_host(g, M, c, p)
        if op == "res":
            r = momg.residual(f, ctx)
            out[kind] = r.download()
        else:
            momg.fast_sweep_step(f, None, ctx)
            out[kind] = f.download()
    a, b = out["split"], out["register"]
    scale = np.maximum(1.0, np.abs(a[0]).max())
    e = float(np.max(np.abs(a[0] - b[0])) / scale)
    ep = float(np.max(np.abs(a[1] - b[1])))
    return e, ep


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        M, nx, ny = map(int, sys.argv[2:5])
        e, ep = run_case(M, nx, ny, sys.argv[5])
        print(f"RESULT {M} {nx} {ny} {sys.argv[5]} coeff {e:.3e} params {ep:.3e}", flush=True)
        sys.exit(0)
    cases = [a.split(",") for a in sys.argv[1:]] or [
        (m, nx, ny, op) for op in ("sweep", "res") for m in (5, 4, 3)
        for nx, ny in ((12, 10), (32, 8), (33, 9), (64, 40), (100, 20), (70, 66))]
    for m, nx, ny, op in cases:
        r = subprocess.run([sys.executable, __file__, "one", str(m), str(nx), str(ny), op], capture_output=True,
                           text=True, timeout=300)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        print(line[0] if line else f"FAIL {m} {nx} {ny} {op}: {r.stderr.strip().splitlines()[-1:]}", flush=True)
