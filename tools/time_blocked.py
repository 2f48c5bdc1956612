"""FS iteration (+ residual) time at 2048^2 (C5 field) for SolveContext.threads
= 1 (exact order) and T > 1 (blocked-parallel, band-aligned blocks)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_13164_b200 import momg  # noqa: E402
from paper_2206_13164_b200.synthetic import c5_field  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
g = momg.Grid2D.uniform(n, n)
c, p = c5_field(n, n, 5, seed=1)
for T in (1, 2, 4, 8, 16, 64):
    ctx = momg.cavity_context(5, 1, knudsen=0.1, lid=0.0)
    ctx.threads = T
    f = momg.CellField.from_host(g, 5, c, p)
    out = momg.CellField(g, 5)
    momg.fast_sweep_residual(f, ctx, out)
    momg.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        momg.fast_sweep_residual(f, ctx, out)
    momg.synchronize()
    print(f"threads={T}: {(time.perf_counter() - t) / 3 * 1e3:.1f} ms per FS iteration + residual", flush=True)
