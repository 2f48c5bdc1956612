"""Small, fixed profiling case for ncu: residual (Jacobi) on nr x nr and one
persistent FS iteration on ns x ns, M=5 order 1, C5-style field."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_13164_b200 import momg  # noqa: E402
from paper_2206_13164_b200.synthetic import c5_field  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nr", type=int, default=512)
ap.add_argument("--ns", type=int, default=256)
ap.add_argument("--M", type=int, default=5)
ap.add_argument("--order", type=int, default=1)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
ctx = momg.cavity_context(a.M, a.order, knudsen=0.1, lid=0.0)
for n, what in ((a.nr, "residual"), (a.ns, "sweep")):
    g = momg.Grid2D.uniform(n, n)
    c, p = c5_field(n, n, a.M, seed=1)
    f = momg.CellField.from_host(g, a.M, c, p)
    for _ in range(a.reps):
        if what == "residual":
            momg.residual(f, ctx)
        else:
            momg.fast_sweep_step(f, None, ctx)
momg.synchronize()
print("done", momg.launch_count())
