"""Profiling case for the band sweep: one FS iteration on an nx x ny grid
(default one band, 32 x 1024, so every sampled warp is on the step loop)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_13164_b200 import momg  # noqa: E402
from paper_2206_13164_b200.synthetic import c5_field  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=32)
ap.add_argument("--ny", type=int, default=1024)
ap.add_argument("--M", type=int, default=5)
ap.add_argument("--order", type=int, default=1)
a = ap.parse_args()
ctx = momg.cavity_context(a.M, a.order, knudsen=0.1, lid=0.0)
g = momg.Grid2D.uniform(a.nx, a.ny)
c, p = c5_field(a.nx, a.ny, a.M, seed=1)
f = momg.CellField.from_host(g, a.M, c, p)
momg.fast_sweep_step(f, None, ctx)
momg.synchronize()
print("done")
