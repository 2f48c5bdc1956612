"""Profiling case for the NMG path: a few V-cycles of C2 (128^2, M=5, order 2,
4 levels) from the uniform Maxwellian, with per-cycle wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_13164_b200 import momg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = momg.Grid2D.uniform(128, 128)
ctx = momg.cavity_context(5, 2, knudsen=0.1, lid=0.1)
f = momg.uniform_field(g, 5, 1.0, (0.0, 0.0, 0.0), 1.0)
for it in range(n):
    t = time.perf_counter()
    momg.nmg_cycle(f, ctx, 4)
    momg.synchronize()
    print(f"cycle {it}: {(time.perf_counter() - t) * 1e3:.1f} ms")
