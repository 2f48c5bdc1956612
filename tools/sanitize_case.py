"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck): the
band kernels' shared-memory staging, named barriers and the relaxed-poll /
acquire / one-step-late release protocol.  k5_band: fused FS + residual on a
70 x 37 M=5 first-order field (3 bands, all 4 directions); k6_band: second
order with an FAS rhs on 40 x 34 (3 bands of 16); plus the transfer kernels.
Checks the results against the oracle so a sanitizer-perturbed schedule that
changes results fails too."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from helpers import BGK, SHAKHOV, Grid, Oracle, c5_field, cavity_ctx  # noqa: E402
from paper_2206_13164_b200 import momg  # noqa: E402
from test_gpu_parity import mctx, mgrid, rel_field, rel_res  # noqa: E402

O = Oracle("port")
M = 5
g = Grid.uniform(70, 37)
octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
c, p = c5_field(70, 37, M, seed=5)
f = momg.CellField.from_host(mgrid(g), M, c, p)
r = momg.fast_sweep_residual(f, mctx(octx))
gc, gp = f.download()
wc, wp, _ = O.fast_sweep(octx, g, c, p)
e1 = rel_field(gc, wc)
e2 = rel_res(r.download()[0], O.residual(octx, g, wc, wp))

g2 = Grid.uniform(40, 34)
octx2 = cavity_ctx(M, 2, SHAKHOV, kn=0.2, lid=0.1, prandtl=2.0 / 3.0)
c2, p2 = c5_field(40, 34, M, seed=6)
rh = (c2 * 1e-3, p2.copy())
f2 = momg.CellField.from_host(mgrid(g2), M, c2, p2)
rhs = momg.CellField.from_host(mgrid(g2), M, *rh)
momg.fast_sweep_step(f2, rhs, mctx(octx2))
wc2, _, _ = O.fast_sweep(octx2, g2, c2, p2, rhs=rh)
e3 = rel_field(f2.download()[0], wc2)
coarse = momg.restrict_solution(f2, mgrid(g2.coarsen()))
momg.fas_correct(f2, coarse, coarse)
momg.synchronize()
print(f"sanitize case: k5 sweep {e1:.2e} residual {e2:.2e} k6 sweep {e3:.2e}")
assert max(e1, e2, e3) < 1e-10
