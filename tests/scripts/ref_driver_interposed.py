"""Run the REFERENCE's own solve_steady (oracle/_ref/libmomg_ref.so, compiled
from its unmodified sources) in a process where
integration/_build/libmomg_gpu_interpose.so is preloaded, so its hot-path
calls resolve to the B200 (test helper of tests/test_gpu_dropin.py).
Usage: LD_PRELOAD=... python ref_driver_interposed.py OUT.npz"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from helpers import BGK, Grid, Oracle, cavity_ctx, uniform_field  # noqa: E402
from paper_2206_13164_b200 import momg  # noqa: E402

calls = ctypes.CDLL(None).momg_interpose_calls
calls.restype = ctypes.c_longlong
R = Oracle("reference")
out = {}
for name, (n, M, solver, levels) in {"c1": (32, 3, 1, 0), "nmg": (32, 5, 2, 3)}.items():
    g = Grid.uniform(n, n)
    octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    c, p = uniform_field(g, M)
    before, launches = calls(), momg.launch_count()
    wc, wp, rep = R.solve_steady(octx, g, c, p, solver=solver, tol=1e-8, levels=levels)
    out[f"{name}_coeffs"] = wc
    out[f"{name}_params"] = wp
    out[f"{name}_iterations"] = rep["iterations"]
    out[f"{name}_converged"] = rep["converged"]
    out[f"{name}_calls"] = calls() - before
    out[f"{name}_launches"] = momg.launch_count() - launches
np.savez(sys.argv[1], **out)
print({k: v for k, v in out.items() if np.ndim(v) == 0})
