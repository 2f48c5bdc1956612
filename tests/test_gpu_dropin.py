"""The drop-in boundary under the reference's UNMODIFIED driver: the
reference library (oracle/_ref, built from its own sources) runs its own
solve_steady / nmg_cycle (multigrid.cpp:166-320) in a process where
integration/_build/libmomg_gpu_interpose.so is preloaded; ELF interposition
sends its residual, fast_sweep_step, mass, restriction, FAS and norm calls
to the B200 (integration/momg_gpu_interpose.cpp).  Checked against the
oracle: C1 (BASELINE configs[0], 32^2 M=3 FS) and a 32^2 M=5 NMG solve over 3
levels -- iteration counts within +-1, macroscopic fields at 1e-8 -- and that
the calls really went through the interposer and launched kernels."""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import BGK, HAVE_REF, Grid, Oracle, cavity_ctx, uniform_field
from test_gpu_parity import macro

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "integration", "_build", "libmomg_gpu_interpose.so")


def test_reference_driver_interposed(tmp_path):
    assert HAVE_REF and os.path.exists(LIB), "build(): make -C oracle ref bridge"
    out = tmp_path / "r.npz"
    env = dict(os.environ, LD_PRELOAD=LIB)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "scripts", "ref_driver_interposed.py"),
                        str(out)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    z = np.load(out)
    O = Oracle("port")
    for name, (n, M, solver, levels) in {"c1": (32, 3, 1, 0), "nmg": (32, 5, 2, 3)}.items():
        assert bool(z[f"{name}_converged"])
        assert int(z[f"{name}_calls"]) > 0 and int(z[f"{name}_launches"]) > 0
        g = Grid.uniform(n, n)
        octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
        c, p = uniform_field(g, M)
        wc, wp, wr = O.solve_steady(octx, g, c, p, solver=solver, tol=1e-8, levels=levels)
        assert abs(int(z[f"{name}_iterations"]) - wr["iterations"]) <= 1
        mg, mw = macro(z[f"{name}_coeffs"], z[f"{name}_params"]), macro(wc, wp)
        assert np.max(np.abs(mg - mw)) <= 1e-8 * np.max(np.abs(mw))
