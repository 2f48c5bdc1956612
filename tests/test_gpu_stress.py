"""Race stress for the band kernels' inter-CTA protocol (relaxed polls, one
acquire once satisfied, one-step-late st.release publication, task claims in
(sweep, band) order).  compute-sanitizer is closed on this GPU pool, so the
protocol is exercised instead under perturbed schedules: MOMG_JITTER=<seed>
makes every task claim, publication and prefetch poll of k5_band / k6_band
sleep a pseudo-random 0-2 us, which reorders the CTAs against each other.
Any missing ordering would show up as a result that differs from the
unperturbed run; the exact Gauss-Seidel order makes every result bitwise
deterministic, so the check is array equality (and the oracle at 1e-10)."""
import os

import numpy as np
import pytest

from helpers import BGK, SHAKHOV, Grid, Oracle, c5_field, cavity_ctx
from test_gpu_parity import mctx, mgrid, rel_field

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
O = Oracle("port")


def _k5(g, octx, c, p):
    f = momg.CellField.from_host(mgrid(g), 5, c, p)
    r = momg.fast_sweep_residual(f, mctx(octx))
    return f.download() + r.download()


def _k6(g, octx, c, p, rh):
    f = momg.CellField.from_host(mgrid(g), 5, c, p)
    rhs = momg.CellField.from_host(mgrid(g), 5, *rh)
    momg.fast_sweep_step(f, rhs, mctx(octx), None, (2, 0, 3, 1))
    return f.download()


@pytest.fixture
def jitter():
    def set_seed(seed):
        if seed:
            os.environ["MOMG_JITTER"] = str(seed)
        else:
            os.environ.pop("MOMG_JITTER", None)
    yield set_seed
    os.environ.pop("MOMG_JITTER", None)


def test_band_protocol_under_jitter(jitter):
    g = Grid.uniform(100, 41)  # 4 bands of 32, partial last band
    octx = cavity_ctx(5, 1, BGK, kn=0.1, lid=0.1)
    c, p = c5_field(100, 41, 5, seed=31)
    g2 = Grid.uniform(56, 30)  # 4 bands of 16 (second order, radius-2 halos)
    octx2 = cavity_ctx(5, 2, SHAKHOV, kn=0.2, lid=0.1, prandtl=2.0 / 3.0)
    c2, p2 = c5_field(56, 30, 5, seed=32)
    rh = (c2 * 1e-3, p2.copy())
    jitter(0)
    base5 = _k5(g, octx, c, p)
    base6 = _k6(g2, octx2, c2, p2, rh)
    wc, _, _ = O.fast_sweep(octx, g, c, p)
    assert rel_field(base5[0], wc) < 1e-10
    for seed in range(1, 9):
        jitter(seed)
        got5 = _k5(g, octx, c, p)
        got6 = _k6(g2, octx2, c2, p2, rh)
        for a, b in zip(got5, base5):
            np.testing.assert_array_equal(a, b, err_msg=f"k5_band, jitter seed {seed}")
        for a, b in zip(got6, base6):
            np.testing.assert_array_equal(a, b, err_msg=f"k6_band, jitter seed {seed}")
