"""The register-resident band kernel (csrc/reg_band.cuh, the default for
first-order exact sweeps and residuals of M <= 5) against the CPU oracle at
1e-10 and against the split band kernel (k5_band) at rounding level, on
multi-band fields with partial last bands, both collision models, consecutive
FS iterations, the fused
sweep + residual against the separate calls, and perturbed schedules (MOMG_JITTER) which must not change
a single bit."""
import os

import numpy as np
import pytest

from helpers import BGK, SHAKHOV, Grid, Oracle, c5_field, cavity_ctx
from test_gpu_parity import mctx, mgrid, rel_field, rel_res

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
O = Oracle("port")

CASES = [
    # (M, model, nx, ny, sweep order)
    (5, BGK, 100, 37, (0, 1, 2, 3)),
    (5, SHAKHOV, 70, 66, (2, 0, 3, 1)),
    (4, BGK, 33, 90, (1, 2, 3, 0)),
    (3, SHAKHOV, 96, 20, (3, 2, 1, 0)),
]


def _ctx(M, model):
    return cavity_ctx(M, 1, model, kn=0.1, lid=0.1, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                      bottom_theta=1.3)


@pytest.mark.parametrize("M,model,nx,ny,order", CASES)
def test_register_kernel_sweep_and_residual(M, model, nx, ny, order):
    g = Grid.uniform(nx, ny)
    octx = _ctx(M, model)
    ctx = mctx(octx)
    c, p = c5_field(nx, ny, M, seed=nx * ny + M)
    momg.set_band_kernel("register")
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    r = momg.fast_sweep_residual(f, ctx, None, None, order)
    gc, gp = f.download()
    rc, rp = r.download()
    wc, wp, _ = O.fast_sweep(octx, g, c, p, sweep_order=list(order))
    assert rel_field(gc, wc) < 1e-10
    assert float(np.max(np.abs(gp - wp))) < 1e-10
    assert rel_res(rc, O.residual(octx, g, wc, wp)) < 1e-10
    np.testing.assert_array_equal(rp, gp)
    # the split kernel: same results to rounding
    momg.set_band_kernel("split")
    try:
        f2 = momg.CellField.from_host(mgrid(g), M, c, p)
        r2 = momg.fast_sweep_residual(f2, ctx, None, None, order)
        sc, sp_ = f2.download()
        assert rel_field(gc, sc) < 1e-13
        assert rel_res(rc, r2.download()[0]) < 1e-12
    finally:
        momg.set_band_kernel("register")


def test_register_kernel_consecutive_sweeps_and_separate_calls():
    """fast_sweep_step then residual == the fused launch, bitwise; three
    consecutive FS iterations against the oracle's at 1e-10."""
    M, nx, ny = 5, 96, 45
    g = Grid.uniform(nx, ny)
    octx = _ctx(M, BGK)
    ctx = mctx(octx)
    c, p = c5_field(nx, ny, M, seed=11)
    f1 = momg.CellField.from_host(mgrid(g), M, c, p)
    momg.fast_sweep_step(f1, None, ctx)
    r1 = momg.residual(f1, ctx)
    f2 = momg.CellField.from_host(mgrid(g), M, c, p)
    r2 = momg.fast_sweep_residual(f2, ctx)
    np.testing.assert_array_equal(f1.download()[0], f2.download()[0])
    np.testing.assert_array_equal(r1.download()[0], r2.download()[0])
    wc, wp, _ = O.fast_sweep(octx, g, c, p)
    for _ in range(2):
        momg.fast_sweep_step(f1, None, ctx)
        wc, wp, _ = O.fast_sweep(octx, g, wc, wp)
    assert rel_field(f1.download()[0], wc) < 1e-10


def test_register_kernel_under_jitter():
    M, nx, ny = 5, 160, 41
    g = Grid.uniform(nx, ny)
    ctx = mctx(_ctx(M, SHAKHOV))
    c, p = c5_field(nx, ny, M, seed=3)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    r = momg.fast_sweep_residual(f, ctx)
    want, wres = f.download(), r.download()
    try:
        for seed in (5, 6, 7):
            os.environ["MOMG_JITTER"] = str(seed)
            f = momg.CellField.from_host(mgrid(g), M, c, p)
            r = momg.fast_sweep_residual(f, ctx)
            got = f.download()
            np.testing.assert_array_equal(got[0], want[0], err_msg=f"jitter {seed}")
            np.testing.assert_array_equal(got[1], want[1])
            np.testing.assert_array_equal(r.download()[0], wres[0])
    finally:
        os.environ.pop("MOMG_JITTER", None)
