"""The register-resident second-order / rhs band kernel (csrc/reg_band2.cuh,
k9_band: the default for exact second-order and FAS sweeps of M <= 5) against
the CPU oracle at 1e-10 and against the split kernel (k6_band) at rounding
level: fields of three and more 32-column bands with partial last bands (the
two-column halos between bands, the two columns of the next band), every
sweep direction first, both collision models, with and without a right-hand
side in its own basis, first order with rhs, a non-uniform grid (slope
denominators per cell), consecutive FS iterations, several iterations fused
in one launch through the NMG cycle, and perturbed schedules (MOMG_JITTER)
which must not change a single bit."""
import os

import numpy as np
import pytest

from helpers import BGK, SHAKHOV, Grid, Oracle, c5_field, cavity_ctx
from test_gpu_parity import mctx, mgrid, rel_field

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
O = Oracle("port")

CASES = [
    # (M, model, nx, ny, sweep order, with rhs, space order)
    (5, BGK, 100, 37, (0, 1, 2, 3), False, 2),
    (5, SHAKHOV, 70, 66, (2, 0, 3, 1), True, 2),
    (4, BGK, 97, 30, (1, 2, 3, 0), True, 2),
    (3, SHAKHOV, 130, 20, (3, 2, 1, 0), False, 2),
    (5, BGK, 66, 40, (3, 1, 0, 2), True, 1),
    (4, SHAKHOV, 33, 90, (0, 3, 2, 1), True, 1),
    # M = 6: the same kernel with 16-column bands and the flux in place in shared memory (BASELINE C4's order)
    (6, BGK, 50, 37, (0, 1, 2, 3), False, 2),
    (6, SHAKHOV, 40, 21, (2, 3, 0, 1), True, 2),
    (6, BGK, 35, 18, (1, 0, 3, 2), True, 1),
    (6, BGK, 20, 33, (3, 2, 1, 0), False, 1),
]


def _ctx(M, space, model):
    return cavity_ctx(M, space, model, kn=0.1, lid=0.1, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                      bottom_theta=1.3)


def _rhs(c, p):
    rp = p.copy()
    rp[:, 0] += 0.01
    rp[:, 3] *= 1.02
    return c * 1e-3, rp


@pytest.mark.parametrize("M,model,nx,ny,order,with_rhs,space", CASES)
def test_register_kernel2_parity(M, model, nx, ny, order, with_rhs, space):
    g = Grid.uniform(nx, ny)
    octx = _ctx(M, space, model)
    ctx = mctx(octx)
    c, p = c5_field(nx, ny, M, seed=nx * ny + M)
    rhs_h = _rhs(c, p) if with_rhs else None
    momg.set_band_kernel("register")
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rhs = momg.CellField.from_host(mgrid(g), M, *rhs_h) if with_rhs else None
    wc, wp = c, p
    for it in range(2):
        wc, wp, _ = O.fast_sweep(octx, g, wc, wp, rhs=rhs_h, sweep_order=list(order))
        momg.fast_sweep_step(f, rhs, ctx, None, order)
        gc, gp = f.download()
        assert rel_field(gc, wc) < 1e-10, f"iteration {it}"
        assert float(np.max(np.abs(gp - wp))) < 1e-10
    # the split kernel (16-column bands): same results to rounding
    momg.set_band_kernel("split")
    try:
        f2 = momg.CellField.from_host(mgrid(g), M, c, p)
        for it in range(2):
            momg.fast_sweep_step(f2, rhs, ctx, None, order)
        sc, sp_ = f2.download()
        assert rel_field(gc, sc) < 1e-12
        assert float(np.max(np.abs(gp - sp_))) < 1e-12
    finally:
        momg.set_band_kernel("register")


def test_register_kernel2_nonuniform_grid():
    """Cell sizes and centres that differ per cell: the slope denominators
    xc[i+1] - xc[i-1] and the offsets dx[i] / 2 of spatial.cpp:34-62."""
    M, nx, ny = 5, 72, 40
    rng = np.random.default_rng(5)
    dx = rng.uniform(0.6, 1.4, nx); dx /= dx.sum()
    dy = rng.uniform(0.6, 1.4, ny); dy /= dy.sum()
    xc = np.cumsum(dx) - 0.5 * dx
    yc = np.cumsum(dy) - 0.5 * dy
    g = Grid(nx, ny, 1.0, 1.0, dx, dy, xc, yc)
    octx = _ctx(M, 2, BGK)
    c, p = c5_field(nx, ny, M, seed=9)
    rhs_h = _rhs(c, p)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rhs = momg.CellField.from_host(mgrid(g), M, *rhs_h)
    momg.fast_sweep_step(f, rhs, mctx(octx))
    wc, wp, _ = O.fast_sweep(octx, g, c, p, rhs=rhs_h)
    gc, gp = f.download()
    assert rel_field(gc, wc) < 1e-10
    assert float(np.max(np.abs(gp - wp))) < 1e-10


def test_register_kernel2_under_jitter():
    M, nx, ny = 5, 130, 41
    g = Grid.uniform(nx, ny)
    ctx = mctx(_ctx(M, 2, SHAKHOV))
    c, p = c5_field(nx, ny, M, seed=3)
    rhs = momg.CellField.from_host(mgrid(g), M, *_rhs(c, p))

    def run():
        f = momg.CellField.from_host(mgrid(g), M, c, p)
        momg.fast_sweep_step(f, rhs, ctx)
        momg.fast_sweep_step(f, rhs, ctx, None, (2, 3, 0, 1))
        return f.download()

    want = run()
    try:
        for seed in (5, 6, 7):
            os.environ["MOMG_JITTER"] = str(seed)
            got = run()
            np.testing.assert_array_equal(got[0], want[0], err_msg=f"jitter {seed}")
            np.testing.assert_array_equal(got[1], want[1])
    finally:
        os.environ.pop("MOMG_JITTER", None)
