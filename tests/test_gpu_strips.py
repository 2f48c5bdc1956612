"""Strip-partitioned multi-GPU path on one GPU: every
strip of a momg_strips partition owned by this process, so one launch runs
all ranks' band tasks over all ranks' separately allocated strips (the
emulation of the ranks as one kernel the profiling guide prescribes).  The
cross-strip halo cells and counters are read in the neighbouring strip's
memory exactly as a peer rank's would be over NVLink.  Required: bitwise
equality with the single-field fused FS + residual (and, through it, the
oracle), over consecutive calls (counter epochs), several strip layouts,
sweep orders and schedule perturbations.  The strip partition runs the split
band kernel (k5_band's strips variant), so the single-field reference here
runs the split kernel too (momg.set_band_kernel("split")); the default
register-resident kernel agrees with it to rounding (test_gpu_rb.py)."""
import os

import numpy as np
import pytest

from helpers import BGK, SHAKHOV, Grid, Oracle, c5_field, cavity_ctx
from test_gpu_parity import mctx, mgrid, rel_field, rel_res

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")


@pytest.fixture(autouse=True)
def split_band_kernel():
    momg.set_band_kernel("split")
    yield
    momg.set_band_kernel("register")

CASES = [
    # (M, model, nx, ny, bounds, sweep order)
    (5, BGK, 128, 70, (0, 64, 128), (0, 1, 2, 3)),
    (5, SHAKHOV, 192, 45, (0, 32, 96, 160, 192), (2, 0, 3, 1)),
    (4, BGK, 256, 33, tuple(range(0, 257, 32)), (1, 2, 3, 0)),
    (3, SHAKHOV, 96, 64, (0, 64, 96), (3, 2, 1, 0)),
]


@pytest.mark.parametrize("M,model,nx,ny,bounds,order", CASES)
def test_strips_match_single_field(M, model, nx, ny, bounds, order):
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, 1, model, kn=0.1, lid=0.1, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                      bottom_theta=1.2)
    ctx = mctx(octx)
    c, p = c5_field(nx, ny, M, seed=nx + ny + M)
    single = momg.CellField.from_host(mgrid(g), M, c, p)
    st = momg.StripSet(mgrid(g), M, bounds)
    st.upload(c, p)
    work = momg.WorkStats()
    for it in range(2):  # consecutive launches: the counters continue from the epoch
        r1 = momg.fast_sweep_residual(single, ctx, None, None, order)
        st.fast_sweep_residual(ctx, order, work)
        a, b = single.download()
        sa, sb = st.download()
        np.testing.assert_array_equal(sa, a, err_msg=f"iteration {it}")
        np.testing.assert_array_equal(sb, b)
        ra, rb = r1.download()
        sra, srb = st.download(residual=True)
        np.testing.assert_array_equal(sra, ra)
        np.testing.assert_array_equal(srb, rb)
        if it == 0:
            wc, wp, _ = Oracle("port").fast_sweep(octx, g, c, p, sweep_order=list(order))
            assert rel_field(sa, wc) < 1e-10
            assert rel_res(sra, Oracle("port").residual(octx, g, wc, wp)) < 1e-10
    assert work.cell_evals == 2 * 4 * nx * ny


def test_strips_under_jitter():
    M, nx, ny = 5, 160, 41
    g = Grid.uniform(nx, ny)
    ctx = mctx(cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1))
    c, p = c5_field(nx, ny, M, seed=3)
    single = momg.CellField.from_host(mgrid(g), M, c, p)
    momg.fast_sweep_residual(single, ctx)
    want = single.download()
    try:
        for seed in (5, 6, 7):
            os.environ["MOMG_JITTER"] = str(seed)
            st = momg.StripSet(mgrid(g), M, (0, 32, 64, 128, 160))
            st.upload(c, p)
            st.fast_sweep_residual(ctx)
            got = st.download()
            np.testing.assert_array_equal(got[0], want[0], err_msg=f"jitter {seed}")
            np.testing.assert_array_equal(got[1], want[1])
    finally:
        os.environ.pop("MOMG_JITTER", None)


def test_strips_argument_checks():
    g = momg.Grid2D.uniform(96, 16)
    with pytest.raises(ValueError):  # MOMG_ERR_ARG
        momg.StripSet(g, 5, (0, 40, 96))  # width not a multiple of 32
    with pytest.raises(ValueError):
        momg.StripSet(momg.Grid2D.uniform(90, 16), 5, (0, 90))
    st = momg.StripSet(g, 5, (0, 32, 96), first=0, last=0)  # rank 0 of 2, peer not attached
    with pytest.raises(ValueError, match="not attached"):
        st.fast_sweep_residual(momg.cavity_context(5, 1))
    with pytest.raises(momg.ConfigError):
        momg.StripSet(g, 5, (0, 32, 96)).fast_sweep_residual(momg.cavity_context(5, 2))  # second order
