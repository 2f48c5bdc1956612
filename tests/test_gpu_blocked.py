"""Blocked-parallel fast sweeping (SolveContext.threads = T > 1), the
reference's threads > 1 path (single_level.cpp:130-161): T workers sweep
contiguous blocks [nx b / T, nx (b+1) / T) of the outer i loop concurrently,
so a block's reads of its neighbour blocks' boundary columns see either
version.  The device realises it deterministically as the outcome of workers
at equal pace: a block sees the block upstream in the sweep direction OLD
and the block downstream NEW (i ascending: blocks visited T-1 .. 0, each
i-ascending; i descending: blocks 0 .. T-1, each i-descending).  The oracle
runs exactly that serial order with its own sweep_cell (sweep_cells), and
the device must match it at the per-sweep tolerance; blocks that do not fall
on 32-column band boundaries run the exact order (the outcome of workers
finishing in block order), which the oracle's plain fast_sweep_step gives."""
import numpy as np
import pytest

from helpers import BGK, SHAKHOV, Grid, Oracle, c5_field, cavity_ctx
from test_gpu_parity import mctx, mgrid, rel_field, rel_res

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
O = Oracle("port")
KS = [(True, True), (False, True), (False, False), (True, False)]  # kSweepDirs, single_level.cpp:116-117


def blocked_cells(nx, ny, T, s):
    i_up, j_up = KS[s]
    lo = [nx * b // T for b in range(T + 1)]
    cells = []
    for b in (range(T - 1, -1, -1) if i_up else range(T)):
        cols = range(lo[b], lo[b + 1]) if i_up else range(lo[b + 1] - 1, lo[b] - 1, -1)
        for i in cols:
            for j in (range(ny) if j_up else range(ny - 1, -1, -1)):
                cells.append((i, j))
    return cells


def oracle_blocked_sweep(octx, g, c, p, T, order, rhs=None):
    c, p = c.copy(), p.copy()
    for s in order:
        O.sweep_cells(octx, g, c, p, blocked_cells(g.nx, g.ny, T, s), rhs=rhs)
    return c, p


@pytest.mark.parametrize("M,model,nx,ny,T,order", [
    (5, BGK, 128, 37, 2, (0, 1, 2, 3)),
    (5, SHAKHOV, 128, 40, 4, (2, 0, 3, 1)),
    (4, BGK, 192, 33, 3, (1, 2, 3, 0)),
    (3, BGK, 96, 50, 3, (3, 2, 1, 0)),
])
def test_blocked_sweep_matches_blocked_order(M, model, nx, ny, T, order):
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, 1, model, kn=0.1, lid=0.1, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0)
    ctx = mctx(octx)
    ctx.threads = T
    c, p = c5_field(nx, ny, M, seed=nx + T)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    wc, wp = c, p
    for it in range(2):
        wc, wp = oracle_blocked_sweep(octx, g, wc, wp, T, order)
        momg.fast_sweep_step(f, None, ctx, None, order)
        gc, gp = f.download()
        assert rel_field(gc, wc) < 1e-10, f"iteration {it}"
        assert np.max(np.abs(gp - wp)) < 1e-10
    # the blocked order really differs from the exact one
    ec, _, _ = O.fast_sweep(octx, g, c, p, sweep_order=list(order))
    assert rel_field(oracle_blocked_sweep(octx, g, c, p, T, order)[0], ec) > 1e-8
    # fused with the residual (nmg_cycle's sequence)
    f2 = momg.CellField.from_host(mgrid(g), M, c, p)
    r = momg.fast_sweep_residual(f2, ctx, None, None, order)
    bc, bp = oracle_blocked_sweep(octx, g, c, p, T, order)
    assert rel_field(f2.download()[0], bc) < 1e-10
    assert rel_res(r.download()[0], O.residual(octx, g, bc, bp)) < 1e-10


def test_unaligned_blocks_run_the_exact_order():
    nx, ny, T, M = 100, 20, 3, 4
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    ctx = mctx(octx)
    ctx.threads = T
    c, p = c5_field(nx, ny, M, seed=5)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    momg.fast_sweep_step(f, None, ctx)
    wc, wp, _ = O.fast_sweep(octx, g, c, p)
    assert rel_field(f.download()[0], wc) < 1e-10


def test_blocked_sweep_jitter():
    import os
    nx, ny, T, M = 128, 33, 4, 5
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    ctx = mctx(octx)
    ctx.threads = T
    c, p = c5_field(nx, ny, M, seed=9)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    momg.fast_sweep_step(f, None, ctx)
    want = f.download()
    try:
        for seed in (3, 4):
            os.environ["MOMG_JITTER"] = str(seed)
            f = momg.CellField.from_host(mgrid(g), M, c, p)
            momg.fast_sweep_step(f, None, ctx)
            got = f.download()
            np.testing.assert_array_equal(got[0], want[0])
            np.testing.assert_array_equal(got[1], want[1])
    finally:
        os.environ.pop("MOMG_JITTER", None)


@pytest.mark.parametrize("M,model,nx,ny,T,order,with_rhs", [
    (5, BGK, 64, 30, 2, (0, 1, 2, 3), False),
    (5, SHAKHOV, 96, 25, 3, (2, 0, 3, 1), True),
    (4, BGK, 128, 20, 4, (1, 2, 3, 0), True),
    (3, BGK, 64, 33, 4, (3, 2, 1, 0), False),
])
def test_blocked_second_order_and_rhs(M, model, nx, ny, T, order, with_rhs):
    """The 16-column second-order / rhs band kernel in blocked mode (2-column
    halos: a block start reads both OLD, a block end the next two NEW)."""
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, 2, model, kn=0.2, lid=0.1, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0)
    ctx = mctx(octx)
    ctx.threads = T
    c, p = c5_field(nx, ny, M, seed=nx + 7 * T)
    rhs_h = None
    if with_rhs:
        rp = p.copy(); rp[:, 0] += 0.01; rp[:, 3] *= 1.02
        rhs_h = (c * 1e-3, rp)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rhs = momg.CellField.from_host(mgrid(g), M, *rhs_h) if with_rhs else None
    wc, wp = c, p
    for it in range(2):
        wc, wp = oracle_blocked_sweep(octx, g, wc, wp, T, order, rhs=rhs_h)
        momg.fast_sweep_step(f, rhs, ctx, None, order)
        gc, gp = f.download()
        assert rel_field(gc, wc) < 1e-10, f"iteration {it}"
        assert np.max(np.abs(gp - wp)) < 1e-10
