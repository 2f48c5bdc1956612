"""Strip-partitioned NMG on one GPU (the ranks emulated in one process,
paper_2206_13164_b200/strips.py StripSolver): the finest level in 2 / 4
column strips (band sweeps over the partition, second order included),
coarse levels gathered on every rank, the coarse cycle replicated, FAS back
into the strips.  Against the single-field device solve: the first V-cycles
field by field at 1e-10, the whole solve in iterations (+-1) and macroscopic
fields (1e-8); against the oracle through the single-field solve's own
parity tests."""
import numpy as np
import pytest

from helpers import BGK, SHAKHOV, Grid, cavity_ctx, uniform_field
from test_gpu_parity import macro, mctx, mgrid, rel_field

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
strips = pytest.importorskip("paper_2206_13164_b200.strips")


def _setup(M, order, model, n, ranks, levels):
    g = Grid.uniform(n, n)
    octx = cavity_ctx(M, order, model, kn=0.1, lid=0.1, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0)
    ctx = mctx(octx)
    c, p = uniform_field(g, M)
    solver = strips.StripSolver(momg, mgrid(g), M, strips.StripComm(), levels, emulate_ranks=ranks)
    solver.fine.upload(c, p)
    single = momg.CellField.from_host(mgrid(g), M, c, p)
    return g, ctx, solver, single


@pytest.mark.parametrize("M,order,model,n,ranks,levels", [(5, 2, BGK, 128, 2, 3), (3, 1, SHAKHOV, 128, 2, 2),
                                                          (4, 2, BGK, 256, 4, 3)])
def test_strip_vcycles_match_single_field(M, order, model, n, ranks, levels):
    g, ctx, solver, single = _setup(M, order, model, n, ranks, levels)
    for it in range(2):
        solver.cycle(ctx)
        momg.nmg_cycle(single, ctx, levels)
        got_c, got_p = solver.fine.set.download()
        want_c, want_p = single.download()
        assert rel_field(got_c, want_c) < 1e-10, f"cycle {it}"
        assert np.max(np.abs(got_p - want_p)) < 1e-10


def test_strip_nmg_solve_c2():
    """C2 (128^2, M=5, second order, NMG over 4 levels) to 1e-8 on 2 strips."""
    M, levels = 5, 4
    g, ctx, solver, single = _setup(M, 2, BGK, 128, 2, levels)
    conv, iters, hist = solver.solve(ctx, 1e-8)
    rep = momg.solve_steady(single, ctx, momg.SolverOptions(momg.SolverKind.nmg, 1e-8, 0, levels))
    assert conv and rep.converged and abs(iters - rep.iterations) <= 1
    # ratios agree to ~1e-12 early; near 1e-8 the residual is a difference of
    # O(1) states, so its relative rounding grows like 1e-16 / ratio
    for it, (a, b) in enumerate(zip(hist, rep.history)):
        assert abs(a - b) <= 1e-8 * b + 1e-14, f"iteration {it + 1}: {a} vs {b}"
    gc, gp = solver.fine.set.download()
    wc, wp = single.download()
    mg, mw = macro(gc, gp), macro(wc, wp)
    assert np.max(np.abs(mg - mw)) <= 1e-8 * np.max(np.abs(mw))
