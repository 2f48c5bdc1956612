"""ES-BGK (anisotropic Gaussian, collision.hpp:52-71, 84-94) on the device
against the oracle: residual and two consecutive FS iterations for M = 3..8,
first and second order, with and without an FAS rhs, fields with a visible
stress (so the Gaussian's coefficients are far from the Maxwellian's); the
NonSpdTensor branch; an NMG solve to 1e-8 (iterations +-1, macroscopic fields
1e-8).  The band kernels (M <= 5) hand ES-BGK to the thread-per-face kernels,
M = 7, 8 run the warp-per-cell kernels."""
import numpy as np
import pytest

from helpers import ES_BGK, Grid, Oracle, cavity_ctx, smooth_field, uniform_field
from oracle.api import MO_NON_SPD, OracleError
from test_gpu_parity import macro, mctx, mgrid, rel_field, rel_res

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
O = Oracle("port")
TOL = 1e-10


def stressed_field(g, M, seed):
    c, p = smooth_field(g, M, seed=seed, amp=0.08, uz=True)
    rng = np.random.default_rng(seed)
    s = rng.uniform(-1, 1, (g.cells, 5)) * 0.03
    c[:, 5], c[:, 6], c[:, 8] = s[:, 0], s[:, 1], s[:, 2]       # e_x+e_y, e_x+e_z, e_y+e_z
    c[:, 4], c[:, 7] = s[:, 3], s[:, 4]                        # 2e_x, 2e_y
    c[:, 9] = -(c[:, 4] + c[:, 7])                             # trace 0: Grad-normalized
    return c, p


CASES = [
    # (M, order, nx, ny, with rhs)
    (3, 1, 9, 7, False),
    (4, 2, 8, 9, True),
    (5, 1, 40, 12, False),
    (5, 2, 12, 10, True),
    (6, 2, 7, 6, False),
    (7, 1, 6, 5, True),
    (8, 2, 5, 6, False),
]


@pytest.mark.parametrize("M,order,nx,ny,with_rhs", CASES)
def test_es_bgk_residual_and_sweeps(M, order, nx, ny, with_rhs):
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, order, ES_BGK, kn=0.2, prandtl=2.0 / 3.0, bottom_theta=1.2)
    c, p = stressed_field(g, M, seed=7 * M + order)
    ctx = mctx(octx)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    got, gp = momg.residual(f, ctx).download()
    assert rel_res(got, O.residual(octx, g, c, p)) < TOL
    np.testing.assert_array_equal(gp, p)
    rhs_h = None
    if with_rhs:
        rp = p.copy(); rp[:, 0] += 0.01; rp[:, 3] *= 1.02
        rhs_h = (c * 1e-3, rp)
    rhs = momg.CellField.from_host(mgrid(g), M, *rhs_h) if with_rhs else None
    wc, wp = c, p
    for it in range(2):
        wc, wp, _ = O.fast_sweep(octx, g, wc, wp, rhs=rhs_h)
        momg.fast_sweep_step(f, rhs, ctx)
        gc, gpp = f.download()
        assert rel_field(gc, wc) < TOL, f"iteration {it}"
        assert np.max(np.abs(gpp - wp)) < TOL


def test_es_bgk_non_spd():
    """Pr = 0.2 (1 - 1/Pr = -4) and a cell with a large normal stress: Lambda
    has a negative eigenvalue -> NonSpdTensor (collision.hpp:88-92)."""
    M = 4
    g = Grid.uniform(6, 5)
    octx = cavity_ctx(M, 1, ES_BGK, kn=0.2, prandtl=0.2)
    c, p = smooth_field(g, M, seed=3)
    c[13, 4], c[13, 7], c[13, 9] = 0.3, -0.15, -0.15
    with pytest.raises(OracleError) as e:
        O.residual(octx, g, c, p)
    assert e.value.code == MO_NON_SPD
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    with pytest.raises(momg.NonSpdTensor):
        momg.residual(f, mctx(octx))
    with pytest.raises(momg.NonSpdTensor):
        momg.fast_sweep_step(f, None, mctx(octx))


def test_es_bgk_nmg_solve():
    M = 3
    g = Grid.uniform(16, 16)
    octx = cavity_ctx(M, 1, ES_BGK, kn=0.1, lid=0.1, prandtl=2.0 / 3.0)
    c, p = uniform_field(g, M)
    wc, wp, wr = O.solve_steady(octx, g, c, p, solver=2, tol=1e-8, levels=2)
    assert wr["converged"]
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rep = momg.solve_steady(f, mctx(octx), momg.SolverOptions(momg.SolverKind.nmg, 1e-8, 0, 2))
    assert rep.converged and abs(rep.iterations - wr["iterations"]) <= 1
    gc, gp = f.download()
    mg, mw = macro(gc, gp), macro(wc, wp)
    assert np.max(np.abs(mg - mw)) <= 1e-8 * np.max(np.abs(mw))
