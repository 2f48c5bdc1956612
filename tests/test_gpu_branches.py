"""GPU parity for the branches and operators the round-1 suite did not force:
the supersonic HLL branches of face_flux (flux.cpp:91-92), the nonphysical
reconstruction fallback of second-order face states (spatial.cpp:53-60,
76-78), residual_scale (multigrid.cpp:224-239), the Euler smoother
(single_level.cpp:31-38, 74-97) with and without an rhs, and the Euler solver
of solve_steady.  Same tolerances as test_gpu_parity.py."""
import numpy as np
import pytest

from helpers import BGK, ES_BGK, SHAKHOV, Grid, Oracle, cavity_ctx, smooth_field, uniform_field
from oracle.api import MO_NONPHYSICAL_STATE, OracleError
from test_gpu_parity import macro, mctx, mgrid, rel_field, rel_res

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
O = Oracle("port")
TOL = 1e-10


def supersonic_field(g, M, seed, c_bound):
    """Interior jets faster than the HLL signal bound: u_x > C sqrt(theta) in
    the middle columns (lambda_- >= 0: full flux of the left state) and
    u_y < -C sqrt(theta) in the middle rows (lambda_+ <= 0: full flux of the
    right state); slow near the walls so the wall fluxes stay physical."""
    c, p = smooth_field(g, M, seed=seed, amp=0.05, uz=True)
    x = np.tile(g.xc, g.ny)
    y = np.repeat(g.yc, g.nx)
    a = 1.35 * c_bound
    p[:, 0] += a * np.sin(np.pi * x) ** 2 * np.sin(np.pi * y)
    p[:, 1] -= a * np.sin(np.pi * y) ** 2 * np.sin(np.pi * x)
    return c, p


def _supersonic_faces(g, p, cb):
    P = p.reshape(g.ny, g.nx, 4)
    sx = ((P[:, :-1, 0] - cb * np.sqrt(P[:, :-1, 3]) >= 0) & (P[:, 1:, 0] - cb * np.sqrt(P[:, 1:, 3]) >= 0)).sum()
    sy = ((P[:-1, :, 1] + cb * np.sqrt(P[:-1, :, 3]) <= 0) & (P[1:, :, 1] + cb * np.sqrt(P[1:, :, 3]) <= 0)).sum()
    return int(sx), int(sy)


@pytest.mark.parametrize("M,order,nx,ny", [(5, 1, 70, 36), (5, 2, 40, 36), (3, 1, 40, 20), (4, 2, 36, 34),
                                           (6, 2, 24, 20), (8, 1, 20, 18)])
def test_supersonic_hll_branches(M, order, nx, ny):
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, order, BGK, kn=0.3)
    c, p = supersonic_field(g, M, 4 + M, octx.c_bound)
    sx, sy = _supersonic_faces(g, p, octx.c_bound)
    assert sx > 0 and sy > 0  # both full-flux branches are taken
    ctx = mctx(octx)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    got, _ = momg.residual(f, ctx).download()
    assert rel_res(got, O.residual(octx, g, c, p)) < TOL
    try:
        wc, wp, _ = O.fast_sweep(octx, g, c, p)
    except OracleError as e:
        # the reference aborts this sweep (e.g. wall_flux: nonpositive wall
        # density once the jet has been swept into a wall cell): the device
        # must raise the same exception class
        assert e.code == MO_NONPHYSICAL_STATE, e
        with pytest.raises(momg.NonphysicalState):
            momg.fast_sweep_step(f, None, ctx)
        return
    momg.fast_sweep_step(f, None, ctx)
    gc, gp = f.download()
    assert rel_field(gc, wc) < TOL and np.max(np.abs(gp - wp)) < TOL


@pytest.mark.parametrize("M,nx,ny,with_rhs", [(3, 20, 14, False), (5, 40, 18, True), (6, 12, 10, False)])
def test_reconstruction_fallback(M, nx, ny, with_rhs):
    """Second order with temperature jumps large enough that the limited
    face temperature goes nonpositive (spatial.cpp:76-78): those faces fall
    back to the cell state (safe_face_state, :53-60)."""
    g = Grid.uniform(nx, ny)
    octx = cavity_ctx(M, 2, BGK, kn=0.3)
    c, p = smooth_field(g, M, seed=9 + M, amp=0.05)
    rng = np.random.default_rng(3 + M)
    p[:, 3] = np.where(rng.random(g.cells) < 0.3, 0.08, 1.0 + rng.random(g.cells))
    T = p[:, 3].reshape(ny, nx)
    h = g.xc[2] - g.xc[0]
    s = (T[:, 2:] - T[:, :-2]) / h
    nonpos = ((T[:, 1:-1] + 0.5 * g.dx[0] * s <= 0) | (T[:, 1:-1] - 0.5 * g.dx[0] * s <= 0)).sum()
    assert nonpos > 0
    ctx = mctx(octx)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    got, _ = momg.residual(f, ctx).download()
    assert rel_res(got, O.residual(octx, g, c, p)) < TOL
    rhs_h = (c * 1e-3, p.copy()) if with_rhs else None
    rhs = momg.CellField.from_host(mgrid(g), M, *rhs_h) if with_rhs else None
    wc, wp, _ = O.fast_sweep(octx, g, c, p, rhs=rhs_h)
    momg.fast_sweep_step(f, rhs, ctx)
    gc, gp = f.download()
    assert rel_field(gc, wc) < TOL and np.max(np.abs(gp - wp)) < TOL


def residual_scale_ref(g, c, p, octx):
    """multigrid.cpp:224-239 restated: max rho (C sqrt(theta)(1/dx + 1/dy) + nu),
    nu = beta sqrt(pi/2)/Kn rho theta^(1-w) (collision.hpp:36-44)."""
    beta = octx.prandtl if octx.collision == ES_BGK else 1.0
    rho = c[:, 0]
    th = p[:, 3]
    nu = beta * np.sqrt(np.arctan(1.0) * 2.0) / octx.knudsen * rho * th ** (1.0 - octx.viscosity_index)
    dx = np.tile(g.dx, g.ny)
    dy = np.repeat(g.dy, g.nx)
    return float(np.max(rho * (octx.cfl_c_bound * np.sqrt(th) * (1.0 / dx + 1.0 / dy) + nu)))


@pytest.mark.parametrize("M,model", [(3, BGK), (5, SHAKHOV), (4, ES_BGK)])
def test_residual_scale(M, model):
    g = Grid.uniform(23, 17, 1.0, 0.8)
    octx = cavity_ctx(M, 1, model, kn=0.2, prandtl=2.0 / 3.0 if model != BGK else 1.0)
    c, p = smooth_field(g, M, seed=21, amp=0.2)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    want = residual_scale_ref(g, c, p, octx)
    assert momg.residual_scale(f, mctx(octx)) == pytest.approx(want, rel=1e-14)


EULER_CASES = [
    # (M, order, model, nx, ny, with rhs)
    (3, 1, BGK, 9, 7, False),
    (4, 2, SHAKHOV, 8, 8, True),
    (5, 1, BGK, 12, 9, True),
    (5, 2, SHAKHOV, 7, 6, False),
    (6, 2, BGK, 6, 5, True),
    (7, 1, BGK, 5, 6, False),
    (8, 2, SHAKHOV, 5, 5, True),
]


@pytest.mark.parametrize("M,order,model,nx,ny,with_rhs", EULER_CASES)
def test_euler_step_parity(M, order, model, nx, ny, with_rhs):
    g = Grid.uniform(nx, ny, 1.0, 1.1)
    octx = cavity_ctx(M, order, model, kn=0.3, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                      bottom_theta=1.3)
    c, p = smooth_field(g, M, seed=40 + M, amp=0.08, uz=True)
    rhs_h = None
    if with_rhs:
        rp = p.copy(); rp[:, 1] += 0.01; rp[:, 3] *= 1.03
        rhs_h = (c * 1e-3, rp)
    wc, wp = O.euler_step(octx, g, c, p, rhs=rhs_h)
    ctx = mctx(octx)
    # residuals evaluated inside, and passed explicitly (solve_steady's use)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rhs = momg.CellField.from_host(mgrid(g), M, *rhs_h) if with_rhs else None
    momg.euler_step(f, None, rhs, ctx)
    gc, gp = f.download()
    assert rel_field(gc, wc) < TOL and np.max(np.abs(gp - wp)) < TOL
    f2 = momg.CellField.from_host(mgrid(g), M, c, p)
    r = momg.residual(f2, ctx)
    momg.euler_step(f2, r, rhs, ctx)
    np.testing.assert_array_equal(f2.download()[0], gc)


def test_euler_nonphysical_dt():
    """global_dt raises NonphysicalState on a nonpositive temperature
    (single_level.cpp:20-21) before any cell is updated."""
    g = Grid.uniform(6, 5)
    octx = cavity_ctx(3, 1, BGK)
    c, p = smooth_field(g, 3, seed=2)
    p[7, 3] = -0.5
    f = momg.CellField.from_host(mgrid(g), 3, c, p)
    r = momg.CellField.from_host(mgrid(g), 3, np.zeros_like(c), p)
    with pytest.raises(momg.NonphysicalState):
        momg.euler_step(f, r, None, mctx(octx))
    np.testing.assert_array_equal(f.download()[0], c)


def test_solve_steady_euler():
    """SolverKind::euler of solve_steady (multigrid.cpp:276-277): iteration
    count within +-1 and macroscopic fields at 1e-8 against the oracle."""
    M = 3
    g = Grid.uniform(8, 8)
    octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    c, p = uniform_field(g, M)
    wc, wp, wr = O.solve_steady(octx, g, c, p, solver=0, tol=1e-4)
    assert wr["converged"]
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rep = momg.solve_steady(f, mctx(octx), momg.SolverOptions(momg.SolverKind.euler, 1e-4))
    assert rep.converged and abs(rep.iterations - wr["iterations"]) <= 1
    gc, gp = f.download()
    mg, mw = macro(gc, gp), macro(wc, wp)
    assert np.max(np.abs(mg - mw)) <= 1e-8 * np.max(np.abs(mw))
