"""Pins the CPU oracle (oracle/momg_oracle.c) before anything is checked
against it:
  (a) known answers from the reference's own unit tests (file:line cited), and
  (b) bit-for-bit agreement with the reference itself, compiled here from
      /root/reference/proj/src against oracle/shim (oracle/_ref).
The reference's own unit tests also run against the shims (oracle/Makefile
ref-tests; test_reference_unit_tests below)."""
import math
import os
import subprocess

import numpy as np
import pytest

from helpers import (BGK, ES_BGK, HAVE_REF, SHAKHOV, Ctx, Grid, Oracle, c_bound, cavity_ctx,
                     count, random_grad_rep, random_rep, smooth_field, uniform_field)

P = Oracle("port")
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def R():
    return Oracle("reference")


# ------------------------------------------------------------ known answers
def test_index_set_known_answers():
    # test_hermite.cpp:13-69
    assert count(3) == 20 and count(5) == 56 and count(10) == 286
    a, down, up, deg, fact = P.index_tables(5)
    assert tuple(a[0]) == (0, 0, 0) and tuple(a[1]) == (1, 0, 0)
    assert tuple(a[2]) == (0, 1, 0) and tuple(a[3]) == (0, 0, 1)
    k = [i for i in range(56) if tuple(a[i]) == (5, 0, 0)][0]
    assert fact[k] == 120.0
    k = [i for i in range(56) if tuple(a[i]) == (3, 2, 0)][0]
    assert fact[k] == 12.0
    # ascending degree, descending lexicographic inside a degree
    for i in range(1, 56):
        assert deg[i] >= deg[i - 1]
        if deg[i] == deg[i - 1]:
            assert tuple(a[i]) < tuple(a[i - 1])
    for d in range(3):
        for k in range(56):
            if down[d, k] >= 0:
                e = np.array(a[k]); e[d] -= 1
                assert tuple(a[down[d, k]]) == tuple(e)


def test_hermite_roots_known_answers():
    # test_hermite.cpp:104-120: C2 = 1, C4 = sqrt(3+sqrt(6)), C6 ~ 3.324257
    assert abs(P.max_hermite_root(2) - 1.0) < 1e-13
    assert abs(P.max_hermite_root(4) - math.sqrt(3 + math.sqrt(6))) < 1e-13
    assert abs(P.max_hermite_root(6) - 3.324257433552119) < 1e-11


def test_projection_known_answers():
    # test_projection.cpp:82-148: identity is bitwise; a Maxwellian shifted by
    # 0.5 along x gains f_e1 = 0.5 (rho = 1); round trip to 1e-12.
    rng = np.random.default_rng(1)
    for M in (3, 5):
        c, p = random_grad_rep(rng, M)
        assert np.array_equal(P.project(M, c, p, p), c)
        to = p + np.array([0.2, -0.1, 0.05, 0.3])
        back = P.project(M, P.project(M, c, p, to), to, p)
        assert np.max(np.abs(back - c)) <= 1e-12 * max(1.0, abs(c[0]))
    c = np.zeros(count(3)); c[0] = 1.0
    out = P.project(3, c, [0.5, 0, 0, 1.0], [0, 0, 0, 1.0])
    assert abs(out[1] - 0.5) < 1e-15


def test_grad_normalize_known_answers():
    # test_projection.cpp:159-201: defect <= 1e-12 after, idempotent
    rng = np.random.default_rng(2)
    c, p = random_grad_rep(rng, 5)
    c[1] += 0.03; c[4] += 0.02
    c2, p2 = P.grad_normalize(5, c, p)
    assert P.grad_defect(5, c2) <= 1e-12
    c3, p3 = P.grad_normalize(5, c2, p2)
    assert np.max(np.abs(c3 - c2)) <= 1e-12 * c2[0]
    bad = c.copy(); bad[0] = -1.0
    with pytest.raises(Exception):
        P.grad_normalize(5, bad, p)


def test_collision_frequency_known_answer():
    # test_collision.cpp:75-90: nu = 12.533141373155003 at Kn 0.1, rho = theta = 1
    ctx = Ctx(M=3, knudsen=0.1)
    c, p = uniform_field(Grid.uniform(1, 1), 3)
    c = c[0].copy(); c[4] = 0.01  # departure so Q != 0: Q = -nu * f
    q = P.collision(ctx, c, p[0])
    nu = -q[4] / 0.01
    assert abs(nu - 12.533141373155003) < 1e-12


def test_half_range_known_answers():
    # test_halfspace.cpp:18-40: a = 0 frozen values
    up, lo = P.half_range_table(4, 0.0)
    inv = 1.0 / math.sqrt(2 * math.pi)
    assert abs(up[0, 0] - 0.5) < 1e-14 and abs(up[0, 1] - inv) < 1e-14
    assert abs(up[1, 0] - inv) < 1e-14 and abs(up[1, 1] - 0.5) < 1e-14
    assert abs(up[0, 2]) < 1e-14 and abs(lo[0, 1] + inv) < 1e-12
    # upper + lower = m! delta
    for m in range(5):
        for q in range(5):
            assert abs(up[m, q] + lo[m, q] - (math.factorial(m) if m == q else 0.0)) < 1e-12


def test_resting_half_mass_flux():
    # test_flux.cpp: resting Maxwellian half mass flux = rho sqrt(theta)/sqrt(2 pi)
    c = np.zeros(count(3)); c[0] = 1.7
    p = np.array([0, 0, 0, 1.3])
    h = P.half_flux(3, c, p, 0, True)
    assert abs(h[0] - 1.7 * math.sqrt(1.3) / math.sqrt(2 * math.pi)) < 1e-13


def test_local_dt_and_dt_halving_known_answers():
    # test_single_level.cpp:42-56 (dt = 0.045 for a resting unit cell, C = 1) and
    # :135-156 (a mass loss only the halved step survives: rho = 1 - 0.5*dt*30;
    # the next one fails loudly and leaves the cell in its pre-update state).
    g = Grid.uniform(1, 1, 0.1, 0.1)
    ctx = Ctx(M=3, c_bound=1.0, cfl_c_bound=1.0, knudsen=1e300)
    c, p = uniform_field(g, 3)
    rhs_c = np.zeros_like(c); rhs_c[0, 0] = 30.0  # delta = R - r = -30 on f0
    out, _, ev, rc, msg = P.fast_sweep(ctx, g, c, p, rhs=(rhs_c, p.copy()), raise_errors=False)
    assert rc == 2 and "after dt halving" in msg  # SolverError on the 2nd visit
    assert ev == 1
    assert out[0, 0] == pytest.approx(1.0 - 0.5 * 0.045 * 30.0, rel=1e-12)


# --------------------------------------------------- bitwise vs the reference
def _check_equal(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


@needs_ref
@pytest.mark.parametrize("M", [3, 5, 8])
def test_primitives_bitwise(R, M):
    rng = np.random.default_rng(10 + M)
    for _ in range(6):
        c, p = random_grad_rep(rng, M)
        c2, p2 = random_grad_rep(rng, M)
        to = p + rng.uniform(-0.3, 0.3, 4); to[3] = abs(to[3]) + 0.2
        _check_equal(P.project(M, c, p, to), R.project(M, c, p, to))
        cc = c.copy(); cc[1] += 0.01; cc[5] += 0.02
        _check_equal(P.grad_normalize(M, cc, p)[0], R.grad_normalize(M, cc, p)[0])
        for axis in range(3):
            for pos in (0, 1):
                _check_equal(P.half_flux(M, c, p, axis, pos), R.half_flux(M, c, p, axis, pos))
            _check_equal(P.full_flux(M, c, p, axis), R.full_flux(M, c, p, axis))
        for axis in range(2):
            cb = c_bound(M)
            _check_equal(P.face_flux(M, c, p, c2, p2, axis, cb)[0],
                         R.face_flux(M, c, p, c2, p2, axis, cb)[0])
            for high in (0, 1):
                _check_equal(P.wall_flux(M, c, p, axis, high, 0.1, 1.2)[0],
                             R.wall_flux(M, c, p, axis, high, 0.1, 1.2)[0])
        for model, pr in ((BGK, 1.0), (SHAKHOV, 2.0 / 3.0), (ES_BGK, 2.0 / 3.0)):
            ctx = Ctx(M=M, collision=model, prandtl=pr, knudsen=0.3)
            _check_equal(P.collision(ctx, c, p), R.collision(ctx, c, p))
    for a in (-2.0, -0.3, 0.0, 0.7, 3.1):
        up1, lo1 = P.half_range_table(M + 1, a)
        up2, lo2 = R.half_range_table(M + 1, a)
        _check_equal(up1, up2)
        _check_equal(lo1, lo2)


@needs_ref
def test_index_tables_and_roots_vs_reference(R):
    for M in (2, 3, 5, 6, 8):
        for x, y in zip(P.index_tables(M), R.index_tables(M)):
            _check_equal(x, y)
        assert abs(P.max_hermite_root(M + 1) - R.max_hermite_root(M + 1)) < 1e-14 * (M + 1)


FIELD_CASES = [
    # (M, order, model, nx, ny)
    (3, 1, BGK, 8, 6),
    (3, 2, BGK, 8, 8),
    (5, 1, SHAKHOV, 6, 7),
    (5, 2, BGK, 8, 8),
    (6, 2, BGK, 5, 6),
]


@needs_ref
@pytest.mark.parametrize("M,order,model,nx,ny", FIELD_CASES)
def test_field_ops_bitwise(R, M, order, model, nx, ny):
    g = Grid.uniform(nx, ny, 1.0, 1.1)
    ctx = cavity_ctx(M, order, model, kn=0.3, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                     bottom_theta=1.3)
    c, p = smooth_field(g, M, seed=nx * 100 + ny + M, uz=(M == 5))
    _check_equal(P.residual(ctx, g, c, p), R.residual(ctx, g, c, p))
    a = P.fast_sweep(ctx, g, c, p)
    b = R.fast_sweep(ctx, g, c, p)
    _check_equal(a[0], b[0]); _check_equal(a[1], b[1]); assert a[2] == b[2] == 4 * nx * ny
    rhs = (c * 1e-3, p.copy())
    a = P.fast_sweep(ctx, g, c, p, rhs=rhs, sweep_order=[2, 0, 3, 1])
    b = R.fast_sweep(ctx, g, c, p, rhs=rhs, sweep_order=[2, 0, 3, 1])
    _check_equal(a[0], b[0]); _check_equal(a[1], b[1])
    assert P.total_mass(g, M, c) == R.total_mass(g, M, c)
    _check_equal(P.mass_correction(g, M, c, 1.01), R.mass_correction(g, M, c, 1.01))
    res = P.residual(ctx, g, c, p)
    assert P.residual_norm(M, g, res, p) == R.residual_norm(M, g, res, p)


@needs_ref
@pytest.mark.parametrize("M", [3, 5])
def test_transfer_ops_bitwise(R, M):
    fg = Grid.uniform(8, 12, 1.0, 1.0)
    cg = fg.coarsen()
    c, p = smooth_field(fg, M, seed=7 + M, amp=0.1, uz=True)
    cc1, cp1 = P.restrict_solution(M, fg, c, p, cg)
    cc2, cp2 = R.restrict_solution(M, fg, c, p, cg)
    _check_equal(cc1, cc2); _check_equal(cp1, cp2)
    ctx = cavity_ctx(M, 1, BGK)
    res = P.residual(ctx, fg, c, p)
    _check_equal(P.restrict_residual(M, fg, -res, p, p, cg, cp1),
                 R.restrict_residual(M, fg, -res, p, p, cg, cp1))
    after = cc1.copy(); after[:, 4:] += 1e-4
    a = P.fas_correct(M, fg, c, p, cg, cc1, cp1, after, cp1)
    b = R.fas_correct(M, fg, c, p, cg, cc1, cp1, after, cp1)
    _check_equal(a[0], b[0]); _check_equal(a[1], b[1])


@needs_ref
@pytest.mark.parametrize("M,order,model", [(3, 1, BGK), (5, 2, SHAKHOV), (4, 1, ES_BGK)])
def test_euler_step_bitwise(R, M, order, model):
    """euler_step (single_level.cpp:74-97) with and without an rhs, and the
    Euler solver of solve_steady, port vs reference bit for bit."""
    g = Grid.uniform(7, 6, 1.0, 1.2)
    ctx = cavity_ctx(M, order, model, kn=0.3, prandtl=2.0 / 3.0 if model != BGK else 1.0,
                     bottom_theta=1.3)
    c, p = smooth_field(g, M, seed=31 + M, uz=True)
    a = P.euler_step(ctx, g, c, p)
    b = R.euler_step(ctx, g, c, p)
    _check_equal(a[0], b[0]); _check_equal(a[1], b[1])
    rp = p.copy(); rp[:, 1] += 0.01; rp[:, 3] *= 1.03
    rhs = (c * 1e-3, rp)
    a = P.euler_step(ctx, g, c, p, rhs=rhs)
    b = R.euler_step(ctx, g, c, p, rhs=rhs)
    _check_equal(a[0], b[0]); _check_equal(a[1], b[1])
    gg = Grid.uniform(8, 8)
    cc, pp = uniform_field(gg, 3)
    cx = cavity_ctx(3, 1, BGK, kn=0.1, lid=0.1)
    a = P.solve_steady(cx, gg, cc, pp, solver=0, tol=1e-3)
    b = R.solve_steady(cx, gg, cc, pp, solver=0, tol=1e-3)
    assert a[2]["iterations"] == b[2]["iterations"] and a[2]["converged"]
    _check_equal(a[0], b[0])


@needs_ref
def test_nmg_and_solve_bitwise(R):
    M = 3
    g = Grid.uniform(16, 16)
    ctx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    c, p = uniform_field(g, M)
    a = P.nmg_cycle(ctx, g, c, p, levels=2)
    b = R.nmg_cycle(ctx, g, c, p, levels=2)
    _check_equal(a[0], b[0]); _check_equal(a[1], b[1]); assert a[2] == b[2]
    a = P.solve_steady(ctx, g, c, p, solver=2, tol=1e-4, levels=2)
    b = R.solve_steady(ctx, g, c, p, solver=2, tol=1e-4, levels=2)
    assert a[2]["iterations"] == b[2]["iterations"] and a[2]["converged"]
    _check_equal(a[2]["history"], b[2]["history"])
    _check_equal(a[0], b[0])


@needs_ref
def test_reference_unit_tests():
    """The reference's own doctest suites pass against the shims (validates the
    Eigen / doctest / nlohmann-json shims that oracle/_ref is built with; the
    scenario suite runs the front end, scenario.cpp, including one NMG solve)."""
    if not os.path.isdir("/root/reference/proj"):
        pytest.skip("reference sources absent")
    here = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle")
    out = subprocess.run(["make", "-s", "-C", here, "ref-tests"], capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("| 0 failed") == 9
