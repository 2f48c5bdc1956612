"""The CPU oracle against the committed golden vectors, which were produced
by the REFERENCE itself (oracle/_ref = /root/reference/proj/src compiled
against oracle/shim) with tools/make_golden.py.  Runs without the reference
sources (e.g. on the GPU box)."""
import os

import numpy as np
import pytest

from helpers import BGK, ES_BGK, SHAKHOV, Ctx, Grid, Oracle, cavity_ctx, uniform_field

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
P = Oracle("port")


def load(name):
    return np.load(os.path.join(GOLD, name))


@pytest.mark.parametrize("M", [3, 5])
def test_primitives_golden(M):
    z = load("primitives.npz")
    c, p = z[f"M{M}_c"], z[f"M{M}_p"]
    np.testing.assert_array_equal(P.project(M, c[0], p[0], z[f"M{M}_to"]), z[f"M{M}_project"])
    gc, gp = P.grad_normalize(M, z[f"M{M}_gn_in"], p[2])
    np.testing.assert_array_equal(gc, z[f"M{M}_gn_c"])
    np.testing.assert_array_equal(gp, z[f"M{M}_gn_p"])
    cb = float(z[f"M{M}_cbound"])
    assert abs(P.max_hermite_root(M + 1) - cb) < 1e-13
    for axis in (0, 1):
        np.testing.assert_array_equal(P.half_flux(M, c[0], p[0], axis, True), z[f"M{M}_half{axis}_up"])
        np.testing.assert_array_equal(P.half_flux(M, c[0], p[0], axis, False), z[f"M{M}_half{axis}_lo"])
        np.testing.assert_array_equal(P.full_flux(M, c[0], p[0], axis), z[f"M{M}_full{axis}"])
        f, fp = P.face_flux(M, c[0], p[0], c[3], p[3], axis, cb)
        np.testing.assert_array_equal(f, z[f"M{M}_face{axis}"])
        np.testing.assert_array_equal(P.wall_flux(M, c[3], p[3], axis, 1, 0.1, 1.2)[0], z[f"M{M}_wall{axis}"])
    for name, model, pr in (("bgk", BGK, 1.0), ("shakhov", SHAKHOV, 2.0 / 3.0), ("es", ES_BGK, 2.0 / 3.0)):
        got = P.collision(Ctx(M=M, collision=model, prandtl=pr, knudsen=0.3), c[1], p[1])
        np.testing.assert_array_equal(got, z[f"M{M}_coll_{name}"])


FIELD_CASES = [(3, 1, BGK, 8, 8), (3, 2, BGK, 9, 7), (5, 1, SHAKHOV, 8, 8), (5, 2, BGK, 8, 8)]


@pytest.mark.parametrize("M,order,model,nx,ny", FIELD_CASES)
def test_fields_golden(M, order, model, nx, ny):
    z = load("fields.npz")
    tag = f"M{M}o{order}m{model}_{nx}x{ny}"
    g = Grid.uniform(nx, ny, 1.0, 1.1)
    ctx = cavity_ctx(M, order, model, kn=0.3, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                     bottom_theta=1.3)
    # the reference's own C_{M+1} (its eigensolver value, a few ulp from the
    # Newton root; dt depends on it at the ulp level)
    ctx.c_bound = ctx.cfl_c_bound = float(load("primitives.npz")[f"M{M}_cbound"])
    c, p = z[tag + "_c"], z[tag + "_p"]
    np.testing.assert_array_equal(P.residual(ctx, g, c, p), z[tag + "_res"])
    fc, fp, _ = P.fast_sweep(ctx, g, c, p)
    np.testing.assert_array_equal(fc, z[tag + "_fs_c"])
    np.testing.assert_array_equal(fp, z[tag + "_fs_p"])
    fc, fp, _ = P.fast_sweep(ctx, g, c, p, rhs=(c * 1e-3, p.copy()), sweep_order=[2, 0, 3, 1])
    np.testing.assert_array_equal(fc, z[tag + "_fsr_c"])
    if tag + "_rs_c" in z:
        cg = g.coarsen()
        cc, cp = P.restrict_solution(M, g, c, p, cg)
        np.testing.assert_array_equal(cc, z[tag + "_rs_c"])
        np.testing.assert_array_equal(P.restrict_residual(M, g, -z[tag + "_res"], p, p, cg, cp), z[tag + "_rr"])
        after = cc.copy(); after[:, 4:] += 1e-4
        np.testing.assert_array_equal(P.fas_correct(M, g, c, p, cg, cc, cp, after, cp)[0], z[tag + "_fas_c"])


def test_c1_golden():
    """C1 (BASELINE configs[0]): 32^2 lid cavity, M=3, FS to 1e-8 -- the
    reference's own iteration count, history and converged field."""
    z = load("c1.npz")
    M = 3
    g = Grid.uniform(32, 32)
    ctx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    ctx.c_bound = ctx.cfl_c_bound = float(z["c_bound"])
    c, p = uniform_field(g, M)
    fc, fp, rep = P.solve_steady(ctx, g, c, p, solver=1, tol=1e-8)
    assert rep["iterations"] == int(z["iterations"]) == 302
    np.testing.assert_array_equal(rep["history"], z["history"])
    np.testing.assert_array_equal(fc, z["coeffs"])
    np.testing.assert_array_equal(fp, z["params"])
