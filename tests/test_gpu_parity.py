"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle
on identical seeded inputs.  Tolerances (north_star): per-sweep moment fields
1e-10 relative (|d| <= 1e-10 max(1, |f0|), the idiom of
test_projection.cpp:144-145); converged macroscopic fields 1e-8; NMG
iteration counts within +-1."""
import numpy as np
import pytest

from helpers import BGK, SHAKHOV, Ctx, Grid, Oracle, c5_field, cavity_ctx, smooth_field, uniform_field

pytestmark = pytest.mark.gpu

momg = pytest.importorskip("paper_2206_13164_b200.momg")
O = Oracle("port")

TOL = 1e-10


def mctx(octx: Ctx) -> "momg.SolveContext":
    """Same configuration as an oracle Ctx, as the product's SolveContext."""
    W = momg.WallSpec
    walls = momg.Walls(*(W(octx.wall_speed[k], octx.wall_theta[k]) for k in range(4)))
    return momg.SolveContext(walls, momg.CollisionModel(momg.CollisionKind(octx.collision), octx.prandtl),
                             momg.GasParams(octx.knudsen, octx.viscosity_index),
                             momg.SpatialScheme(octx.space_order, octx.c_bound),
                             momg.CflPolicy(octx.cfl, octx.c_bound if octx.cfl_c_bound is None else octx.cfl_c_bound))


def mgrid(g: Grid) -> "momg.Grid2D":
    return momg.Grid2D(g.nx, g.ny, g.Lx, g.Ly, g.dx.copy(), g.dy.copy(), g.xc.copy(), g.yc.copy())


def rel_field(got, want):
    scale = np.maximum(1.0, np.abs(want[:, :1]))
    return float(np.max(np.abs(got - want) / scale))


def rel_res(got, want):
    scale = np.maximum(1.0, np.max(np.abs(want), axis=1, keepdims=True))
    return float(np.max(np.abs(got - want) / scale))


@pytest.fixture(params=["persistent", "warp", "diag"])
def sweep_mode(request):
    momg.set_sweep_mode(request.param)
    yield request.param
    momg.set_sweep_mode("persistent")


CASES = [
    # (M, order, model, nx, ny, uz)
    (3, 1, BGK, 8, 6, False),
    (3, 2, BGK, 9, 8, False),
    (4, 1, SHAKHOV, 7, 7, True),
    (5, 1, SHAKHOV, 7, 6, True),
    (5, 2, BGK, 8, 8, False),
    (6, 2, BGK, 6, 5, False),
    (7, 1, BGK, 5, 6, True),
    (8, 2, SHAKHOV, 6, 6, False),
]


def _setup(M, order, model, nx, ny, uz, seed=3):
    g = Grid.uniform(nx, ny, 1.0, 1.1)
    octx = cavity_ctx(M, order, model, kn=0.3, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                      bottom_theta=1.3)
    c, p = smooth_field(g, M, seed=seed + 10 * M + nx, amp=0.08, uz=uz)
    return g, octx, c, p


@pytest.mark.parametrize("M,order,model,nx,ny,uz", CASES)
def test_residual_parity(M, order, model, nx, ny, uz):
    g, octx, c, p = _setup(M, order, model, nx, ny, uz)
    want = O.residual(octx, g, c, p)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    got, gp = momg.residual(f, mctx(octx)).download()
    assert rel_res(got, want) < TOL
    np.testing.assert_array_equal(gp, p)  # residual params = cell params (spatial.cpp:128)


@pytest.mark.parametrize("M,order,model,nx,ny,uz", CASES)
def test_fast_sweep_parity(M, order, model, nx, ny, uz, sweep_mode):
    g, octx, c, p = _setup(M, order, model, nx, ny, uz)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    ctx = mctx(octx)
    wc, wp = c, p
    for it in range(2):  # two consecutive FS iterations, each checked
        wc, wp, ev = O.fast_sweep(octx, g, wc, wp)
        work = momg.WorkStats()
        momg.fast_sweep_step(f, None, ctx, work)
        gc, gp = f.download()
        assert work.cell_evals == ev == 4 * nx * ny
        assert rel_field(gc, wc) < TOL, f"iteration {it}"
        assert np.max(np.abs(gp - wp)) < TOL


@pytest.mark.parametrize("order", [[2, 0, 3, 1], [1, 1, 3, 3]])
def test_sweep_order_and_rhs(order, sweep_mode):
    M = 5
    g, octx, c, p = _setup(M, 2, BGK, 9, 7, False)
    rc = c * 1e-3
    rp = p.copy(); rp[:, 0] += 0.01; rp[:, 3] *= 1.02  # rhs in its own basis
    wc, wp, _ = O.fast_sweep(octx, g, c, p, rhs=(rc, rp), sweep_order=order)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rhs = momg.CellField.from_host(mgrid(g), M, rc, rp)
    momg.fast_sweep_step(f, rhs, mctx(octx), None, tuple(order))
    gc, gp = f.download()
    assert rel_field(gc, wc) < TOL
    assert np.max(np.abs(gp - wp)) < TOL


# Band tasks (M <= 5): grids wider than one band (32 columns at first order
# without rhs, k5_band; 16 columns at second order or with an FAS rhs,
# k6_band), so the inter-band halos (radius 2 at second order), partial bands
# and every sweep direction are exercised.
BAND_CASES = [
    # (M, model, nx, ny, sweep order, with rhs, space order)
    (5, BGK, 70, 37, (0, 1, 2, 3), False, 1),
    (3, SHAKHOV, 33, 5, (2, 0, 3, 1), True, 1),
    (4, BGK, 64, 40, (1, 1, 3, 3), True, 1),
    (5, SHAKHOV, 40, 66, (3, 2, 1, 0), True, 1),
    (5, BGK, 50, 35, (0, 1, 2, 3), False, 2),
    (3, SHAKHOV, 34, 20, (2, 0, 3, 1), True, 2),
    (4, BGK, 40, 33, (1, 1, 3, 3), True, 2),
    (5, SHAKHOV, 17, 48, (3, 2, 1, 0), True, 2),
]


@pytest.mark.parametrize("M,model,nx,ny,order,with_rhs,space", BAND_CASES)
def test_band_sweep_parity(M, model, nx, ny, order, with_rhs, space):
    g, octx, c, p = _setup(M, space, model, nx, ny, True)
    rhs_h = None
    if with_rhs:
        rc = c * 1e-3
        rp = p.copy(); rp[:, 0] += 0.01; rp[:, 3] *= 1.02
        rhs_h = (rc, rp)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rhs = momg.CellField.from_host(mgrid(g), M, *rhs_h) if with_rhs else None
    wc, wp = c, p
    for it in range(2):
        wc, wp, _ = O.fast_sweep(octx, g, wc, wp, rhs=rhs_h, sweep_order=list(order))
        momg.fast_sweep_step(f, rhs, mctx(octx), None, order)
        gc, gp = f.download()
        assert rel_field(gc, wc) < TOL, f"iteration {it}"
        assert np.max(np.abs(gp - wp)) < TOL


@pytest.mark.parametrize("M,nx,ny,order", [(5, 70, 37, (0, 1, 2, 3)), (3, 33, 50, (2, 0, 3, 1)), (4, 9, 7, (1, 2, 3, 0))])
def test_fused_sweep_residual(M, nx, ny, order):
    """momg_fast_sweep_residual == fast_sweep_step then residual (bitwise), and
    both against the oracle."""
    g, octx, c, p = _setup(M, 1, SHAKHOV if M == 3 else BGK, nx, ny, True)
    ctx = mctx(octx)
    f1 = momg.CellField.from_host(mgrid(g), M, c, p)
    momg.fast_sweep_step(f1, None, ctx, None, order)
    r1 = momg.residual(f1, ctx)
    f2 = momg.CellField.from_host(mgrid(g), M, c, p)
    r2 = momg.fast_sweep_residual(f2, ctx, None, None, order)
    a1, b1 = f1.download()
    a2, b2 = f2.download()
    np.testing.assert_array_equal(a1, a2)
    np.testing.assert_array_equal(b1, b2)
    rc1, rp1 = r1.download()
    rc2, rp2 = r2.download()
    np.testing.assert_array_equal(rc1, rc2)
    np.testing.assert_array_equal(rp1, rp2)
    wc, wp, _ = O.fast_sweep(octx, g, c, p, sweep_order=list(order))
    assert rel_field(a2, wc) < TOL
    assert rel_res(rc2, O.residual(octx, g, wc, wp)) < TOL


@pytest.mark.parametrize("M,model,nx,ny", [(5, BGK, 70, 37), (3, SHAKHOV, 40, 65), (4, BGK, 33, 9)])
def test_band_residual_multiband(M, model, nx, ny):
    """First-order residual on the band kernel (residual mode): several bands,
    diagonal chunks starting mid-band, against the oracle."""
    g, octx, c, p = _setup(M, 1, model, nx, ny, True)
    want = O.residual(octx, g, c, p)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    got, gp = momg.residual(f, mctx(octx)).download()
    assert rel_res(got, want) < TOL
    np.testing.assert_array_equal(gp, p)


def test_overlapped_transfers_double_buffer():
    """momg_field_{upload,download}_overlapped: a double-buffered stream of
    solves gives the same results as the synchronous path."""
    g, octx, c, p = _setup(5, 1, BGK, 40, 24, True)
    ctx = mctx(octx)
    f0 = momg.CellField.from_host(mgrid(g), 5, c, p)
    momg.fast_sweep_step(f0, None, ctx)
    want_c, want_p = f0.download()
    L, C = momg.lib(), momg.C
    flds = [momg.CellField(mgrid(g), 5), momg.CellField(mgrid(g), 5)]
    hc, hp = np.ascontiguousarray(c), np.ascontiguousarray(p)
    outs = [(np.zeros_like(c), np.zeros_like(p)) for _ in range(3)]
    e = momg._Err()
    assert L.momg_field_upload_overlapped(flds[0].handle, momg._dp(hc), momg._dp(hp), C.byref(e)) == 0
    for s_ in range(3):
        cur, nxt = flds[s_ % 2], flds[(s_ + 1) % 2]
        momg.fast_sweep_step(cur, None, ctx)
        if s_ < 2:
            assert L.momg_field_upload_overlapped(nxt.handle, momg._dp(hc), momg._dp(hp), C.byref(e)) == 0
        oc, op = outs[s_]
        assert L.momg_field_download_overlapped(cur.handle, momg._dp(oc), momg._dp(op), C.byref(e)) == 0
    assert L.momg_copy_barrier(C.byref(e)) == 0
    assert L.momg_synchronize(C.byref(e)) == 0
    for oc, op in outs:
        np.testing.assert_array_equal(oc, want_c)
        np.testing.assert_array_equal(op, want_p)


@pytest.mark.parametrize("M", [3, 5, 6, 8])
def test_transfer_operators_parity(M):
    fg = Grid.uniform(8, 12, 1.0, 1.0)
    cg = fg.coarsen()
    c, p = smooth_field(fg, M, seed=11 + M, amp=0.1, uz=True)
    wc, wp = O.restrict_solution(M, fg, c, p, cg)
    fine = momg.CellField.from_host(mgrid(fg), M, c, p)
    coarse = momg.restrict_solution(fine, mgrid(cg))
    gc, gp = coarse.download()
    assert rel_field(gc, wc) < TOL and np.max(np.abs(gp - wp)) < TOL
    # restrict_residual of a defect carrying its own basis
    octx = cavity_ctx(M, 1, BGK)
    res = O.residual(octx, fg, c, p)
    dp = p.copy(); dp[:, 1] += 0.02
    want = O.restrict_residual(M, fg, -res, dp, p, cg, wp)
    arrays = momg.CellField.from_host(mgrid(fg), M, -res, dp)
    got, gpp = momg.restrict_residual(arrays, fine, coarse).download()
    assert rel_res(got, want) < TOL
    np.testing.assert_array_equal(gpp, gp)
    # fas_correct
    after = wc.copy(); after[:, 4:] += 1e-4 * np.sin(np.arange(after[:, 4:].size)).reshape(after[:, 4:].shape)
    ap = wp.copy(); ap[:, 0] += 1e-3
    want_c, want_p = O.fas_correct(M, fg, c, p, cg, wc, wp, after, ap)
    before_f = momg.CellField.from_host(mgrid(cg), M, wc, wp)
    after_f = momg.CellField.from_host(mgrid(cg), M, after, ap)
    momg.fas_correct(fine, before_f, after_f)
    gc2, gp2 = fine.download()
    assert rel_field(gc2, want_c) < TOL and np.max(np.abs(gp2 - want_p)) < TOL


def test_mass_and_norms_parity():
    M = 5
    g = Grid.uniform(33, 17, 1.3, 0.7)
    c, p = c5_field(g.nx, g.ny, M, seed=5)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    assert abs(momg.total_mass(f) - O.total_mass(g, M, c)) <= 1e-14 * abs(O.total_mass(g, M, c))
    momg.mass_correction(f, 0.77)
    gc, _ = f.download()
    assert rel_field(gc, O.mass_correction(g, M, c, 0.77)) < 1e-14
    octx = cavity_ctx(M, 1, BGK)
    res = O.residual(octx, g, c, p)
    rf = momg.CellField.from_host(mgrid(g), M, res, p)
    f2 = momg.CellField.from_host(mgrid(g), M, c, p)
    want = O.residual_norm(M, g, res, p)
    assert abs(momg.residual_norm(rf, f2) - want) <= 1e-13 * want


def test_nmg_cycle_parity():
    M = 3
    g = Grid.uniform(16, 16)
    octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    c, p = uniform_field(g, M)
    wc, wp, ww = O.nmg_cycle(octx, g, c, p, levels=2)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    work = momg.WorkStats()
    momg.nmg_cycle(f, mctx(octx), levels=2, work=work)
    gc, gp = f.download()
    assert work.cell_evals == ww
    assert rel_field(gc, wc) < TOL and np.max(np.abs(gp - wp)) < TOL


def macro(c, p):
    """rho, u, theta, heat flux, stress of Grad-normalized cells (extract_macro)."""
    rho = c[:, 0]
    q = np.stack([3 * c[:, 10] + c[:, 13] + c[:, 15], 3 * c[:, 16] + c[:, 11] + c[:, 18],
                  3 * c[:, 19] + c[:, 12] + c[:, 17]], axis=1)
    sig = np.stack([2 * c[:, 4], c[:, 5], c[:, 6], 2 * c[:, 7], c[:, 8], 2 * c[:, 9]], axis=1)
    return np.concatenate([rho[:, None], p, q, sig], axis=1)


@pytest.mark.parametrize("solver,nx,levels", [("nmg", 16, 2), ("fs", 16, 0), ("nmg", 32, 0)])
def test_solve_steady_parity(solver, nx, levels):
    """Converged macroscopic fields within 1e-8 and iteration counts within +-1
    (acceptance-style cavity, M = 3, first order)."""
    M = 3
    g = Grid.uniform(nx, nx)
    octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    c, p = uniform_field(g, M)
    kind = {"fs": 1, "nmg": 2}[solver]
    wc, wp, wr = O.solve_steady(octx, g, c, p, solver=kind, tol=1e-8, levels=levels)
    assert wr["converged"]
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    opts = momg.SolverOptions(momg.SolverKind(kind), 1e-8, 0, levels)
    replays = momg.graph_replays()
    launches = momg.launch_count()
    rep = momg.solve_steady(f, mctx(octx), opts)
    assert rep.converged
    assert abs(rep.iterations - wr["iterations"]) <= 1
    # iterations 2.. are replays of the captured iteration graph; the launch
    # counter still counts every kernel of every iteration
    assert momg.graph_replays() - replays == rep.iterations - 2
    assert momg.launch_count() - launches >= 3 * rep.iterations
    gc, gp = f.download()
    mg, mw = macro(gc, gp), macro(wc, wp)
    assert np.max(np.abs(mg - mw)) <= 1e-8 * np.max(np.abs(mw))


def test_dt_halving_and_solver_error(sweep_mode):
    """test_single_level.cpp:135-156 on the device: the first visit survives
    only at dt/2 (rho = 1 - 0.5*0.045*30), the second raises SolverError and
    leaves the cell in its pre-update state."""
    g = momg.Grid2D.uniform(1, 1, 0.1, 0.1)
    ctx = momg.SolveContext(scheme=momg.SpatialScheme(1, 1.0), cfl=momg.CflPolicy(0.9, 1.0),
                            gas=momg.GasParams(1e300))
    f = momg.uniform_field(g, 3, 1.0, (0.0, 0.0, 0.0), 1.0)
    rc = np.zeros((1, 20)); rc[0, 0] = 30.0
    rhs = momg.CellField.from_host(g, 3, rc, np.array([[0, 0, 0, 1.0]]))
    with pytest.raises(momg.SolverError):
        momg.fast_sweep_step(f, rhs, ctx)
    c, _ = f.download()
    assert c[0, 0] == pytest.approx(1.0 - 0.5 * 0.045 * 30.0, rel=1e-12)


def test_nonconvergence_carries_report():
    M = 3
    g = momg.Grid2D.uniform(16, 16)
    ctx = momg.cavity_context(M, 1)
    f = momg.uniform_field(g, M, 1.0, (0, 0, 0), 1.0)
    with pytest.raises(momg.NonConvergence) as ei:
        momg.solve_steady(f, ctx, momg.SolverOptions(momg.SolverKind.fs, 1e-8, 3))
    assert ei.value.report.iterations == 3 and len(ei.value.report.history) == 3


def _golden(name):
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name))


def _macro_rel(got, want):
    # relative to each quantity's own scale (rho, u, theta, q, sigma columns)
    scale = np.maximum(np.max(np.abs(want), axis=0), 1e-12)
    return float(np.max(np.abs(got - want) / scale))


def test_c1_against_reference_golden():
    """BASELINE configs[0] (C1): 32^2, M=3, first order, BGK Kn 0.1, FS to 1e-8.
    Golden = the reference's own run (302 iterations)."""
    z = _golden("c1.npz")
    M = 3
    g = Grid.uniform(32, 32)
    octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
    octx.c_bound = octx.cfl_c_bound = float(z["c_bound"])
    c, p = uniform_field(g, M)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rep = momg.solve_steady(f, mctx(octx), momg.SolverOptions(momg.SolverKind.fs, 1e-8))
    assert rep.converged and abs(rep.iterations - int(z["iterations"])) <= 1
    gc, gp = f.download()
    assert _macro_rel(macro(gc, gp), macro(z["coeffs"], z["params"])) <= 1e-8


def test_c2_against_reference_golden():
    """BASELINE configs[1] (C2): 128^2, M=5, second order, BGK Kn 0.1, NMG over
    4 levels (V(2,2), s3=4) to 1e-8.  Golden = the CPU oracle run (99 NMG
    iterations, 1231 s single-threaded): the reference itself (oracle/_ref, tools/make_golden.py)."""
    z = _golden("c2.npz")
    M = 5
    g = Grid.uniform(128, 128)
    octx = cavity_ctx(M, 2, BGK, kn=0.1, lid=0.1)
    octx.c_bound = octx.cfl_c_bound = float(z["c_bound"])
    c, p = uniform_field(g, M)
    f = momg.CellField.from_host(mgrid(g), M, c, p)
    rep = momg.solve_steady(f, mctx(octx), momg.SolverOptions(momg.SolverKind.nmg, 1e-8, 0, 4))
    assert rep.converged and abs(rep.iterations - int(z["iterations"])) <= 1
    gc, gp = f.download()
    q = np.stack([3 * gc[:, 10] + gc[:, 13] + gc[:, 15], 3 * gc[:, 16] + gc[:, 11] + gc[:, 18]], axis=1)
    mg = np.concatenate([gc[:, :1], gp, q, 2 * gc[:, 4:5], gc[:, 5:6], 2 * gc[:, 7:8]], axis=1)
    want = z["macro"]
    # u_z is identically zero in the cavity: compare it absolutely
    cols = [k for k in range(want.shape[1]) if k != 3]
    assert _macro_rel(mg[:, cols], want[:, cols]) <= 1e-8
    assert np.max(np.abs(mg[:, 3])) <= 1e-12


def test_reference_program_through_bridge():
    """The reference's own C++ (its Grid2D/SolveContext/solve_steady), switched
    to the B200 by integration/momg_gpu_bridge.hpp: C1 on CPU (reference) and
    GPU agree (iterations +-1, macro 1e-8).  Binary built here by
    `make -C oracle bridge` (needs the reference sources) and shipped."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "bridge_demo")
    if not os.path.exists(exe):
        pytest.skip("bridge_demo not built (needs /root/reference at build time)")
    out = subprocess.run([exe, "32"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    import json
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["cpu_iterations"] == 302 and abs(d["gpu_iterations"] - 302) <= 1
