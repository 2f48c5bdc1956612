"""ctypes front end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads either the plain-C restatement (``oracle/liboracle.so``, kind="port") or
the reference itself compiled against the shims (``oracle/_ref/libmomg_ref.so``,
kind="reference").  Both export the API of ``oracle/momg_oracle.h``.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import
this module; the product package never does.

Arrays: ``coeffs`` is (cells, N) float64 C-contiguous, ``params`` is (cells, 4)
= (mean_x, mean_y, mean_z, spread); cell index = j*nx + i (grid.hpp:64).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libmomg_ref.so")
REF_SRC = "/root/reference/proj"

MO_OK, MO_NONPHYSICAL_STATE, MO_SOLVER_ERROR, MO_ERROR, MO_NON_SPD, MO_CONFIG, MO_NONCONVERGENCE = range(7)
BGK, ES_BGK, SHAKHOV = 0, 1, 2
EULER, FS, NMG = 0, 1, 2

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class MoErr(C.Structure):
    _fields_ = [("code", C.c_int), ("msg", C.c_char * 256)]


class MoGrid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("Lx", C.c_double), ("Ly", C.c_double),
                ("dx", _dp), ("dy", _dp), ("xc", _dp), ("yc", _dp)]


class MoCtx(C.Structure):
    _fields_ = [("M", C.c_int), ("space_order", C.c_int), ("c_bound", C.c_double),
                ("cfl", C.c_double), ("cfl_c_bound", C.c_double), ("collision", C.c_int),
                ("prandtl", C.c_double), ("knudsen", C.c_double),
                ("viscosity_index", C.c_double), ("wall_speed", C.c_double * 4),
                ("wall_theta", C.c_double * 4), ("threads", C.c_int)]


class MoReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("r0_norm", C.c_double),
                ("final_norm", C.c_double), ("final_ratio", C.c_double),
                ("work", C.c_longlong), ("seconds", C.c_double), ("history_len", C.c_int),
                ("history", _dp), ("history_cap", C.c_int)]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def count(M: int) -> int:
    return (M + 1) * (M + 2) * (M + 3) // 6


@dataclass
class Grid:
    """Grid2D (grid.hpp:12-37) with per-cell sizes and centres."""
    nx: int
    ny: int
    Lx: float
    Ly: float
    dx: np.ndarray
    dy: np.ndarray
    xc: np.ndarray
    yc: np.ndarray

    @staticmethod
    def uniform(nx: int, ny: int, Lx: float = 1.0, Ly: float = 1.0) -> "Grid":
        # Grid2D::uniform, grid.hpp:18-33 (same float operations, same order)
        dx = np.full(nx, Lx / nx)
        dy = np.full(ny, Ly / ny)
        xc = np.array([(i + 0.5) * Lx / nx for i in range(nx)])
        yc = np.array([(j + 0.5) * Ly / ny for j in range(ny)])
        return Grid(nx, ny, Lx, Ly, dx, dy, xc, yc)

    def coarsen(self) -> "Grid":
        # coarsen, multigrid.cpp:12-35
        nx, ny = self.nx // 2, self.ny // 2
        dx = np.empty(nx); xc = np.empty(nx); dy = np.empty(ny); yc = np.empty(ny)
        x = 0.0
        for i in range(nx):
            dx[i] = self.dx[2 * i] + self.dx[2 * i + 1]
            xc[i] = x + 0.5 * dx[i]
            x += dx[i]
        y = 0.0
        for j in range(ny):
            dy[j] = self.dy[2 * j] + self.dy[2 * j + 1]
            yc[j] = y + 0.5 * dy[j]
            y += dy[j]
        return Grid(nx, ny, self.Lx, self.Ly, dx, dy, xc, yc)

    @property
    def cells(self) -> int:
        return self.nx * self.ny

    def c(self) -> MoGrid:
        for a in ("dx", "dy", "xc", "yc"):
            setattr(self, a, np.ascontiguousarray(getattr(self, a), dtype=np.float64))
        return MoGrid(self.nx, self.ny, self.Lx, self.Ly, _ptr(self.dx), _ptr(self.dy),
                      _ptr(self.xc), _ptr(self.yc))


@dataclass
class Ctx:
    """SolveContext (single_level.hpp:27-34) with the scenario's convention
    cfl.c_bound = scheme.c_bound (scenario.cpp:421)."""
    M: int = 3
    space_order: int = 1
    c_bound: float = 1.0
    cfl: float = 0.9
    cfl_c_bound: float | None = None
    collision: int = BGK
    prandtl: float = 1.0
    knudsen: float = 1.0
    viscosity_index: float = 0.81
    wall_speed: tuple = (0.0, 0.0, 0.0, 0.0)  # left, right, bottom, top
    wall_theta: tuple = (1.0, 1.0, 1.0, 1.0)
    threads: int = 1

    def c(self) -> MoCtx:
        cb = self.c_bound if self.cfl_c_bound is None else self.cfl_c_bound
        return MoCtx(self.M, self.space_order, self.c_bound, self.cfl, cb, self.collision,
                     self.prandtl, self.knudsen, self.viscosity_index,
                     (C.c_double * 4)(*self.wall_speed), (C.c_double * 4)(*self.wall_theta),
                     self.threads)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _arr(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


class Oracle:
    """One loaded oracle library ("port" = C restatement, "reference" = the
    reference compiled against the shims)."""

    def __init__(self, kind: str = "port"):
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            build(kind)
        self.kind = kind
        self.lib = C.CDLL(path)
        L = self.lib
        L.mo_max_hermite_root.restype = C.c_double
        L.mo_grad_defect.restype = C.c_double
        L.mo_total_mass.restype = C.c_double
        L.mo_residual_norm.restype = C.c_double

    # ---------------------------------------------------------------- helpers
    def _check(self, rc: int, err: MoErr):
        if rc != MO_OK:
            raise OracleError(rc, err.msg.decode(errors="replace"))

    def index_tables(self, M: int):
        n = count(M)
        a = np.zeros(3 * n, np.int32); dn = np.zeros(3 * n, np.int32); up = np.zeros(3 * n, np.int32)
        deg = np.zeros(n, np.int32); fact = np.zeros(n)
        ip = lambda x: x.ctypes.data_as(_ip)
        self.lib.mo_index_tables(M, ip(a), ip(dn), ip(up), ip(deg), _ptr(fact))
        return a.reshape(n, 3), dn.reshape(3, n), up.reshape(3, n), deg, fact

    def max_hermite_root(self, degree: int) -> float:
        return self.lib.mo_max_hermite_root(degree)

    # ------------------------------------------------------------- primitives
    def project(self, M, coeffs, frm, to):
        c = _arr(coeffs); out = np.empty_like(c); err = MoErr()
        self._check(self.lib.mo_project(M, _ptr(c), _ptr(_arr(frm)), _ptr(_arr(to)), _ptr(out),
                                        C.byref(err)), err)
        return out

    def grad_normalize(self, M, coeffs, params):
        c = _arr(coeffs).copy(); p = _arr(params).copy(); err = MoErr()
        self._check(self.lib.mo_grad_normalize(M, _ptr(c), _ptr(p), C.byref(err)), err)
        return c, p

    def grad_defect(self, M, coeffs):
        return self.lib.mo_grad_defect(M, _ptr(_arr(coeffs)))

    def half_range_table(self, pmax, a):
        up = np.zeros((pmax + 1) ** 2); lo = np.zeros((pmax + 1) ** 2)
        self.lib.mo_half_range_table(pmax, C.c_double(a), _ptr(up), _ptr(lo))
        return up.reshape(pmax + 1, pmax + 1), lo.reshape(pmax + 1, pmax + 1)

    def half_flux(self, M, coeffs, params, axis, positive):
        c = _arr(coeffs); out = np.empty_like(c); err = MoErr()
        self._check(self.lib.mo_half_flux(M, _ptr(c), _ptr(_arr(params)), axis, int(positive),
                                          _ptr(out), C.byref(err)), err)
        return out

    def full_flux(self, M, coeffs, params, axis):
        c = _arr(coeffs); out = np.empty_like(c)
        self.lib.mo_full_flux(M, _ptr(c), _ptr(_arr(params)), axis, _ptr(out))
        return out

    def face_flux(self, M, lc, lp, rc, rp, axis, c_bound):
        out = np.empty(count(M)); fp = np.empty(4); err = MoErr()
        self._check(self.lib.mo_face_flux(M, _ptr(_arr(lc)), _ptr(_arr(lp)), _ptr(_arr(rc)),
                                          _ptr(_arr(rp)), axis, C.c_double(c_bound), _ptr(out),
                                          _ptr(fp), C.byref(err)), err)
        return out, fp

    def wall_flux(self, M, c, p, axis, high, speed, theta):
        out = np.empty(count(M)); wp = np.empty(4); err = MoErr()
        self._check(self.lib.mo_wall_flux(M, _ptr(_arr(c)), _ptr(_arr(p)), axis, int(high),
                                          C.c_double(speed), C.c_double(theta), _ptr(out),
                                          _ptr(wp), C.byref(err)), err)
        return out, wp

    def collision(self, ctx: Ctx, coeffs, params):
        c = _arr(coeffs); out = np.empty_like(c); err = MoErr(); cc = ctx.c()
        self._check(self.lib.mo_collision(C.byref(cc), _ptr(c), _ptr(_arr(params)), _ptr(out),
                                          C.byref(err)), err)
        return out

    # ------------------------------------------------------- field operations
    def residual(self, ctx: Ctx, g: Grid, coeffs, params):
        n = count(ctx.M)
        c = _arr(coeffs, (g.cells, n)); p = _arr(params, (g.cells, 4))
        out = np.empty_like(c); err = MoErr(); cc = ctx.c(); gg = g.c()
        self._check(self.lib.mo_residual(C.byref(cc), C.byref(gg), _ptr(c), _ptr(p), _ptr(out),
                                         C.byref(err)), err)
        return out

    def fast_sweep(self, ctx: Ctx, g: Grid, coeffs, params, rhs=None, sweep_order=None,
                   raise_errors=True):
        """Returns (coeffs, params, evals[, rc, msg]); inputs are not modified."""
        n = count(ctx.M)
        c = _arr(coeffs, (g.cells, n)).copy(); p = _arr(params, (g.cells, 4)).copy()
        rc_, rp_ = (None, None) if rhs is None else (_arr(rhs[0], (g.cells, n)), _arr(rhs[1], (g.cells, 4)))
        order = None if sweep_order is None else (C.c_int * 4)(*sweep_order)
        ev = C.c_longlong(0); err = MoErr(); cc = ctx.c(); gg = g.c()
        rc = self.lib.mo_fast_sweep(C.byref(cc), C.byref(gg), _ptr(c), _ptr(p), _ptr(rc_),
                                    _ptr(rp_), order, C.byref(ev), C.byref(err))
        if raise_errors:
            self._check(rc, err)
            return c, p, ev.value
        return c, p, ev.value, rc, err.msg.decode(errors="replace")

    def sweep_cells(self, ctx: Ctx, g: Grid, coeffs, params, cells, rhs=None):
        """sweep_cell for each (i, j) in order, IN PLACE on coeffs/params
        (C-contiguous float64 arrays).  Port only (test infrastructure)."""
        cl = np.ascontiguousarray(np.asarray(cells, dtype=np.int32).reshape(-1, 2))
        err = MoErr(); cc = ctx.c(); gg = g.c()
        rc_, rp_ = (None, None) if rhs is None else (rhs[0], rhs[1])
        self._check(self.lib.mo_sweep_cells(C.byref(cc), C.byref(gg), _ptr(coeffs), _ptr(params),
                                            _ptr(rc_), _ptr(rp_), cl.ctypes.data_as(_ip), len(cl),
                                            C.byref(err)), err)

    def total_mass(self, g: Grid, M, coeffs):
        gg = g.c()
        return self.lib.mo_total_mass(C.byref(gg), M, _ptr(_arr(coeffs)))

    def mass_correction(self, g: Grid, M, coeffs, target):
        c = _arr(coeffs).copy(); err = MoErr(); gg = g.c()
        self._check(self.lib.mo_mass_correction(C.byref(gg), M, _ptr(c), C.c_double(target),
                                                C.byref(err)), err)
        return c

    def restrict_solution(self, M, fine: Grid, fc, fp, coarse: Grid):
        n = count(M)
        cc = np.empty((coarse.cells, n)); cp = np.empty((coarse.cells, 4)); err = MoErr()
        fg = fine.c(); cg = coarse.c()
        self._check(self.lib.mo_restrict_solution(M, C.byref(fg), _ptr(_arr(fc)), _ptr(_arr(fp)),
                                                  C.byref(cg), _ptr(cc), _ptr(cp), C.byref(err)), err)
        return cc, cp

    def restrict_residual(self, M, fine: Grid, arr_c, arr_p, fine_params, coarse: Grid, coarse_params):
        n = count(M)
        out = np.empty((coarse.cells, n)); err = MoErr(); fg = fine.c(); cg = coarse.c()
        self._check(self.lib.mo_restrict_residual(M, C.byref(fg), _ptr(_arr(arr_c)), _ptr(_arr(arr_p)),
                                                  _ptr(_arr(fine_params)), C.byref(cg),
                                                  _ptr(_arr(coarse_params)), _ptr(out),
                                                  C.byref(err)), err)
        return out

    def fas_correct(self, M, fine: Grid, fc, fp, coarse: Grid, bc, bp, ac, ap):
        c = _arr(fc).copy(); p = _arr(fp).copy(); err = MoErr(); fg = fine.c(); cg = coarse.c()
        self._check(self.lib.mo_fas_correct(M, C.byref(fg), _ptr(c), _ptr(p), C.byref(cg),
                                            _ptr(_arr(bc)), _ptr(_arr(bp)), _ptr(_arr(ac)),
                                            _ptr(_arr(ap)), C.byref(err)), err)
        return c, p

    def residual_norm(self, M, g: Grid, res, field_params):
        gg = g.c()
        return self.lib.mo_residual_norm(M, C.byref(gg), _ptr(_arr(res)), _ptr(_arr(field_params)))

    def nmg_cycle(self, ctx: Ctx, g: Grid, coeffs, params, levels=0, s1=2, s2=2, s3=4, gamma=1):
        c = _arr(coeffs).copy(); p = _arr(params).copy(); w = C.c_longlong(0); err = MoErr()
        cc = ctx.c(); gg = g.c()
        self._check(self.lib.mo_nmg_cycle(C.byref(cc), C.byref(gg), _ptr(c), _ptr(p), levels, s1,
                                          s2, s3, gamma, C.byref(w), C.byref(err)), err)
        return c, p, w.value

    def euler_step(self, ctx: Ctx, g: Grid, coeffs, params, rhs=None):
        """residual + euler_step (single_level.cpp:74-97); rhs = (coeffs, params) or None."""
        c = _arr(coeffs).copy(); p = _arr(params).copy(); err = MoErr(); cc = ctx.c(); gg = g.c()
        if rhs is None:
            self._check(self.lib.mo_euler_step(C.byref(cc), C.byref(gg), _ptr(c), _ptr(p),
                                               C.byref(err)), err)
        else:
            self._check(self.lib.mo_euler_step_rhs(C.byref(cc), C.byref(gg), _ptr(c), _ptr(p),
                                                   _ptr(_arr(rhs[0])), _ptr(_arr(rhs[1])),
                                                   C.byref(err)), err)
        return c, p

    def solve_steady(self, ctx: Ctx, g: Grid, coeffs, params, solver=NMG, tol=1e-8,
                     max_iterations=0, levels=0, s1=2, s2=2, s3=4, gamma=1, history_cap=100000):
        """Returns (coeffs, params, report dict); report['rc'] / ['msg'] carry the
        NonConvergence / error mapping instead of raising."""
        c = _arr(coeffs).copy(); p = _arr(params).copy(); err = MoErr(); cc = ctx.c(); gg = g.c()
        hist = np.zeros(history_cap)
        rep = MoReport(0, 0, 0.0, 0.0, 0.0, 0, 0.0, 0, _ptr(hist), history_cap)
        rc = self.lib.mo_solve_steady(C.byref(cc), C.byref(gg), _ptr(c), _ptr(p), solver,
                                      C.c_double(tol), max_iterations, levels, s1, s2, s3, gamma,
                                      C.byref(rep), C.byref(err))
        hl = min(rep.history_len, history_cap)
        report = dict(rc=rc, msg=err.msg.decode(errors="replace"), converged=bool(rep.converged),
                      iterations=rep.iterations, r0_norm=rep.r0_norm, final_norm=rep.final_norm,
                      final_ratio=rep.final_ratio, work=rep.work, seconds=rep.seconds,
                      history=hist[:hl].copy())
        return c, p, report


def build(kind: str = "port") -> None:
    """Builds the restatement (always possible) or the reference (needs
    /root/reference) with oracle/Makefile."""
    target = "all" if kind == "port" else "ref"
    if kind != "port" and not os.path.isdir(REF_SRC):
        raise FileNotFoundError("reference sources absent; oracle/_ref must be prebuilt")
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def uniform_field(g: Grid, M: int, rho=1.0, u=(0.0, 0.0, 0.0), theta=1.0):
    """uniform_field + maxwellian_rep (grid.hpp:79-85, moment_rep.hpp:47-59)."""
    n = count(M)
    c = np.zeros((g.cells, n)); c[:, 0] = rho
    p = np.zeros((g.cells, 4)); p[:, 0:3] = u; p[:, 3] = theta
    return c, p
