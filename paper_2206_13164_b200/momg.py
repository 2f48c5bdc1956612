"""Python mirror of the reference's solver API over the C ABI (include/momg_gpu.h).

Names, argument meaning and error behaviour follow the reference's C++
interface (namespace momg, /root/reference/proj/include/momg/*.hpp):

    Grid2D.uniform            grid.hpp:18-33
    SolveContext              single_level.hpp:27-34 (+ Walls, CollisionModel,
                              GasParams, SpatialScheme, CflPolicy)
    CellField                 grid.hpp:54-85   (device-resident here)
    residual                  spatial.hpp:52-56
    fast_sweep_step           single_level.hpp:63-65
    total_mass/mass_correction single_level.hpp:68-73
    restrict_solution         multigrid.hpp:41
    restrict_residual         multigrid.hpp:45-47
    fas_correct               multigrid.hpp:52-53
    residual_norm             multigrid.hpp:67-68
    nmg_cycle                 multigrid.hpp:59-61
    solve_steady              multigrid.hpp:114-116

Errors raise the reference's exception types (types.hpp:20-57;
NonConvergence carries the partial SolveReport).  There is no CPU fallback:
without the built library or a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOMG_GPU_LIB") or os.path.join(HERE, "_lib", "libmomg_gpu.so")  # env: A/B builds
CSRC = os.path.join(HERE, "csrc")


# ------------------------------------------------------------------- errors
class Error(RuntimeError):
    """momg::Error (types.hpp:20)."""


class ConfigError(Error):
    """momg::ConfigError (types.hpp:26)."""


class NonphysicalState(Error):
    """momg::NonphysicalState (types.hpp:33)."""


class NonSpdTensor(Error):
    """momg::NonSpdTensor (types.hpp:46)."""


class SolverError(Error):
    """momg::SolverError (types.hpp:54)."""


class NonConvergence(Error):
    """momg::NonConvergence (multigrid.hpp:89-97); .report is the partial report."""

    def __init__(self, what: str, report: "SolveReport"):
        super().__init__(what)
        self.report = report


class DeviceUnavailable(Error):
    """No CUDA device / library: the product has no CPU fallback."""


_EXC = {1: NonphysicalState, 2: SolverError, 3: Error, 4: NonSpdTensor, 5: ConfigError,
        100: DeviceUnavailable, 101: Error, 102: ValueError}


class _Err(C.Structure):
    _fields_ = [("code", C.c_int), ("i", C.c_int), ("j", C.c_int), ("msg", C.c_char * 256)]


class _Grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("Lx", C.c_double), ("Ly", C.c_double),
                ("dx", C.POINTER(C.c_double)), ("dy", C.POINTER(C.c_double)),
                ("xc", C.POINTER(C.c_double)), ("yc", C.POINTER(C.c_double))]


class _Ctx(C.Structure):
    _fields_ = [("M", C.c_int), ("space_order", C.c_int), ("c_bound", C.c_double),
                ("cfl", C.c_double), ("cfl_c_bound", C.c_double), ("collision", C.c_int),
                ("prandtl", C.c_double), ("knudsen", C.c_double), ("viscosity_index", C.c_double),
                ("wall_speed", C.c_double * 4), ("wall_theta", C.c_double * 4),
                ("threads", C.c_int)]


class _Opts(C.Structure):
    _fields_ = [("kind", C.c_int), ("tol", C.c_double), ("max_iterations", C.c_int),
                ("levels", C.c_int), ("s1", C.c_int), ("s2", C.c_int), ("s3", C.c_int),
                ("gamma", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("r0_norm", C.c_double),
                ("final_norm", C.c_double), ("final_ratio", C.c_double), ("work", C.c_longlong),
                ("seconds", C.c_double), ("history_len", C.c_int),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int),
                ("history_seconds", C.POINTER(C.c_double))]


_lib = None


def build(extra: str = "", orders: str | None = None) -> str:
    """Compiles the sm_100a library in-tree (csrc/Makefile)."""
    cmd = ["make", "-s", "-j8", "-C", CSRC]
    if extra:
        cmd.append(f"EXTRA={extra}")
    if orders:
        cmd.append(f"ORDERS={orders}")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailable(f"{LIB_PATH} is not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.momg_max_hermite_root.restype = C.c_double
        L.momg_version.restype = C.c_char_p
        L.momg_get_stream.restype = C.c_void_p
        L.momg_launch_count.restype = C.c_longlong
        L.momg_graph_replays.restype = C.c_longlong
        _lib = L
    return _lib


def _raise(rc: int, err: _Err):
    if rc == 0:
        return
    cls = _EXC.get(rc, Error)
    msg = err.msg.decode(errors="replace")
    raise cls(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# -------------------------------------------------------------------- config
@dataclass
class Grid2D:
    """Grid2D (grid.hpp:12-37): per-cell sizes and centres."""
    nx: int
    ny: int
    Lx: float
    Ly: float
    dx: np.ndarray
    dy: np.ndarray
    xc: np.ndarray
    yc: np.ndarray

    @staticmethod
    def uniform(nx: int, ny: int, Lx: float = 1.0, Ly: float = 1.0) -> "Grid2D":
        if nx < 1 or ny < 1 or not Lx > 0 or not Ly > 0:
            raise ConfigError("Grid2D: cell counts and extents must be positive")
        return Grid2D(nx, ny, Lx, Ly, np.full(nx, Lx / nx), np.full(ny, Ly / ny),
                      np.array([(i + 0.5) * Lx / nx for i in range(nx)]),
                      np.array([(j + 0.5) * Ly / ny for j in range(ny)]))

    def area(self, i, j):
        return self.dx[i] * self.dy[j]

    def cells(self) -> int:
        return self.nx * self.ny

    def _c(self) -> _Grid:
        for a in ("dx", "dy", "xc", "yc"):
            setattr(self, a, np.ascontiguousarray(getattr(self, a), dtype=np.float64))
        return _Grid(self.nx, self.ny, self.Lx, self.Ly, _dp(self.dx), _dp(self.dy),
                     _dp(self.xc), _dp(self.yc))


@dataclass
class WallSpec:
    """grid.hpp:42-45"""
    speed: float = 0.0
    theta: float = 1.0


@dataclass
class Walls:
    left: WallSpec = field(default_factory=WallSpec)
    right: WallSpec = field(default_factory=WallSpec)
    bottom: WallSpec = field(default_factory=WallSpec)
    top: WallSpec = field(default_factory=WallSpec)


class CollisionKind(IntEnum):
    bgk = 0
    es_bgk = 1
    shakhov = 2


@dataclass
class CollisionModel:
    """collision.hpp:17-24"""
    kind: CollisionKind = CollisionKind.bgk
    prandtl: float = 1.0


@dataclass
class GasParams:
    """collision.hpp:29-33"""
    knudsen: float = 1.0
    viscosity_index: float = 0.81
    molecule_mass: float = 6.63e-26


def max_hermite_root(degree: int) -> float:
    """tables.cpp:22-41"""
    return lib().momg_max_hermite_root(degree)


@dataclass
class SpatialScheme:
    """spatial.hpp:16-22"""
    order: int = 1
    c_bound: float = 1.0

    @staticmethod
    def for_moment_order(moment_order: int, space_order: int) -> "SpatialScheme":
        if space_order not in (1, 2):
            raise ConfigError("SpatialScheme: reconstruction order must be 1 or 2")
        return SpatialScheme(space_order, max_hermite_root(moment_order + 1))


@dataclass
class CflPolicy:
    """single_level.hpp:13-16"""
    cfl: float = 0.9
    c_bound: float = 1.0


@dataclass
class SolveContext:
    """single_level.hpp:27-34"""
    walls: Walls = field(default_factory=Walls)
    model: CollisionModel = field(default_factory=CollisionModel)
    gas: GasParams = field(default_factory=GasParams)
    scheme: SpatialScheme = field(default_factory=SpatialScheme)
    cfl: CflPolicy = field(default_factory=CflPolicy)
    threads: int = 1

    def _c(self, M: int) -> _Ctx:
        w = self.walls
        return _Ctx(M, self.scheme.order, self.scheme.c_bound, self.cfl.cfl, self.cfl.c_bound,
                    int(self.model.kind), self.model.prandtl, self.gas.knudsen,
                    self.gas.viscosity_index,
                    (C.c_double * 4)(w.left.speed, w.right.speed, w.bottom.speed, w.top.speed),
                    (C.c_double * 4)(w.left.theta, w.right.theta, w.bottom.theta, w.top.theta),
                    self.threads)


@dataclass
class CyclePolicy:
    """multigrid.hpp:30-35"""
    s1: int = 2
    s2: int = 2
    s3: int = 4
    gamma: int = 1


class SolverKind(IntEnum):
    euler = 0
    fs = 1
    nmg = 2


@dataclass
class SolverOptions:
    """multigrid.hpp:101-107"""
    kind: SolverKind = SolverKind.nmg
    tol: float = 1e-8
    max_iterations: int = 0
    levels: int = 0
    cycle: CyclePolicy = field(default_factory=CyclePolicy)


@dataclass
class WorkStats:
    """single_level.hpp:38-40"""
    cell_evals: int = 0


@dataclass
class SolveReport:
    """multigrid.hpp:78-87 (history: rel_residual per iteration)"""
    converged: bool = False
    iterations: int = 0
    r0_norm: float = 0.0
    final_norm: float = 0.0
    final_ratio: float = 0.0
    work: int = 0
    seconds: float = 0.0
    history: list = field(default_factory=list)
    history_seconds: list = field(default_factory=list)  # HistoryEntry.seconds


def count(order: int) -> int:
    """IndexSet::count (multi_index.hpp:82-84)"""
    return (order + 1) * (order + 2) * (order + 3) // 6


# ------------------------------------------------------------------ fields
class CellField:
    """Device-resident CellField (grid.hpp:54-76): one grid level in HBM."""

    def __init__(self, grid: Grid2D, order: int):
        self.grid = grid
        self.order = order
        self.N = count(order)
        h = C.c_void_p()
        err = _Err()
        g = grid._c()
        _raise(lib().momg_field_create(C.byref(g), order, C.byref(h), C.byref(err)), err)
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and getattr(self, "_owned", True):
            _lib.momg_field_destroy(h)
            self._h = None

    @classmethod
    def _view(cls, grid: Grid2D, order: int, handle: int, keep) -> "CellField":
        """A field owned by another object (a strip of a StripSet)."""
        f = cls.__new__(cls)
        f.grid, f.order, f.N = grid, order, count(order)
        f._h = C.c_void_p(handle)
        f._owned = False
        f._keep = keep
        return f

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        return self.grid.cells()

    def upload(self, coeffs: np.ndarray, params: np.ndarray) -> "CellField":
        c = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(self.size(), self.N)
        p = np.ascontiguousarray(params, dtype=np.float64).reshape(self.size(), 4)
        err = _Err()
        _raise(lib().momg_field_upload(self._h, _dp(c), _dp(p), C.byref(err)), err)
        return self

    def download(self):
        c = np.empty((self.size(), self.N))
        p = np.empty((self.size(), 4))
        err = _Err()
        _raise(lib().momg_field_download(self._h, _dp(c), _dp(p), C.byref(err)), err)
        return c, p

    def copy(self) -> "CellField":
        out = CellField(self.grid, self.order)
        err = _Err()
        _raise(lib().momg_field_copy(out._h, self._h, C.byref(err)), err)
        return out

    @staticmethod
    def from_host(grid: Grid2D, order: int, coeffs, params) -> "CellField":
        return CellField(grid, order).upload(coeffs, params)


def uniform_field(grid: Grid2D, order: int, rho: float, u, theta: float) -> CellField:
    """grid.hpp:79-85"""
    f = CellField(grid, order)
    err = _Err()
    uu = (C.c_double * 3)(*u)
    _raise(lib().momg_field_fill_maxwellian(f._h, C.c_double(rho), uu, C.c_double(theta),
                                             C.byref(err)), err)
    return f


# ---------------------------------------------------------------- hot path
def residual(field: CellField, ctx: SolveContext) -> CellField:
    """spatial.cpp:135-159; result params = field params."""
    out = CellField(field.grid, field.order)
    err = _Err()
    c = ctx._c(field.order)
    _raise(lib().momg_residual(C.byref(c), field._h, out._h, C.byref(err)), err)
    return out


def fast_sweep_step(field: CellField, rhs: CellField | None, ctx: SolveContext,
                    work: WorkStats | None = None, sweep_order=(0, 1, 2, 3)) -> None:
    """single_level.cpp:121-166 (exact lexicographic Gauss-Seidel order)."""
    err = _Err()
    c = ctx._c(field.order)
    ev = C.c_longlong(0)
    order = (C.c_int * 4)(*sweep_order)
    rc = lib().momg_fast_sweep(C.byref(c), field._h, rhs._h if rhs is not None else None, order,
                               C.byref(ev), C.byref(err))
    if work is not None:
        work.cell_evals += ev.value
    _raise(rc, err)


def fast_sweep_residual(field: CellField, ctx: SolveContext, out: CellField | None = None,
                        work: WorkStats | None = None, sweep_order=(0, 1, 2, 3)) -> CellField:
    """fast_sweep_step (no rhs) then residual (the sequence of nmg_cycle,
    multigrid.cpp:170-176), fused into one launch where the band kernels
    apply; returns the residual field (params = cell params)."""
    out = out or CellField(field.grid, field.order)
    err = _Err()
    c = ctx._c(field.order)
    ev = C.c_longlong(0)
    order = (C.c_int * 4)(*sweep_order)
    rc = lib().momg_fast_sweep_residual(C.byref(c), field._h, order, out._h, C.byref(ev), C.byref(err))
    if work is not None:
        work.cell_evals += ev.value
    _raise(rc, err)
    return out


def euler_step(field: CellField, residuals: CellField | None, rhs: CellField | None,
               ctx: SolveContext) -> None:
    """single_level.cpp:74-97: f <- f + dt (R - rhs) with the single global dt
    (global_dt, :31-38), re-normalisation and the dt/2 retry.  `residuals` =
    residual(field, ctx) on the incoming field (None: evaluated here)."""
    err = _Err()
    c = ctx._c(field.order)
    _raise(lib().momg_euler_step(C.byref(c), field._h, residuals._h if residuals is not None else None,
                                 rhs._h if rhs is not None else None, C.byref(err)), err)


def total_mass(field: CellField) -> float:
    v = C.c_double(0)
    err = _Err()
    _raise(lib().momg_total_mass(field._h, C.byref(v), C.byref(err)), err)
    return v.value


def mass_correction(field: CellField, target_mass: float) -> None:
    err = _Err()
    _raise(lib().momg_mass_correction(field._h, C.c_double(target_mass), C.byref(err)), err)


def restrict_solution(fine: CellField, coarse: Grid2D) -> CellField:
    out = CellField(coarse, fine.order)
    err = _Err()
    _raise(lib().momg_restrict_solution(fine._h, out._h, C.byref(err)), err)
    return out


def restrict_residual(fine_arrays: CellField, fine: CellField, coarse: CellField) -> CellField:
    """fine_arrays carries its own params (single_level.hpp:42-45)."""
    out = CellField(coarse.grid, coarse.order)
    err = _Err()
    _raise(lib().momg_restrict_residual(fine_arrays._h, coarse._h, out._h, C.byref(err)), err)
    return out


def fas_correct(fine: CellField, coarse_before: CellField, coarse_after: CellField) -> None:
    err = _Err()
    _raise(lib().momg_fas_correct(fine._h, coarse_before._h, coarse_after._h, C.byref(err)), err)


def residual_norm(residuals: CellField, field: CellField) -> float:
    v = C.c_double(0)
    err = _Err()
    _raise(lib().momg_residual_norm(residuals._h, field._h, C.byref(v), C.byref(err)), err)
    return v.value


def residual_scale(field: CellField, ctx: SolveContext) -> float:
    v = C.c_double(0)
    err = _Err()
    c = ctx._c(field.order)
    _raise(lib().momg_residual_scale(C.byref(c), field._h, C.byref(v), C.byref(err)), err)
    return v.value


def nmg_cycle(field: CellField, ctx: SolveContext, levels: int = 0,
              policy: CyclePolicy | None = None, work: WorkStats | None = None) -> None:
    """One V-cycle (multigrid.cpp:166-200) on GridHierarchy::build(grid, levels)."""
    p = policy or CyclePolicy()
    err = _Err()
    c = ctx._c(field.order)
    w = C.c_longlong(0)
    rc = lib().momg_nmg_cycle(C.byref(c), field._h, levels, p.s1, p.s2, p.s3, p.gamma,
                              C.byref(w), C.byref(err))
    if work is not None:
        work.cell_evals += w.value
    _raise(rc, err)


def solve_steady(field: CellField, ctx: SolveContext, options: SolverOptions,
                 history_cap: int = 100000) -> SolveReport:
    """multigrid.cpp:243-320; raises NonConvergence(report) like the reference."""
    err = _Err()
    c = ctx._c(field.order)
    o = _Opts(int(options.kind), options.tol, options.max_iterations, options.levels,
              options.cycle.s1, options.cycle.s2, options.cycle.s3, options.cycle.gamma)
    hist = np.zeros(history_cap)
    secs = np.zeros(history_cap)
    rep = _Report(0, 0, 0.0, 0.0, 0.0, 0, 0.0, 0, _dp(hist), history_cap, _dp(secs))
    rc = lib().momg_solve_steady(C.byref(c), field._h, C.byref(o), C.byref(rep), C.byref(err))
    n = min(rep.history_len, history_cap)
    report = SolveReport(bool(rep.converged), rep.iterations, rep.r0_norm, rep.final_norm,
                         rep.final_ratio, rep.work, rep.seconds, list(hist[:n]), list(secs[:n]))
    if rc == 6:
        raise NonConvergence(err.msg.decode(errors="replace"), report)
    _raise(rc, err)
    return report


# --------------------------------------------------------- front-end output
class _Units(C.Structure):
    _fields_ = [("length", C.c_double), ("density", C.c_double), ("theta", C.c_double),
                ("speed", C.c_double), ("molecule_mass", C.c_double)]


def field_table(field: CellField, length: float, density: float, theta: float, speed: float,
                molecule_mass: float) -> np.ndarray:
    """export_field's table (scenario.cpp:372-399) evaluated on the device: per cell,
    row-major with j outermost, x y rho u1 u2 T sigma11 sigma12 sigma22 q1 q2 in
    laboratory units (momg_field_table).  NonphysicalState at a cell with rho <= 0."""
    out = np.empty((field.size(), 11))
    err = _Err()
    u = _Units(length, density, theta, speed, molecule_mass)
    rows = C.c_longlong(0)
    _raise(lib().momg_field_table(field._h, C.byref(u), _dp(out), C.byref(rows), C.byref(err)), err)
    return out


def export_field_tsv(field: CellField, path: str, length: float, density: float, theta: float,
                     speed: float, molecule_mass: float) -> None:
    """export_field (scenario.cpp:372-399): the table as TSV (%.17g) at path
    (momg_export_field; the formatting runs in the library on all host threads)."""
    err = _Err()
    u = _Units(length, density, theta, speed, molecule_mass)
    _raise(lib().momg_export_field(field._h, C.byref(u), os.fsencode(path), C.byref(err)), err)


# ------------------------------------------------------------------ strips
STRIP_HANDLE_BYTES = 320


def strip_grid(grid: Grid2D, i0: int, i1: int) -> Grid2D:
    """The sub-grid of columns [i0, i1) (a strip's own level)."""
    dx = np.ascontiguousarray(grid.dx[i0:i1], dtype=np.float64)
    return Grid2D(i1 - i0, grid.ny, float(np.sum(dx)), grid.Ly, dx, np.array(grid.dy, dtype=np.float64),
                  np.ascontiguousarray(grid.xc[i0:i1], dtype=np.float64), np.array(grid.yc, dtype=np.float64))


class StripSet:
    """momg_strips (include/momg_gpu.h): a level split into column strips
    [bounds[r], bounds[r+1]); this process owns strips first..last (device
    fields here), the others are attached from their owners' handles (CUDA
    IPC, peer memory).  fast_sweep_residual runs the owned strips' band tasks
    of the fused FS iteration + residual; with every strip owned it is the
    one-GPU emulation of all ranks in one kernel."""

    def __init__(self, grid: Grid2D, order: int, bounds, first: int = 0, last: int | None = None):
        self.grid, self.order = grid, order
        self.bounds = [int(b) for b in bounds]
        self.n = len(self.bounds) - 1
        self.first, self.last = first, (self.n - 1 if last is None else last)
        b = (C.c_int * (self.n + 1))(*self.bounds)
        h = C.c_void_p()
        err = _Err()
        g = grid._c()
        _raise(lib().momg_strips_create(C.byref(g), order, self.n, b, self.first, self.last, C.byref(h),
                                        C.byref(err)), err)
        self._h = h
        self._fields = {}
        for r in range(self.first, self.last + 1):
            fh, rh = C.c_void_p(), C.c_void_p()
            if lib().momg_strips_field(self._h, r, C.byref(fh), C.byref(rh)):
                raise Error("momg_strips_field failed")
            sg = strip_grid(grid, self.bounds[r], self.bounds[r + 1])
            self._fields[r] = (CellField._view(sg, order, fh.value, self), CellField._view(sg, order, rh.value, self))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.momg_strips_destroy(h)
            self._h = None

    def field(self, r: int) -> CellField:
        return self._fields[r][0]

    def residual_field(self, r: int) -> CellField:
        return self._fields[r][1]

    def export(self, r: int) -> bytes:
        buf = (C.c_char * STRIP_HANDLE_BYTES)()
        err = _Err()
        _raise(lib().momg_strips_export(self._h, r, buf, C.byref(err)), err)
        return bytes(buf)

    def attach(self, r: int, handle: bytes) -> None:
        buf = (C.c_char * STRIP_HANDLE_BYTES).from_buffer_copy(handle)
        err = _Err()
        _raise(lib().momg_strips_import(self._h, r, buf, C.byref(err)), err)

    def upload(self, coeffs: np.ndarray, params: np.ndarray) -> None:
        """Owned strips' columns of a global host field (reference order)."""
        n = count(self.order)
        c = np.asarray(coeffs).reshape(self.grid.ny, self.grid.nx, n)
        p = np.asarray(params).reshape(self.grid.ny, self.grid.nx, 4)
        for r, (f, _) in self._fields.items():
            i0, i1 = self.bounds[r], self.bounds[r + 1]
            f.upload(c[:, i0:i1].reshape(-1, n), p[:, i0:i1].reshape(-1, 4))

    def download(self, residual: bool = False):
        """Owned strips' columns assembled into global-layout arrays (other
        columns NaN)."""
        n = count(self.order)
        c = np.full((self.grid.ny, self.grid.nx, n), np.nan)
        p = np.full((self.grid.ny, self.grid.nx, 4), np.nan)
        for r, pair in self._fields.items():
            i0, i1 = self.bounds[r], self.bounds[r + 1]
            sc, sp = pair[1 if residual else 0].download()
            c[:, i0:i1] = sc.reshape(self.grid.ny, i1 - i0, n)
            p[:, i0:i1] = sp.reshape(self.grid.ny, i1 - i0, 4)
        return c.reshape(-1, n), p.reshape(-1, 4)

    def fast_sweep(self, ctx: SolveContext, iters: int = 1, sweep_order=(0, 1, 2, 3),
                   work: WorkStats | None = None):
        """`iters` (<= 4) consecutive fast_sweep_step calls over the partition, one launch."""
        err = _Err()
        c = ctx._c(self.order)
        ev = C.c_longlong(0)
        order = (C.c_int * 4)(*sweep_order)
        rc = lib().momg_strips_fast_sweep(C.byref(c), self._h, order, iters, C.byref(ev), C.byref(err))
        if work is not None:
            work.cell_evals += ev.value
        _raise(rc, err)

    def residual(self, ctx: SolveContext):
        """residual of the owned strips into their residual fields."""
        err = _Err()
        c = ctx._c(self.order)
        _raise(lib().momg_strips_residual(C.byref(c), self._h, C.byref(err)), err)

    def gather(self, which: int, full: CellField):
        err = _Err()
        _raise(lib().momg_strips_gather(self._h, which, full._h, C.byref(err)), err)

    def scatter(self, which: int, full: CellField):
        err = _Err()
        _raise(lib().momg_strips_scatter(self._h, which, full._h, C.byref(err)), err)

    def fast_sweep_residual(self, ctx: SolveContext, sweep_order=(0, 1, 2, 3), work: WorkStats | None = None):
        err = _Err()
        c = ctx._c(self.order)
        ev = C.c_longlong(0)
        order = (C.c_int * 4)(*sweep_order)
        rc = lib().momg_strips_fast_sweep_residual(C.byref(c), self._h, order, C.byref(ev), C.byref(err))
        if work is not None:
            work.cell_evals += ev.value
        _raise(rc, err)


def field_scale(field: CellField, factor: float) -> None:
    """coeffs *= factor (mass_correction's rescale with a caller-computed factor)."""
    err = _Err()
    _raise(lib().momg_field_scale(field._h, C.c_double(factor), C.byref(err)), err)


def nmg_cycle_rhs(field: CellField, rhs: CellField | None, ctx: SolveContext, levels: int = 0,
                  policy: CyclePolicy | None = None, work: WorkStats | None = None) -> None:
    """nmg_cycle for R(f) = rhs on GridHierarchy::build(field grid, levels)
    (multigrid.cpp:166-200), the coarse problem of an outer cycle."""
    p = policy or CyclePolicy()
    err = _Err()
    c = ctx._c(field.order)
    w = C.c_longlong(0)
    rc = lib().momg_nmg_cycle_rhs(C.byref(c), field._h, rhs._h if rhs is not None else None, levels, p.s1, p.s2,
                                  p.s3, p.gamma, C.byref(w), C.byref(err))
    if work is not None:
        work.cell_evals += w.value
    _raise(rc, err)


def synchronize() -> None:
    err = _Err()
    _raise(lib().momg_synchronize(C.byref(err)), err)


def launch_count() -> int:
    return lib().momg_launch_count()


def graph_replays() -> int:
    """solve_steady iterations replayed from a captured CUDA graph since load."""
    return lib().momg_graph_replays()


def cavity_context(M: int, space_order: int = 1, model: CollisionKind = CollisionKind.bgk,
                   knudsen: float = 0.1, lid: float = 0.1, prandtl: float = 1.0,
                   bottom_theta: float = 1.0) -> SolveContext:
    """Lid-driven / bottom-heated cavity in solver units (scenario.cpp:401-430):
    walls theta = 1 (bottom_theta at the bottom), top lid speed `lid`,
    cfl.c_bound = scheme.c_bound (scenario.cpp:421)."""
    scheme = SpatialScheme.for_moment_order(M, space_order)
    walls = Walls(WallSpec(0.0, 1.0), WallSpec(0.0, 1.0), WallSpec(0.0, bottom_theta),
                  WallSpec(lid, 1.0))
    return SolveContext(walls, CollisionModel(model, prandtl), GasParams(knudsen, 0.81),
                        scheme, CflPolicy(0.9, scheme.c_bound))


def set_sweep_mode(mode: str) -> None:
    """'persistent' (default: one dataflow kernel per fast_sweep_step; the band
    kernels for M <= 5), 'warp' (the same without the band kernels:
    thread-per-face / warp-per-cell) or 'diag' (one launch per
    anti-diagonal).  Results are identical up to rounding."""
    rc = lib().momg_set_sweep_mode({"diag": 0, "persistent": 1, "warp": 2}[mode])
    if rc:
        raise ValueError(mode)


def set_band_kernel(kind: str) -> None:
    """Band kernel of the first-order exact sweeps and residuals (M <= 5):
    'register' (default: one thread per face side, moment vectors in
    registers) or 'split' (each face cut 4 ways across warps through shared
    memory).  Results agree to rounding."""
    rc = lib().momg_set_band_kernel({"split": 0, "register": 1}[kind])
    if rc:
        raise ValueError(kind)
