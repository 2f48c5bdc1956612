"""Multi-GPU host layer: one process per GPU, a level split into column
strips, one strip per rank.

The device side is momg_strips (include/momg_gpu.h, csrc/strips.cu): every
rank allocates its strip, exports CUDA IPC handles of its arrays, and
attaches its neighbours' strips as peer memory (NVLink / NVSwitch).  The
fused FS iteration + residual (fast_sweep_step then residual, the sequence of
nmg_cycle multigrid.cpp:170-176 and of the C5 step) then runs each rank's
band tasks; a task of the first band of a strip polls the counter of the
neighbour strip's halo cell in peer memory and loads the cell from there, so
the exact Gauss-Seidel wavefront (single_level.cpp:121-166) pipelines across
ranks with no collective on the data path.  Everything else in the C5 step
is strip-local: strip widths are multiples of 32 (even), so restriction
(multigrid.cpp:67-142) and the FAS correction (:144-164) of a strip only touch
its own cells.  The scalar reductions of the solver are combined here:
total_mass (single_level.cpp:168-174) is a sum of per-strip sums;
residual_norm (multigrid.cpp:202-218) a root of the summed per-strip squares.

Ordering between ranks: a strip is only written by an operation other than
the fused sweep (FAS, mass correction, uploads) while no rank is inside the
fused sweep, so the sweep call is bracketed by a stream sync + barrier on
both sides (StripComm.fence).

StripComm is torch.distributed (NCCL on the GPU box, gloo in the CPU tests)
or a single process (world 1: every strip owned here, the one-GPU emulation
of all ranks in one kernel).
"""
from __future__ import annotations

import math
from typing import Sequence

BAND = 32  # columns of one band task of the band kernels


def strip_bounds(nx: int, nranks: int, band: int = BAND) -> list[int]:
    """Column bounds of nranks strips of whole bands, as even as the bands
    allow (the first nx/band % nranks strips get one band more)."""
    if nx % band:
        raise ValueError(f"nx = {nx} must be a multiple of the band width {band}")
    nb = nx // band
    if not 1 <= nranks <= min(nb, 8):
        raise ValueError(f"1 <= ranks <= min(bands = {nb}, 8)")
    q, r = divmod(nb, nranks)
    out = [0]
    for k in range(nranks):
        out.append(out[-1] + (q + (1 if k < r else 0)) * band)
    return out


class StripComm:
    """The few collectives the strip layer needs, over torch.distributed
    (dist=None: one process)."""

    def __init__(self, dist=None, device=None):
        self.dist = dist
        self.device = device
        self.rank = dist.get_rank() if dist else 0
        self.world = dist.get_world_size() if dist else 1

    def fence(self, sync=None):
        """Everything this rank queued is done and every rank got here."""
        if sync:
            sync()
        if self.dist:
            self.dist.barrier()

    def allgather_bytes(self, b: bytes) -> list[bytes]:
        if not self.dist:
            return [b]
        out = [None] * self.world
        self.dist.all_gather_object(out, b)
        return out

    def allreduce_sum(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t)
        return float(t.item())

    def allreduce_max(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def combine_mass(comm: StripComm, local_masses: Sequence[float]) -> float:
    """total_mass of the whole level: sum of rho * area over every strip."""
    return comm.allreduce_sum(math.fsum(local_masses))


def combine_norm(comm: StripComm, local: Sequence[tuple[float, float]], Lx: float, Ly: float) -> float:
    """residual_norm of the whole level from per-strip (norm, strip Lx):
    each strip's norm is sqrt(S_r / (Lx_r Ly)) over its own cells."""
    s = math.fsum(n * n * lx * Ly for n, lx in local)
    return math.sqrt(comm.allreduce_sum(s) / (Lx * Ly))


class StripLevel:
    """One level of a rank-partitioned field: this rank's strip on its GPU
    (all strips when world == 1), neighbours attached over IPC."""

    def __init__(self, momg, grid, order: int, comm: StripComm, emulate_ranks: int | None = None,
                 bounds: Sequence[int] | None = None, band: int = BAND):
        self.momg, self.grid, self.order, self.comm = momg, grid, order, comm
        nr = emulate_ranks if comm.world == 1 else comm.world
        self.bounds = list(bounds) if bounds is not None else strip_bounds(grid.nx, nr if nr else 1, band)
        if comm.world == 1:
            self.owned = list(range(len(self.bounds) - 1))
            self.set = momg.StripSet(grid, order, self.bounds)
        else:
            r = comm.rank
            self.owned = [r]
            self.set = momg.StripSet(grid, order, self.bounds, first=r, last=r)
            handles = comm.allgather_bytes(self.set.export(r))
            # every peer strip (the sweep needs the neighbours, a gather all)
            for peer in range(comm.world):
                if peer != r:
                    self.set.attach(peer, handles[peer])

    def field(self, r):
        return self.set.field(r)

    def residual_field(self, r):
        return self.set.residual_field(r)

    def upload(self, coeffs, params):
        self.set.upload(coeffs, params)

    def sweep_residual(self, ctx, sweep_order=(0, 1, 2, 3), work=None, fence: bool = True):
        """fast_sweep_step + residual over the whole partition (every rank
        calls it in the same sequence)."""
        sync = self.momg.synchronize
        if fence:
            self.comm.fence(sync)
        self.set.fast_sweep_residual(ctx, sweep_order, work)
        if fence:
            self.comm.fence(sync)

    def total_mass(self) -> float:
        return combine_mass(self.comm, [self.momg.total_mass(self.field(r)) for r in self.owned])

    def residual_norm(self) -> float:
        loc = [(self.momg.residual_norm(self.residual_field(r), self.field(r)), self.field(r).grid.Lx)
               for r in self.owned]
        return combine_norm(self.comm, loc, self.grid.Lx, self.grid.Ly)


def coarse_grid(momg, g):
    """coarsen (multigrid.cpp:12-35): 2x2 agglomeration of a Grid2D."""
    import numpy as np
    dx = np.asarray(g.dx[0::2]) + np.asarray(g.dx[1::2])
    dy = np.asarray(g.dy[0::2]) + np.asarray(g.dy[1::2])
    return momg.Grid2D(g.nx // 2, g.ny // 2, g.Lx, g.Ly, dx, dy, np.cumsum(dx) - 0.5 * dx, np.cumsum(dy) - 0.5 * dy)


class StripSolver:
    """solve_steady (multigrid.cpp:243-320) with the NMG V-cycle (:166-200)
    whose FINEST level is strip-partitioned across the ranks and whose
    coarser levels are agglomerated on every rank: each rank restricts its
    strip, the coarse strips are gathered (peer memory) into a full coarse
    level on every rank, every rank runs the identical coarse cycle
    (momg_nmg_cycle_rhs, deterministic), and each rank prolongs (FAS) into
    its own strip.  The finest level holds ~3/4 of the work; the coarse
    levels are small.  Strip widths are multiples of 64 so the coarse strips
    are whole 32-column bands too.  The operation sequence is the single-field
    driver's (driver.cu), so the result equals a one-GPU solve up to the
    summation order of the combined mass and norm."""

    def __init__(self, momg, grid, order: int, comm: StripComm, levels: int, policy=None,
                 emulate_ranks: int | None = None):
        self.momg, self.comm, self.levels = momg, comm, levels
        self.policy = policy or momg.CyclePolicy()
        self.fine = StripLevel(momg, grid, order, comm, emulate_ranks, band=2 * BAND)
        cg = coarse_grid(momg, grid)
        self.coarse = StripLevel(momg, cg, order, comm, bounds=[b // 2 for b in self.fine.bounds])
        self.cgrid = cg
        self.Fc, self.Fb = momg.CellField(cg, order), momg.CellField(cg, order)
        self.crhs, self.cres = momg.CellField(cg, order), momg.CellField(cg, order)
        self.work = momg.WorkStats()

    def _fence(self):
        self.comm.fence(self.momg.synchronize)

    def _sweeps(self, ctx, n):
        while n > 0:
            k = min(n, 4)
            self._fence()
            self.fine.set.fast_sweep(ctx, k, work=self.work)
            n -= k
        self._fence()

    def _call(self, name, *args):
        m = self.momg
        err = m._Err()
        m._raise(getattr(m.lib(), name)(*[a.handle if hasattr(a, "handle") else a for a in args], m.C.byref(err)), err)

    def cycle(self, ctx):
        m, f, c, pol = self.momg, self.fine, self.coarse, self.policy
        self._sweeps(ctx, pol.s1)
        f.set.residual(ctx)
        for r in f.owned:
            fr, rr = f.field(r), f.residual_field(r)
            self._call("momg_defect", rr, None, rr)
            self._call("momg_restrict_solution", fr, c.field(r))
            self._call("momg_restrict_residual", rr, c.field(r), c.residual_field(r))
        self._fence()
        c.set.gather(0, self.Fc)
        c.set.gather(1, self.crhs)
        self._call("momg_field_copy", self.Fb, self.Fc)
        self._res(ctx)
        self._call("momg_axpy", self.crhs, self.cres)
        for _ in range(pol.gamma):
            m.nmg_cycle_rhs(self.Fc, self.crhs, ctx, self.levels - 1, pol, self.work)
        c.set.scatter(0, self.Fc)
        c.set.scatter(1, self.Fb)
        for r in f.owned:
            self._call("momg_fas_correct", f.field(r), c.residual_field(r), c.field(r))
        self._sweeps(ctx, pol.s2)

    def _res(self, ctx):
        m = self.momg
        err = m._Err()
        cc = ctx._c(self.Fc.order)
        m._raise(m.lib().momg_residual(m.C.byref(cc), self.Fc.handle, self.cres.handle, m.C.byref(err)), err)
        return self.cres

    def norm(self, ctx):
        self.fine.set.residual(ctx)
        return self.fine.residual_norm()

    def solve(self, ctx, tol: float = 1e-8, max_iterations: int = 0):
        """The loop of solve_steady; returns (converged, iterations, history)."""
        m = self.momg
        cap = max_iterations or 200
        self._fence()
        r0 = self.norm(ctx)
        scale = self.comm.allreduce_max(max(m.residual_scale(self.fine.field(r), ctx) for r in self.fine.owned))
        if r0 <= 1e-12 * scale:
            return True, 0, []
        target = self.fine.total_mass()
        hist = []
        for n in range(1, cap + 1):
            try:
                self.cycle(ctx)
                current = self.fine.total_mass()
                if not (current > 0.0) or not math.isfinite(current):
                    raise m.NonphysicalState(f"mass_correction: nonpositive total mass {current}")
                for r in self.fine.owned:
                    m.field_scale(self.fine.field(r), target / current)
                self._fence()
                ratio = self.norm(ctx) / r0
            except (m.SolverError, m.NonphysicalState) as e:
                raise m.NonConvergence(f"iteration step failed: {e}",
                                       m.SolveReport(False, n - 1, r0, 0.0, 0.0, self.work.cell_evals, 0.0, hist))
            hist.append(ratio)
            if not math.isfinite(ratio) or ratio > 1e6:
                raise m.NonConvergence(f"residual diverged: ratio {ratio} at iteration {n}",
                                       m.SolveReport(False, n, r0, 0.0, ratio, self.work.cell_evals, 0.0, hist))
            if ratio <= tol:
                return True, n, hist
        return False, cap, hist
