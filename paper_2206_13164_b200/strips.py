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

    def __init__(self, momg, grid, order: int, comm: StripComm, emulate_ranks: int | None = None):
        self.momg, self.grid, self.order, self.comm = momg, grid, order, comm
        nr = emulate_ranks if comm.world == 1 else comm.world
        self.bounds = strip_bounds(grid.nx, nr if nr else 1)
        if comm.world == 1:
            self.owned = list(range(len(self.bounds) - 1))
            self.set = momg.StripSet(grid, order, self.bounds)
        else:
            r = comm.rank
            self.owned = [r]
            self.set = momg.StripSet(grid, order, self.bounds, first=r, last=r)
            handles = comm.allgather_bytes(self.set.export(r))
            for peer in (r - 1, r + 1):
                if 0 <= peer < comm.world:
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
