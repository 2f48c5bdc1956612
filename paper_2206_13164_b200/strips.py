"""Row-strip partition of one grid level across ranks, and the pipelined
exact-order fast-sweeping schedule.

Rank r owns rows [j0, j1) (even heights, so 2x2 coarsening stays
strip-local).  The halo is h = 1 row at first order and h = 2 at second
order (the radius-2 cross of spatial.cpp:34-50 via the neighbour face states
of spatial.cpp:118-121).

fast_sweep_step (single_level.cpp:121-166) visits cells i-outer, j-inner in
four directions.  Across strips its Gauss-Seidel dependencies are carried by
the boundary rows:

* before each sweep every rank exchanges h boundary rows in both directions
  (old values: the post-previous-sweep state);
* in a j-ascending sweep, rows flow rank r-1 -> r; in a j-descending one
  r+1 -> r.  A rank walks column chunks of B columns in the sweep's i order;
  for each chunk it receives the upstream rank's h boundary rows of those
  columns (new values), updates its own cells of the chunk in serial order,
  and sends its own h boundary rows of the chunk downstream.

Every cell then sees exactly the neighbour versions of the serial order:
upstream rows are new (received after the upstream rank updated them),
downstream rows are old (copied before the sweep, and the downstream rank
cannot update them before receiving this rank's new rows).  The scheme is a
pipeline of depth = number of ranks; its collectives are point-to-point
send/recv of h x B x (N + 4) doubles (torch.distributed: NCCL on GPUs,
gloo in the CPU tests).  The per-cell update is a pluggable backend.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

KSWEEP_DIRS = [(True, True), (False, True), (False, False), (True, False)]  # single_level.cpp:116-117


@dataclass
class StripPartition:
    nx: int
    ny: int
    nranks: int
    order: int  # spatial order: halo rows = order

    def __post_init__(self):
        if self.ny % (2 * self.nranks) != 0 and self.nranks > 1:
            # even strip heights keep 2x2 coarsening strip-local
            raise ValueError("ny must be divisible by 2 * nranks")
        base = self.ny // self.nranks
        self.rows = [(r * base, (r + 1) * base) for r in range(self.nranks)]
        self.halo = 2 if self.order == 2 else 1

    def owner(self, j: int) -> int:
        for r, (a, b) in enumerate(self.rows):
            if a <= j < b:
                return r
        raise IndexError(j)

    def chunks(self, i_up: bool, B: int):
        cols = list(range(self.nx)) if i_up else list(range(self.nx - 1, -1, -1))
        return [cols[k:k + B] for k in range(0, self.nx, B)]

    def own_cells(self, rank: int, cols: Sequence[int], j_up: bool):
        """Own cells of column chunk `cols` in the serial order (i-outer,
        j-inner in the sweep's j direction)."""
        j0, j1 = self.rows[rank]
        js = range(j0, j1) if j_up else range(j1 - 1, j0 - 1, -1)
        return [(i, j) for i in cols for j in js]

    def boundary_rows(self, rank: int, toward_high: bool):
        """The h own rows adjacent to the neighbour above (toward_high) or below."""
        j0, j1 = self.rows[rank]
        h = self.halo
        return list(range(j1 - h, j1)) if toward_high else list(range(j0, j0 + h))

    def halo_rows(self, rank: int, from_high: bool):
        j0, j1 = self.rows[rank]
        h = self.halo
        rows = list(range(j1, j1 + h)) if from_high else list(range(j0 - h, j0))
        return [j for j in rows if 0 <= j < self.ny]


class Exchange:
    """Point-to-point row exchange over torch.distributed."""

    def __init__(self, dist):
        self.dist = dist

    def send(self, arr: np.ndarray, dst: int):
        import torch
        self.dist.send(torch.from_numpy(np.ascontiguousarray(arr)), dst)

    def recv(self, shape, src: int) -> np.ndarray:
        import torch
        t = torch.empty(shape, dtype=torch.float64)
        self.dist.recv(t, src)
        return t.numpy()

    def isend(self, arr: np.ndarray, dst: int):
        import torch
        return self.dist.isend(torch.from_numpy(np.ascontiguousarray(arr)), dst)

    def irecv(self, shape, src: int):
        import torch
        t = torch.empty(shape, dtype=torch.float64)
        return t, self.dist.irecv(t, src)


def _rows_pack(coeffs, params, nx, rows, cols):
    idx = np.array([j * nx + i for j in rows for i in cols], dtype=np.int64)
    return np.concatenate([coeffs[idx], params[idx]], axis=1)


def _rows_unpack(buf, coeffs, params, nx, rows, cols):
    idx = np.array([j * nx + i for j in rows for i in cols], dtype=np.int64)
    n = coeffs.shape[1]
    coeffs[idx] = buf[:, :n]
    params[idx] = buf[:, n:]


def exchange_halos(part: StripPartition, rank: int, ex: Exchange, coeffs, params):
    """Old-value halo exchange in both directions (all columns), non-blocking."""
    cols = list(range(part.nx))
    n = coeffs.shape[1] + 4
    reqs, recvs = [], []
    for peer, high in ((rank + 1, True), (rank - 1, False)):
        if not (0 <= peer < part.nranks):
            continue
        rows_in = part.halo_rows(rank, from_high=high)
        t, rq = ex.irecv((len(rows_in) * part.nx, n), peer)
        recvs.append((t, rq, rows_in))
        reqs.append(ex.isend(_rows_pack(coeffs, params, part.nx, part.boundary_rows(rank, high), cols), peer))
    for t, rq, rows_in in recvs:
        rq.wait()
        _rows_unpack(t.numpy(), coeffs, params, part.nx, rows_in, cols)
    for rq in reqs:
        rq.wait()


def strip_fast_sweep(part: StripPartition, rank: int, ex: Exchange, coeffs: np.ndarray,
                     params: np.ndarray, update_cells: Callable, sweep_order=(0, 1, 2, 3),
                     chunk: int = 8):
    """One fast_sweep_step of this rank's strip in the exact serial GS order.
    `coeffs`/`params` are global-size arrays of which this rank's strip (and
    halo, after the exchanges) is current; update_cells(list of (i, j))
    applies sweep_cell in order, in place."""
    n = coeffs.shape[1] + 4
    for s in sweep_order:
        i_up, j_up = KSWEEP_DIRS[s]
        exchange_halos(part, rank, ex, coeffs, params)
        upstream = rank - 1 if j_up else rank + 1
        downstream = rank + 1 if j_up else rank - 1
        has_up = 0 <= upstream < part.nranks
        has_down = 0 <= downstream < part.nranks
        for cols in part.chunks(i_up, chunk):
            if has_up:
                rows = part.halo_rows(rank, from_high=not j_up)
                buf = ex.recv((len(rows) * len(cols), n), upstream)
                _rows_unpack(buf, coeffs, params, part.nx, rows, cols)
            update_cells(part.own_cells(rank, cols, j_up))
            if has_down:
                rows = part.boundary_rows(rank, toward_high=j_up)
                ex.send(_rows_pack(coeffs, params, part.nx, rows, cols), downstream)


def gather_strips(part: StripPartition, rank: int, ex: Exchange, coeffs, params):
    """Assembles the full field on rank 0 (returns None elsewhere)."""
    n = coeffs.shape[1] + 4
    cols = list(range(part.nx))
    if rank != 0:
        j0, j1 = part.rows[rank]
        ex.send(_rows_pack(coeffs, params, part.nx, list(range(j0, j1)), cols), 0)
        return None
    c, p = coeffs.copy(), params.copy()
    for r in range(1, part.nranks):
        j0, j1 = part.rows[r]
        buf = ex.recv(((j1 - j0) * part.nx, n), r)
        _rows_unpack(buf, c, p, part.nx, list(range(j0, j1)), cols)
    return c, p
