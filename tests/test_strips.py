"""Multi-rank host layer of the strip partition (paper_2206_13164_b200/strips.py)
on CPU: world_size 2 over gloo, the collectives the GPU path uses (IPC
handle all-gather, barriers, the scalar reductions of total_mass and
residual_norm combined from per-strip values).  The per-strip values are the
oracle's own total_mass / residual_norm on each strip's sub-grid, so the
combination is checked against the oracle on the whole level.  The device
side of the partition (one kernel over all strips, bitwise equal to the
single-field sweep) is tests/test_gpu_strips.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import BGK, Grid, Oracle, c5_field, cavity_ctx

from paper_2206_13164_b200.strips import StripComm, combine_mass, combine_norm, strip_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def sub_grid(g: Grid, i0: int, i1: int) -> Grid:
    dx = g.dx[i0:i1].copy()
    return Grid(i1 - i0, g.ny, float(np.sum(dx)), g.Ly, dx, g.dy.copy(), g.xc[i0:i1].copy(), g.yc.copy())


def columns(a, g, i0, i1):
    return a.reshape(g.ny, g.nx, -1)[:, i0:i1].reshape(-1, a.shape[1])


def _worker(rank, world, port, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = StripComm(dist)
        # IPC handle exchange: every rank sees every rank's 320-byte handle
        mine = bytes([rank + 1]) * 320
        handles = comm.allgather_bytes(mine)
        ok_handles = [h == bytes([r + 1]) * 320 for r, h in enumerate(handles)]
        calls = []
        comm.fence(lambda: calls.append(1))
        # per-strip scalars on this rank's strip, combined across ranks
        M, nx, ny = 5, 96, 10
        g = Grid.uniform(nx, ny, 1.0, 0.7)
        b = strip_bounds(nx, world)
        i0, i1 = b[rank], b[rank + 1]
        O = Oracle("port")
        octx = cavity_ctx(M, 1, BGK, kn=0.1, lid=0.1)
        c, p = c5_field(nx, ny, M, seed=4)
        res = O.residual(octx, g, c, p)
        sg = sub_grid(g, i0, i1)
        mass = combine_mass(comm, [O.total_mass(sg, M, columns(c, g, i0, i1))])
        norm = combine_norm(comm, [(O.residual_norm(M, sg, columns(res, g, i0, i1), columns(p, g, i0, i1)), sg.Lx)],
                            g.Lx, g.Ly)
        if rank == 0:
            out_q.put((ok_handles, calls, b, mass, O.total_mass(g, M, c), norm, O.residual_norm(M, g, res, p)))
    finally:
        dist.destroy_process_group()


def test_strip_layer_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    try:
        ok_handles, calls, b, mass, want_mass, norm, want_norm = q.get(timeout=240)
    finally:
        for pr in procs:
            pr.join(timeout=60)
    assert all(ok_handles) and calls == [1]
    assert b == [0, 64, 96]
    assert mass == pytest.approx(want_mass, rel=1e-14)
    assert norm == pytest.approx(want_norm, rel=1e-13)


def test_strip_bounds():
    assert strip_bounds(2048, 1) == [0, 2048]
    assert strip_bounds(2048, 8) == [256 * k for k in range(9)]
    assert strip_bounds(160, 2) == [0, 96, 160]
    b = strip_bounds(2048, 3)
    assert b[-1] == 2048 and all((y - x) % 32 == 0 and y > x for x, y in zip(b, b[1:]))
    with pytest.raises(ValueError):
        strip_bounds(100, 2)
    with pytest.raises(ValueError):
        strip_bounds(64, 3)  # more ranks than bands
