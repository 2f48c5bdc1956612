"""Row-strip multi-rank path (world_size 2, gloo, CPU): the pipelined
exact-order sweep over strips reproduces the serial fast_sweep_step bit for
bit (per-cell updates by the CPU oracle), for first and second order and a
non-empty rhs; the halo exchange reproduces the serial residual."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import BGK, SHAKHOV, Grid, Oracle, cavity_ctx, smooth_field


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_q):
    import torch.distributed as dist

    from paper_2206_13164_b200.strips import Exchange, StripPartition, gather_strips, strip_fast_sweep
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M, order, model, nx, ny, use_rhs, chunk = case
        O = Oracle("port")
        g = Grid.uniform(nx, ny)
        ctx = cavity_ctx(M, order, model, kn=0.3, prandtl=2.0 / 3.0 if model == SHAKHOV else 1.0,
                         bottom_theta=1.2)
        c, p = smooth_field(g, M, seed=nx + ny + M, amp=0.08)
        rhs = (c * 1e-3, p.copy()) if use_rhs else None
        part = StripPartition(nx, ny, world, order)
        ex = Exchange(dist)
        cc, pp = c.copy(), p.copy()

        def update(cells):
            O.sweep_cells(ctx, g, cc, pp, cells, rhs=rhs)

        strip_fast_sweep(part, rank, ex, cc, pp, update, chunk=chunk)
        full = gather_strips(part, rank, ex, cc, pp)
        if rank == 0:
            want_c, want_p, _ = O.fast_sweep(ctx, g, c, p, rhs=rhs)
            out_q.put((bool(np.array_equal(full[0], want_c)), bool(np.array_equal(full[1], want_p)),
                       float(np.max(np.abs(full[0] - want_c)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (3, 1, BGK, 10, 8, False, 3),
    (3, 2, BGK, 9, 12, False, 4),
    (5, 2, SHAKHOV, 8, 8, True, 8),
])
def test_strip_sweep_matches_serial(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    try:
        eq_c, eq_p, diff = q.get(timeout=240)
    finally:
        for pr in procs:
            pr.join(timeout=60)
    assert eq_c and eq_p, diff


def test_partition_geometry():
    from paper_2206_13164_b200.strips import StripPartition
    part = StripPartition(16, 16, 4, 2)
    assert part.rows == [(0, 4), (4, 8), (8, 12), (12, 16)]
    assert part.halo == 2
    assert part.halo_rows(0, from_high=False) == []
    assert part.halo_rows(1, from_high=False) == [2, 3]
    assert part.boundary_rows(1, toward_high=True) == [6, 7]
    with pytest.raises(ValueError):
        StripPartition(16, 14, 4, 1)
