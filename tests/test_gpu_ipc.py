"""The multi-process plumbing of the strip partition on one GPU: two
processes (ranks over gloo), each owning one strip, exchange CUDA IPC handles
(StripLevel: momg_strips_export / momg_strips_import) and then use the peer
strip's memory: a gather of the whole level (momg_strips_gather reads the
peer strip through its IPC mapping) and the strip residual (the halo columns
come from the peer strip) must equal the single-field results bit for bit.
Only operations that do not wait on the other rank run here: two ranks whose
kernels poll each other must not share one GPU (B200_PROFILING.md); the
cross-rank sweep itself is covered by the one-process emulation
(test_gpu_strips.py), which runs the same kernel over the same strip tables."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from helpers import BGK, Grid, c5_field, cavity_ctx
    from paper_2206_13164_b200 import momg
    from paper_2206_13164_b200.strips import StripComm, StripLevel
    from test_gpu_parity import mctx, mgrid
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        M, nx, ny = 5, 128, 24
        g = Grid.uniform(nx, ny)
        c, p = c5_field(nx, ny, M, seed=77)
        comm = StripComm(dist)
        level = StripLevel(momg, mgrid(g), M, comm)
        level.upload(c, p)
        comm.fence(momg.synchronize)
        if rank == 0:  # the whole level, half of it read from the peer process
            full = momg.CellField(mgrid(g), M)
            level.set.gather(0, full)
            gc, gp = full.download()
            out["gather"] = bool(np.array_equal(gc, c) and np.array_equal(gp, p))
        for order in (1, 2):  # strip residual with peer halo columns
            ctx = mctx(cavity_ctx(M, order, BGK, kn=0.1, lid=0.1))
            level.set.residual(ctx)
            rc, rp = level.set.download(residual=True)
            single = momg.CellField.from_host(mgrid(g), M, c, p)
            want, wp = momg.residual(single, ctx).download()
            b = level.bounds
            cols = np.zeros((ny, nx), bool)
            cols[:, b[rank]:b[rank + 1]] = True
            cols = cols.ravel()
            out[f"residual_o{order}"] = bool(np.array_equal(rc[cols], want[cols]) and np.array_equal(rp[cols], wp[cols]))
        comm.fence(momg.synchronize)
    except Exception as e:  # reported by the parent
        out["error"] = repr(e)
    finally:
        q.put((rank, out))
        dist.destroy_process_group()


def test_strips_across_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    try:
        res = dict(q.get(timeout=180) for _ in range(2))
    finally:
        for pr in procs:
            pr.join(timeout=60)
    assert not any("error" in r for r in res.values()), res
    assert res[0]["gather"]
    for r in (0, 1):
        assert res[r]["residual_o1"] and res[r]["residual_o2"], res
