"""Benchmark of the B200 NMG / fast-sweeping hot path (BASELINE.json metric:
smoother cell-updates/s (FP64) + NMG wall time to residual 1e-8).

Workload (BASELINE.json configs[4], "C5"): 2048x2048 cells, M = 5 (56
moments/cell), FP64, seeded random field (rho~U[0.9,1.1], u_x,u_y~N(0,0.05),
u_z=0, theta~U[0.9,1.1], f_alpha~N(0,1e-3)*0.5^|alpha|), diffuse walls at
theta = 1, BGK Kn = 0.1, first-order FV.  One step = one full four-direction
fast-sweeping iteration (the exact-order dataflow kernel) + one residual + one
restrict/prolong pair (restrict_solution, restrict_residual of the defect,
fas_correct with after = before + seeded delta).  value = 4*nx*ny smoother
cell updates / step time (residual and transfer time included).

Default run also reports NMG time-to-1e-8 on C2 (128^2, M = 5, second order,
NMG over 4 levels) as "nmg".  --impl reference times the reference's own CPU
implementation (oracle/_ref: /root/reference compiled against the shims,
OpenMP blocked FS with every host thread) on a bounded sample of the same
workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# the FS iteration and the residual of a step as one launch (momg_fast_sweep_residual)
FUSED = True
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FLOPS_PER_UPDATE_C5 = 16290.0  # M=5, order 1, 3-axis shifts (C5)
FLOPS_RESIDUAL_C5 = 9400.0     # residual per cell, M=5, 3-axis (C5)
BYTES_PER_UPDATE_C5 = 960.0    # 2*(N+4)*8 minimum HBM bytes per cell update


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nx", type=int, default=2048)
    ap.add_argument("--M", type=int, default=5)
    ap.add_argument("--order", type=int, default=1)
    ap.add_argument("--seed", type=int, default=2206)
    ap.add_argument("--no-nmg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=128)
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--strips", type=int, default=0,
                    help="world 1: run the strip-partitioned path with this many strips in one process "
                         "(the one-GPU emulation of the ranks); world > 1 always runs one strip per rank")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.path = f"/tmp/momg_clocks_{os.getpid()}.csv"
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx = max(mx, float(f[2]))
                except ValueError:
                    continue
                for n, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def band_traffic(nx):
    """DRAM bytes (read + write) per launch of the band sweep measured by ncu at
    this grid size (profiles/r2_k8_traffic.json, from tools/profile_k8.sh; the
    round-1 figure of the split kernel as the fallback), or None."""
    for name in ("r2_k8_traffic.json", "r1_band_traffic.json"):
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", name)))
            if d.get("nx") == nx:
                return d["bytes_per_launch"]
        except (OSError, ValueError, KeyError):
            pass
    return None


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["fp64_tflops"], "measured DFMA probe (profiles/fp64_peak.json, tools/fp64_peak.cu)"
    return 37.0, "nominal B200 FP64 (unmeasured fallback)"


# --------------------------------------------------------------- CPU legs
def cpu_sample_rate(kind: str, nx: int, M: int, order: int, threads: int, seed: int,
                    steps: int = 1):
    """Cell-updates/s of the CPU implementation on an nx x nx sample of the
    C5 workload (FS + residual + restrict pair per step, like the GPU step)."""
    from oracle.api import BGK, Ctx, Grid, Oracle
    from paper_2206_13164_b200.synthetic import c5_field

    o = Oracle(kind)
    g = Grid.uniform(nx, nx)
    cg = g.coarsen()
    cb = o.max_hermite_root(M + 1)
    ctx = Ctx(M=M, space_order=order, c_bound=cb, cfl=0.9, cfl_c_bound=cb, collision=BGK,
              knudsen=0.1, threads=threads)
    c, p = c5_field(nx, nx, M, seed=seed)
    t0 = time.perf_counter()
    for _ in range(steps):
        c, p, _ = o.fast_sweep(ctx, g, c, p)
        res = o.residual(ctx, g, c, p)
        cc, cp = o.restrict_solution(M, g, c, p, cg)
        o.restrict_residual(M, g, -res, p, p, cg, cp)
        after = cc.copy()
        after[:, 10:] += 1e-6
        c, p = o.fas_correct(M, g, c, p, cg, cc, cp, after, cp)
    dt = time.perf_counter() - t0
    return 4.0 * nx * nx * steps / dt, dt


def c5_config(nx, M, order):
    """The workload (BASELINE configs[4]) both arms report in `config`; how
    each arm runs it goes into `impl_detail`."""
    N = (M + 1) * (M + 2) * (M + 3) // 6
    return {"workload": f"C5: {nx}x{nx}, M={M} ({N} moments), order {order}, BGK Kn 0.1, "
                        "walls theta=1; step = FS iteration + residual + restrict/prolong pair",
            "global_cells": nx * nx,
            "l2": "inputs larger than L2 (field %.2f GB)" % (nx * nx * (N + 4) * 8 / 1e9)}


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    metric = "smoother cell-updates/s (FP64)"
    nx = 128
    from oracle.api import REF_LIB
    if not os.path.exists(REF_LIB):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libmomg_ref.so not built (needs /root/reference)"}))
        return
    rates = []
    for s in range(a.warmup + a.steps):
        r, dt = cpu_sample_rate("reference", nx, a.M, a.order, threads, a.seed + s)
        if s >= a.warmup:
            rates.append((r, dt))
    value = statistics.median(r for r, _ in rates)
    # measured: wall time of one sample step (what this run spent per step);
    # the full-size equivalent is an extrapolation and says so
    ms = 1e3 * statistics.median(dt for _, dt in rates)
    line = {"impl": "reference", "metric": metric, "value": value, "unit": "cell-updates/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "ms_per_step_measured_on": f"{nx}x{nx} sample step (FS + residual + restrict pair)",
            "extrapolated_full_step_ms": 1e3 * 4 * a.nx * a.nx / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": c5_config(a.nx, a.M, a.order),
            "impl_detail": {"fs": "reference OpenMP blocked fast_sweep_step (threads=%d, non-exact order)" % threads,
                            "sample": f"the rate is measured on a {nx}x{nx} sub-field of the workload (a CPU "
                                      "sweep's cost per cell update does not depend on the grid size; one "
                                      f"{a.nx}x{a.nx} step would take ~{4 * a.nx * a.nx / value:.0f} s)"},
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": threads,
                             "kind": "reference",
                             "sample": f"{nx}x{nx} C5 sub-field, 1 FS + residual + restrict pair per step"},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------- GPU arm
def ours(a):
    import torch

    from paper_2206_13164_b200 import momg
    from paper_2206_13164_b200.synthetic import c5_field

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    err = momg._Err()
    momg.lib().momg_init(local, momg.C.byref(err))
    momg.lib().momg_set_stream(momg.C.c_void_p(stream.cuda_stream))

    nx, M = a.nx, a.M
    N = momg.count(M)
    g = momg.Grid2D.uniform(nx, nx)
    cgrid = momg.Grid2D(nx // 2, nx // 2, 1.0, 1.0, *_coarse_arrays(g))
    ctx = momg.cavity_context(M, a.order, knudsen=0.1, lid=0.0)
    c_host, p_host = c5_field(nx, nx, M, seed=a.seed + rank)
    f = momg.CellField.from_host(g, M, c_host, p_host)
    res = momg.CellField(g, M)
    coarse = momg.CellField(cgrid, M)
    before = momg.CellField(cgrid, M)
    after = momg.CellField(cgrid, M)
    crhs = momg.CellField(cgrid, M)
    dc, _ = c5_field(nx // 2, nx // 2, M, seed=a.seed + 99)
    dc[:, :10] = 0.0
    dc *= 1e-3
    delta = momg.CellField.from_host(cgrid, M, dc, np.zeros((cgrid.cells(), 4)))
    L = momg.lib()
    E = momg._Err
    C = momg.C

    def ck(rc, e):
        if rc:
            raise RuntimeError(f"momg rc {rc}: {e.msg.decode(errors='replace')}")

    def step(evs=None, fld=None):
        fld = fld or f
        e = E()
        if evs:
            evs[0].record(stream)
        c = ctx._c(M)
        if FUSED:
            # fast_sweep_step + residual as one launch (momg_fast_sweep_residual)
            momg.fast_sweep_residual(fld, ctx, res)
            if evs:
                evs[1].record(stream)
                evs[2].record(stream)
        else:
            momg.fast_sweep_step(fld, None, ctx)
            if evs:
                evs[1].record(stream)
            ck(L.momg_residual(C.byref(c), fld.handle, res.handle, C.byref(e)), e)
            if evs:
                evs[2].record(stream)
        ck(L.momg_restrict_solution(fld.handle, coarse.handle, C.byref(e)), e)
        ck(L.momg_field_copy(before.handle, coarse.handle, C.byref(e)), e)
        ck(L.momg_defect(res.handle, None, res.handle, C.byref(e)), e)
        ck(L.momg_restrict_residual(res.handle, coarse.handle, crhs.handle, C.byref(e)), e)
        ck(L.momg_field_copy(after.handle, coarse.handle, C.byref(e)), e)
        ck(L.momg_axpy(after.handle, delta.handle, C.byref(e)), e)
        ck(L.momg_fas_correct(fld.handle, before.handle, after.handle, C.byref(e)), e)
        if evs:
            evs[3].record(stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.steps)]
    launches0 = momg.launch_count()
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for s in range(a.steps):
            step(evs[s])
        t1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    launches = momg.launch_count() - launches0
    total_ms = t0.elapsed_time(t1)
    if dist:
        tt = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / a.steps
    sweep_ms = [e[0].elapsed_time(e[1]) for e in evs]
    resid_ms = [e[1].elapsed_time(e[2]) for e in evs]
    xfer_ms = [e[2].elapsed_time(e[3]) for e in evs]
    updates = 4.0 * nx * nx
    value = updates * world / (ms_step * 1e-3)

    # ---- end to end through the C ABI: host (pinned) -> device -> step -> host.
    # Streaming many solves: two device fields double-buffer the stream, the
    # upload of step i+1 and the download of step i run on the library's copy
    # streams under the compute of step i (momg_field_{upload,download}_overlapped).
    # Every step still uploads its whole input and downloads its whole result
    # inside the timed region.
    e2e = None
    if not a.no_e2e:
        pin = lambda *shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()  # noqa: E731
        hc, hp = pin(nx * nx, N), pin(nx * nx, 4)
        hc[:] = c_host
        hp[:] = p_host
        oc = [pin(nx * nx, N) for _ in range(2)]
        op = [pin(nx * nx, 4) for _ in range(2)]
        f2 = momg.CellField(g, M)
        flds = [f, f2]
        ec, ep = momg._dp(hc), momg._dp(hp)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e = E()
        e0.record(stream)
        ck(L.momg_field_upload_overlapped(flds[0].handle, ec, ep, C.byref(e)), e)
        for s_ in range(a.steps):
            cur, nxt = flds[s_ % 2], flds[(s_ + 1) % 2]
            # the upload of step i+1 is enqueued BEFORE step i: it runs on the
            # H2D copy stream under step i's compute (the library stream waits
            # for it only when step i+1 first touches the field)
            if s_ + 1 < a.steps:
                ck(L.momg_field_upload_overlapped(nxt.handle, ec, ep, C.byref(e)), e)
            step(fld=cur)
            ck(L.momg_field_download_overlapped(cur.handle, momg._dp(oc[s_ % 2]), momg._dp(op[s_ % 2]),
                                                C.byref(e)), e)
        ck(L.momg_copy_barrier(C.byref(e)), e)
        e1.record(stream)
        torch.cuda.synchronize()
        ck(L.momg_synchronize(C.byref(e)), e)
        e2e_ms = e0.elapsed_time(e1) / a.steps
        if dist:
            tt = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        assert np.isfinite(oc[(a.steps - 1) % 2][:, 0]).all()
        nbytes = hc.nbytes + hp.nbytes
        e2e = {"value": updates * world / (e2e_ms * 1e-3), "unit": "cell-updates/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": oc[0].nbytes + op[0].nbytes,
               "ms_per_step": e2e_ms,
               "mode": "double-buffered stream of solves: the H2D of step i+1 is enqueued before step i and "
                       "the D2H of step i after it, on the library's copy streams (pinned host buffers, C ABI "
                       "*_overlapped calls with a deferred per-field wait); ms_per_step vs the device-timed "
                       "ms_per_step shows what the copies cost (the first upload and the last download are "
                       "not hidden: pipeline fill and drain, amortised over the K timed steps)"}

    # ---- NMG time-to-1e-8 on C2 (128^2, M=5, order 2, 4 levels)
    nmg = None
    if not a.no_nmg and rank == 0:
        nmg = run_nmg_c2(momg)
        nmg["other_configs"] = run_nmg_configs(momg)

    # ---- roofline of the dominant kernel (persistent FS sweep)
    peak, peak_src = fp64_peak()
    sweep_med = statistics.median(sweep_ms)
    # fused launch: the kernel's algorithmic work is the FS iteration plus the residual
    kflops = FLOPS_PER_UPDATE_C5 * updates + (FLOPS_RESIDUAL_C5 * nx * nx if FUSED else 0.0)
    achieved = kflops / (sweep_med * 1e-3) / 1e12
    roof = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": band_traffic(nx), "kernel": "rb::k8_band<5>" if a.order == 1 else "sp::k6_band<5>",
            "flops_per_update": FLOPS_PER_UPDATE_C5,
            "flops_per_launch": kflops, "fused_residual": FUSED, "peak_source": peak_src,
            "kernel_ms": sweep_med,
            "note": ("FP64 CUDA cores (no tensor-core path); hbm bytes/update >= 960, AI ~17 flop/B. "
                     "Exact Gauss-Seidel order: the sweep DAG has ~2.5 (nx+ny) dependent levels per "
                     "FS iteration, so the kernel is bound by the latency of one 32-cell diagonal "
                     "step (kernel_ms / levels), not by FP64 or HBM throughput (DESIGN.md sec. 5)")}

    # the reference's threads > 1 semantics (blocked-parallel sweep, 16
    # workers, the reference arm's configuration) realised deterministically
    # on the device: informational, the headline is the exact order above
    blocked = None
    if rank == 0 and a.order == 1:
        ctx16 = momg.cavity_context(M, a.order, knudsen=0.1, lid=0.0)
        ctx16.threads = 16
        fb = momg.CellField.from_host(g, M, c_host, p_host)
        momg.fast_sweep_residual(fb, ctx16, res)
        eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eb0.record(stream)
        for _ in range(3):
            momg.fast_sweep_residual(fb, ctx16, res)
        eb1.record(stream)
        torch.cuda.synchronize()
        bms = eb0.elapsed_time(eb1) / 3
        blocked = {"threads": 16, "fs_residual_ms": bms, "cell_updates_per_s": updates / (bms * 1e-3),
                   "note": "SolveContext.threads = 16: the reference's blocked-parallel FS (single_level.cpp:"
                           "130-161; its --impl reference arm) realised deterministically (tests/"
                           "test_gpu_blocked.py); not the exact order the headline value measures"}
        del fb

    steps_info = None
    if not a.no_trace and rank == 0 and a.order == 1:
        steps_info = band_step_stats(momg, f, ctx, nx, FLOPS_PER_UPDATE_C5, peak)
    if steps_info:
        roof["band_steps"] = steps_info

    cpu = None
    if not a.no_cpu and rank == 0 and world == 1:
        from oracle.api import REF_LIB
        kind = "reference" if os.path.exists(REF_LIB) else "port"
        r, dt = cpu_sample_rate(kind, a.cpu_sample, M, a.order, 1, a.seed, steps=2)
        what = ("the reference itself (oracle/_ref: /root/reference/proj/src compiled -O2 against the "
                "Eigen/doctest shims), threads=1 = its exact serial Gauss-Seidel FS" if kind == "reference"
                else "C restatement oracle/momg_oracle.c, 1 thread")
        cpu = {"value": r, "unit": "cell-updates/s", "cores": 1, "kind": kind,
               "sample": f"{a.cpu_sample}x{a.cpu_sample} C5 sub-field, 2 steps of FS + residual + restrict pair "
                         f"({dt:.1f} s; {what})"}

    if rank == 0:
        line = {"metric": "smoother cell-updates/s (FP64)", "value": value, "unit": "cell-updates/s",
                "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": c5_config(nx, M, a.order),
                "impl_detail": {"parallelism": f"replicas x{world}",
                                "sweep": "persistent dataflow, exact lexicographic GS order"},
                "breakdown_ms": ({"fast_sweep+residual (one launch)": sweep_med} if FUSED else
                                 {"fast_sweep": sweep_med, "residual": statistics.median(resid_ms)})
                | {"restrict_prolong": statistics.median(xfer_ms)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "nmg": nmg, "blocked_fs": blocked}
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def band_step_stats(momg, f, ctx, nx, flops_per_update, peak_tflops):
    """One extra FS iteration (outside every timed region) with the band
    kernel's %globaltimer trace on: per-diagonal step latency, tasks in flight,
    SM-busy fraction and the DAG-bound ceiling of the exact-order sweep."""
    import ctypes as C
    L = momg.lib()
    nb = (nx + 31) // 32
    cap = 4 * nb
    L.momg_debug_trace(C.c_longlong(4 * cap))
    momg.fast_sweep_step(f, None, ctx)
    buf = np.zeros((cap, 32), dtype=np.uint64)
    got = L.momg_debug_trace_read(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_longlong(4 * cap)) // 4
    L.momg_debug_trace(C.c_longlong(0))
    if got <= 0:
        return None
    t = buf[:got].astype(np.float64)
    steps = (buf[:got, 2] & 0xfffff).astype(np.float64)
    busy_ns = float(np.sum(t[:, 1] - t[:, 0]))
    span_ns = float(t[:, 1].max() - t[:, 0].min())
    step_us = busy_ns / float(np.sum(steps)) / 1e3
    in_flight = busy_ns / span_ns
    levels = span_ns / 1e3 / step_us  # dependent diagonal steps on the critical path
    # compute floor of one 32-cell step on one SM at its share of the FP64 peak
    floor_step_us = 32 * flops_per_update / (peak_tflops * 1e12 / 148) * 1e6
    ideal_ms = 4.0 * nx * nx * flops_per_update / (peak_tflops * 1e12) * 1e3
    return {"us_per_diagonal_step": step_us, "span_ms": span_ns / 1e6, "tasks": int(got),
            "tasks_in_flight_mean": in_flight, "sm_busy_frac": in_flight / 148.0,
            "dag_levels": levels, "compute_floor_step_us": floor_step_us,
            "dag_bound_ceiling_frac": ideal_ms / (levels * floor_step_us / 1e3),
            "note": "one FS iteration with the debug trace on (not timed): a 32-cell band step at the "
                    "per-SM FP64 floor still leaves the sweep DAG-latency bound at dag_bound_ceiling_frac"}


def _coarse_arrays(g):
    nx, ny = g.nx // 2, g.ny // 2
    dx = g.dx[0::2] + g.dx[1::2]
    dy = g.dy[0::2] + g.dy[1::2]
    xc = np.cumsum(dx) - 0.5 * dx
    yc = np.cumsum(dy) - 0.5 * dy
    return dx, dy, xc, yc


def run_nmg_c2(momg):
    """C2: 128x128 lid cavity, Kn 0.1, M = 5, second order, NMG over 4 levels,
    uniform Maxwellian start, until ||R||/||R0|| <= 1e-8 (multigrid.cpp:243-320)."""
    import torch
    g = momg.Grid2D.uniform(128, 128)
    ctx = momg.cavity_context(5, 2, knudsen=0.1, lid=0.1)
    f = momg.uniform_field(g, 5, 1.0, (0.0, 0.0, 0.0), 1.0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    try:
        rep = momg.solve_steady(f, ctx, momg.SolverOptions(momg.SolverKind.nmg, 1e-8, 0, 4))
        ok = True
    except momg.NonConvergence as e:
        rep, ok = e.report, False
    wall = time.perf_counter() - t
    # algorithmic FS flops of the solve: SURVEY.md §8(a) model, M=5 order 2,
    # x/y shifts only (the cavity keeps u_z = 0 exactly); finest level without
    # rhs, coarse levels with the FAS rhs
    n2 = 128 * 128
    per_cycle = {"128^2": (4 * 4 * n2, 15300.0), "64^2": (4 * 4 * n2 // 4, 16000.0),
                 "32^2": (4 * 4 * n2 // 16, 16000.0), "16^2": (4 * 4 * n2 // 64, 16000.0)}
    flops_cycle = sum(u * fl for u, fl in per_cycle.values())
    peak, _ = fp64_peak()
    achieved = flops_cycle * rep.iterations / wall / 1e12
    out = {"config": "C2 128x128 M=5 order 2 BGK Kn 0.1 NMG levels 4 (V(2,2), s3=4)",
           "seconds": wall, "converged": ok, "iterations": rep.iterations,
           "final_ratio": rep.final_ratio, "work_cell_updates": rep.work,
           "ms_per_vcycle": 1e3 * wall / max(1, rep.iterations),
           "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak, "flops_per_vcycle_fs": flops_cycle,
                        "note": "FS flops only (residual / transfer work excluded); the V-cycle is bound by "
                                "the DAG depth of the exact-order sweeps x the per-diagonal step latency"}}
    out["cpu"] = nmg_cpu_c2(rep.iterations)
    # the reference's threads > 1 semantics on the device (blocked-parallel
    # sweeps, 8 workers: one 16-column band per block on the 128^2 level;
    # coarser levels' blocks are not band-aligned and run the exact order)
    ctx8 = momg.cavity_context(5, 2, knudsen=0.1, lid=0.1)
    ctx8.threads = 8
    f8 = momg.uniform_field(g, 5, 1.0, (0.0, 0.0, 0.0), 1.0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    try:
        rep8 = momg.solve_steady(f8, ctx8, momg.SolverOptions(momg.SolverKind.nmg, 1e-8, 0, 4))
        ok8 = True
    except momg.NonConvergence as e:
        rep8, ok8 = e.report, False
    out["blocked_threads8"] = {"seconds": time.perf_counter() - t, "converged": ok8, "iterations": rep8.iterations,
                               "note": "SolveContext.threads = 8 (the reference's blocked-parallel FS realised "
                                       "deterministically, DESIGN.md sec. 5); not the exact order above"}
    return out


def run_nmg_configs(momg, cycles=3):
    """V-cycle time of the other BASELINE NMG configs on the device (C3: 256^2,
    M = 8, Shakhov, Kn 0.01, 5 levels; C4: 512^2, M = 6, heated bottom wall, 6
    levels): `cycles` NMG cycles from the uniform Maxwellian start, timed
    after one warm-up cycle.  Their full solves and parity against the oracle
    are in tests/test_gpu_configs.py and profiles/r2_configs_device.json; here
    only the per-cycle time and its FP64 fraction (FS flops, SURVEY.md §8(a):
    28,191 flop per cell update at M = 6 order 2, 70,484 at M = 8)."""
    import torch
    peak, _ = fp64_peak()
    out = {}
    for name, (n, M, model, kn, pr, lid, bt, levels, fl) in {
            "C3": (256, 8, momg.CollisionKind.shakhov, 0.01, 2.0 / 3.0, 0.1, 1.0, 5, 70484.0),
            "C4": (512, 6, momg.CollisionKind.bgk, 0.1, 1.0, 0.0, 2.0, 6, 28191.0)}.items():
        ctx = momg.cavity_context(M, 2, model, knudsen=kn, lid=lid, prandtl=pr, bottom_theta=bt)
        f = momg.uniform_field(momg.Grid2D.uniform(n, n), M, 1.0, (0.0, 0.0, 0.0), 1.0)
        momg.nmg_cycle(f, ctx, levels)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(cycles):
            momg.nmg_cycle(f, ctx, levels)
        momg.synchronize()
        ms = 1e3 * (time.perf_counter() - t) / cycles
        updates = sum(16 * (n >> l) ** 2 for l in range(levels))  # 4 FS iterations x 4 sweeps per level
        achieved = updates * fl / (ms * 1e-3) / 1e12
        out[name] = {"config": f"{n}x{n} M={M} order 2 NMG levels {levels}", "ms_per_vcycle": ms,
                     "cell_updates_per_vcycle": updates,
                     "kernel": "rb::k9_band<6,16> (register-resident, 16-column bands)" if M == 6 else "k_sweep_persistent (warp per cell)",
                     "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                                  "frac": achieved / peak}}
        del f
    return out


def nmg_cpu_c2(iterations, cycles=1):
    """The reference's own solve on C2, same run, same host: `cycles` NMG
    V-cycles (+ mass correction + residual + norm, as solve_steady iterates)
    of oracle/_ref at threads=1, timed, then extrapolated to the GPU's
    iteration count (a full 99-cycle CPU solve takes ~18 min)."""
    from oracle.api import REF_LIB, BGK, Ctx, Grid, Oracle, uniform_field
    kind = "reference" if os.path.exists(REF_LIB) else "port"
    o = Oracle(kind)
    g = Grid.uniform(128, 128)
    cb = o.max_hermite_root(6)
    ctx = Ctx(M=5, space_order=2, c_bound=cb, cfl=0.9, cfl_c_bound=cb, collision=BGK, knudsen=0.1,
              wall_speed=(0, 0, 0, 0.1))
    c, p = uniform_field(g, 5)
    t = time.perf_counter()
    _, _, rep = o.solve_steady(ctx, g, c, p, solver=2, tol=1e-8, levels=4, max_iterations=cycles)
    dt = time.perf_counter() - t
    return {"kind": kind, "cores": 1, "measured_cycles": cycles, "measured_s": dt,
            "extrapolated_s": dt / cycles * iterations,
            "note": f"{cycles} V-cycle(s) of the reference's solve_steady (threads=1, exact FS) timed on this "
                    f"host, extrapolated to {iterations} iterations (labelled extrapolated)"}


def strips_arm(a):
    """C5 strong-scaling step on N GPUs (torchrun, one process per GPU): the
    2048^2 field split into N column strips (one per rank, peer-mapped over
    NVLink), the fused FS iteration + residual as one band launch per rank that
    pipelines the wavefront across strips (momg_strips_fast_sweep_residual),
    then the strip-local restrict/prolong pair.  With world 1 and --strips K it
    runs the K-strip partition in one process (all ranks in one kernel)."""
    import torch

    from paper_2206_13164_b200 import momg
    from paper_2206_13164_b200.strips import StripComm, StripLevel
    from paper_2206_13164_b200.synthetic import c5_field

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    err = momg._Err()
    momg.lib().momg_init(local, momg.C.byref(err))
    momg.lib().momg_set_stream(momg.C.c_void_p(stream.cuda_stream))
    comm = StripComm(dist, device=torch.device("cuda", local))
    nx, M = a.nx, a.M
    N = momg.count(M)
    g = momg.Grid2D.uniform(nx, nx)
    ctx = momg.cavity_context(M, a.order, knudsen=0.1, lid=0.0)
    c_host, p_host = c5_field(nx, nx, M, seed=a.seed)  # one global field, every rank uploads its columns
    level = StripLevel(momg, g, M, comm, emulate_ranks=a.strips or None)
    level.upload(c_host, p_host)
    per = {}
    for r in level.owned:
        f = level.field(r)
        cg = momg.Grid2D(f.grid.nx // 2, f.grid.ny // 2, f.grid.Lx, f.grid.Ly, *_coarse_arrays(f.grid))
        dc, _ = c5_field(cg.nx, cg.ny, M, seed=a.seed + 99 + r)
        dc[:, :10] = 0.0
        dc *= 1e-3
        per[r] = dict(coarse=momg.CellField(cg, M), before=momg.CellField(cg, M), after=momg.CellField(cg, M),
                      crhs=momg.CellField(cg, M),
                      delta=momg.CellField.from_host(cg, M, dc, np.zeros((cg.cells(), 4))))
    L, E, C = momg.lib(), momg._Err, momg.C

    def ck(rc, e):
        if rc:
            raise RuntimeError(f"momg rc {rc}: {e.msg.decode(errors='replace')}")

    def step(evs=None):
        e = E()
        if evs:
            evs[0].record(stream)
        level.sweep_residual(ctx)
        if evs:
            evs[1].record(stream)
        for r, b in per.items():
            f, res = level.field(r), level.residual_field(r)
            ck(L.momg_restrict_solution(f.handle, b["coarse"].handle, C.byref(e)), e)
            ck(L.momg_field_copy(b["before"].handle, b["coarse"].handle, C.byref(e)), e)
            ck(L.momg_defect(res.handle, None, res.handle, C.byref(e)), e)
            ck(L.momg_restrict_residual(res.handle, b["coarse"].handle, b["crhs"].handle, C.byref(e)), e)
            ck(L.momg_field_copy(b["after"].handle, b["coarse"].handle, C.byref(e)), e)
            ck(L.momg_axpy(b["after"].handle, b["delta"].handle, C.byref(e)), e)
            ck(L.momg_fas_correct(f.handle, b["before"].handle, b["after"].handle, C.byref(e)), e)
        if evs:
            evs[2].record(stream)

    for _ in range(a.warmup):
        step()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.steps)]
    launches0 = momg.launch_count()
    with Clocks(local) as clk:
        comm.fence(torch.cuda.synchronize)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for s_ in range(a.steps):
            step(evs[s_])
        t1.record(stream)
        comm.fence(torch.cuda.synchronize)
    launches = momg.launch_count() - launches0
    ms_step = comm.allreduce_max(t0.elapsed_time(t1)) / a.steps
    sweep_med = statistics.median([e[0].elapsed_time(e[1]) for e in evs])
    xfer_med = statistics.median([e[1].elapsed_time(e[2]) for e in evs])
    updates = 4.0 * nx * nx
    value = updates / (ms_step * 1e-3)
    # end to end: every rank uploads its strip's columns from pinned host
    # memory, runs the step and downloads its strip, all inside the timed region
    e2e = None
    if not a.no_e2e:
        pin = lambda *shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()  # noqa: E731
        host = {}
        for r in level.owned:
            i0, i1 = level.bounds[r], level.bounds[r + 1]
            hc = pin(nx * (i1 - i0), N)
            hp = pin(nx * (i1 - i0), 4)
            hc[:] = c_host.reshape(nx, nx, N)[:, i0:i1].reshape(-1, N)
            hp[:] = p_host.reshape(nx, nx, 4)[:, i0:i1].reshape(-1, 4)
            host[r] = (hc, hp, pin(nx * (i1 - i0), N), pin(nx * (i1 - i0), 4))
        comm.fence(torch.cuda.synchronize)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e = E()
        e0.record(stream)
        for _ in range(a.steps):
            for r, (hc, hp, oc, op) in host.items():
                ck(L.momg_field_upload_overlapped(level.field(r).handle, momg._dp(hc), momg._dp(hp), C.byref(e)), e)
            step()
            for r, (hc, hp, oc, op) in host.items():
                ck(L.momg_field_download_overlapped(level.field(r).handle, momg._dp(oc), momg._dp(op),
                                                    C.byref(e)), e)
        ck(L.momg_copy_barrier(C.byref(e)), e)
        e1.record(stream)
        comm.fence(torch.cuda.synchronize)
        ck(L.momg_synchronize(C.byref(e)), e)
        e2e_ms = comm.allreduce_max(e0.elapsed_time(e1) / a.steps)
        hb = sum(h[0].nbytes + h[1].nbytes for h in host.values())
        db = sum(h[2].nbytes + h[3].nbytes for h in host.values())
        e2e = {"value": updates / (e2e_ms * 1e-3), "unit": "cell-updates/s",
               "h2d_bytes_per_step": int(comm.allreduce_sum(hb)), "d2h_bytes_per_step": int(comm.allreduce_sum(db)),
               "ms_per_step": e2e_ms,
               "mode": "each rank uploads its strip (pinned host), runs the step, downloads its strip"}
    # NMG over strips: C2 (128^2, M=5, second order, NMG 4 levels) to 1e-8 with
    # the finest level in 2 strips (strips of whole 64-column pairs of bands)
    # and the coarse levels agglomerated on every rank (strips.StripSolver)
    nmg = None
    if not a.no_nmg and len(level.bounds) - 1 == 2:
        from paper_2206_13164_b200.strips import StripSolver
        g2 = momg.Grid2D.uniform(128, 128)
        ctx2 = momg.cavity_context(5, 2, knudsen=0.1, lid=0.1)
        solver = StripSolver(momg, g2, 5, comm, 4, emulate_ranks=2)
        cc = np.zeros((128 * 128, momg.count(5)))
        cc[:, 0] = 1.0
        pp = np.zeros((128 * 128, 4))
        pp[:, 3] = 1.0
        solver.fine.upload(cc, pp)
        comm.fence(torch.cuda.synchronize)
        t = time.perf_counter()
        conv, iters, hist = solver.solve(ctx2, 1e-8)
        comm.fence(torch.cuda.synchronize)
        wall = comm.allreduce_max(time.perf_counter() - t)
        nmg = {"config": "C2 128x128 M=5 order 2 BGK Kn 0.1 NMG levels 4, finest level in 2 column strips, "
                         "coarse levels agglomerated on every rank", "seconds": wall, "converged": conv,
               "iterations": iters, "final_ratio": hist[-1] if hist else None,
               "ms_per_vcycle": 1e3 * wall / max(1, iters)}
    if rank == 0:
        nstrips = len(level.bounds) - 1
        line = {"metric": "smoother cell-updates/s (FP64)", "value": value, "unit": "cell-updates/s",
                "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": c5_config(nx, M, a.order),
                "impl_detail": {"parallelism": f"column strips x{nstrips} "
                                + ("(one per rank, peer memory over NVLink)" if world > 1 else "(one process)"),
                                "strip_bounds": level.bounds,
                                "sweep": "band dataflow across strips, exact lexicographic GS order"},
                "breakdown_ms": {"fast_sweep+residual (strips, fenced)": sweep_med, "restrict_prolong": xfer_med},
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "nmg": nmg}
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1 or a.strips:
        strips_arm(a)
    else:
        ours(a)


if __name__ == "__main__":
    main()
