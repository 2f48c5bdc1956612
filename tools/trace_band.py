"""Per-task timeline of the band-persistent sweep (debug trace).

usage: python tools/trace_band.py [n] [M] [space order]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_13164_b200 import momg  # noqa: E402
from paper_2206_13164_b200.synthetic import c5_field  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
M = int(sys.argv[2]) if len(sys.argv) > 2 else 5
SO = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = momg.Grid2D.uniform(n, n)
ctx = momg.cavity_context(M, SO, knudsen=0.1, lid=0.0)
c, p = c5_field(n, n, M, seed=1)
f = momg.CellField.from_host(g, M, c, p)
momg.fast_sweep_step(f, None, ctx)
L = momg.lib()
bw = 16 if M == 6 else 32
nb = (n + bw - 1) // bw
cap = 4 * nb
L.momg_debug_trace(C.c_longlong(4 * cap))
momg.fast_sweep_step(f, None, ctx)
buf = np.zeros((cap, 32), dtype=np.uint64)
got = L.momg_debug_trace_read(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_longlong(4 * cap)) // 4
t = buf[:got].astype(np.float64)
steps = (buf[:got, 2] & 0xfffff).astype(np.float64)
sk = [(int(v >> 20) & 0xff, int(v >> 28)) for v in buf[:got, 2]]
t0 = t[:, 0].min()
S = np.sum(steps)
print(f"tasks {got}  span {(t[:, 1].max() - t0) / 1e3:.1f} us")
if np.sum(t[:, 10]) == 0:  # register-resident kernel (k8_band): its own stamp set
    m = lambda q: np.sum(t[:, q]) / S / 1e3
    print("k8_band per-step means, us from step start: write-back %.2f  faces(barrier A) %.2f  assembled(barrier B) %.2f"
          "  updated(warp 0) %.2f  end(barrier C) %.2f;  loop time/step %.2f"
          % (m(3), m(4), m(12), m(5), m(7), np.sum(t[:, 1] - t[:, 0]) / S / 1e3))
    print("step durations, share of steps in bins <9 <10 <11 <12.5 <15 <20 <40 >=40 us: all tasks",
          " ".join("%.3f" % (np.sum(t[:, 16 + w]) / S) for w in range(8)))
    rt = buf[:got, 6]
    print("steps with a dt/2 retry in the warp: %.4f   steps with an update > 3 us: %.4f"
          % (np.sum(rt & 0xffffffff) / S, np.sum(rt >> 32) / S))
    for r in (0, 1, 4, 8, 16, 32, 48, 63, 64, 80, 127, 128, 192, 255):
        if r < got:
            print("   task %3d (s %d k %2d):" % (r, sk[r][0], sk[r][1]),
                  " ".join("%.3f" % (t[r, 16 + w] / steps[r]) for w in range(8)))
    print("per-warp arrival at barrier C:", " ".join("%.2f" % m(24 + w) for w in range(8)))
    print("mid-role stamps, warps 2..7 (2-4 after the release, 5-6 after the cp.async issue, 7 after the halo poll):",
          " ".join("%.2f" % m(q) for q in (8, 9, 11, 14, 13)), "(warps 2, 3, 5, 6, 7)")
    ups = (t[:, 1] - t[:, 0]) / np.maximum(steps, 1) / 1e3
    for sw in range(4):
        rows_ = [r for r in range(got) if sk[r][0] == sw]
        if rows_:
            q = np.array_split(np.array(rows_), 4)
            print(f"sweep {sw}: us/step by band quarter:", " ".join("%.2f" % ups[x].mean() for x in q if len(x)),
                  "| start %.1f ms end %.1f ms" % ((t[rows_, 0].min() - t0) / 1e6, (t[rows_, 1].max() - t0) / 1e6))
    # per sweep and band quarter: the phases of the step and the SM clock the loop saw
    # (load dependence: the bands at both ends of the launch run with fewer active SMs)
    print("sweep.quarter: active-window ms | faces  B  update  tail  step (us) | SM MHz")
    for sw in range(4):
        rows_ = np.array([r for r in range(got) if sk[r][0] == sw])
        if not len(rows_):
            continue
        for qi, x in enumerate(np.array_split(rows_, 4)):
            if not len(x):
                continue
            Sx = np.sum(steps[x])
            mq = lambda q: np.sum(t[x, q]) / Sx / 1e3
            mhz = np.sum(t[x, 15]) / np.maximum(np.sum(t[x, 1] - t[x, 0]), 1) * 1e3
            print(f"  {sw}.{qi}: {(t[x, 0].min() - t0) / 1e6:6.1f}-{(t[x, 1].max() - t0) / 1e6:6.1f} | "
                  f"{mq(4):5.2f} {mq(12) - mq(4):5.2f} {mq(5) - mq(12):5.2f} {mq(7) - mq(5):5.2f} {mq(7):6.2f} | {mhz:5.0f}")
    print(" task  s   k  loop(us)  end(us)  steps  us/step")
    for r in (list(range(0, min(4, got))) + list(range(nb - 2, nb + 2)) + list(range(got - 3, got))):
        if 0 <= r < got:
            s_, k_ = sk[r]
            print(f"{r:5d} {s_:2d} {k_:3d} {(t[r,0]-t0)/1e3:8.1f} {(t[r,1]-t0)/1e3:8.1f} "
                  f"{int(steps[r]):6d} {(t[r,1]-t[r,0])/steps[r]/1e3:8.2f}")
    sys.exit(0)
print("per-step means, us from step start: copies %.2f  faces %.2f  update %.2f  prefetch %.2f  end %.2f;"
      "  loop time/step %.2f" % tuple([np.sum(t[:, q]) / S / 1e3 for q in (3, 4, 5, 6, 7)]
                                      + [np.sum(t[:, 1] - t[:, 0]) / S / 1e3]))
print("update detail, us from step start: scalars %.2f  assembled %.2f  normalized %.2f  written %.2f;"
      "  normalize iterations/step %.2f" % tuple([np.sum(t[:, q]) / S / 1e3 for q in (11, 12, 14, 15)]
                                                 + [np.sum(t[:, 13]) / S]))
print("face detail (group 0), us from step start: projected %.2f  flux %.2f" % tuple(
    np.sum(t[:, q]) / S / 1e3 for q in (8, 9)))
print("per-warp arrival at the end-of-step barrier, us from step start:",
      " ".join("%.2f" % (np.sum(t[:, 16 + w]) / S / 1e3) for w in range(16)))
print("effective SM clock over the step loops: %.0f MHz (median over tasks)" % np.median(
    t[:, 10] / np.maximum(t[:, 1] - t[:, 0], 1) * 1e3))
print(" task  s   k  loop(us)  end(us)  steps  us/step")
rows = [int(x) for x in os.environ.get('ROWS', '').split(',') if x] or (list(range(0, min(4, got))) + list(range(nb - 2, nb + 2)) + list(range(got - 3, got)))
for r in rows:
    if 0 <= r < got:
        s, k = sk[r]
        print(f"{r:5d} {s:2d} {k:3d} {(t[r,0]-t0)/1e3:8.1f} {(t[r,1]-t0)/1e3:8.1f} "
              f"{int(steps[r]):6d} {(t[r,1]-t[r,0])/steps[r]/1e3:8.2f}")
for r in [int(x) for x in os.environ.get('WROWS', '0,1,2,64').split(',') if x]:
    if 0 <= r < got:
        print(f"task {r}: per-warp arrival (us from step start):",
              " ".join("%.2f" % (t[r, 16 + w] / steps[r] / 1e3) for w in range(16)),
              "| faces %.2f update %.2f end %.2f" % tuple(t[r, q] / steps[r] / 1e3 for q in (4, 5, 7)))
