"""Per-item latency breakdown of the split persistent sweep (debug trace)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_13164_b200 import momg  # noqa: E402
from paper_2206_13164_b200.synthetic import c5_field  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
M = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = momg.Grid2D.uniform(n, n)
ctx = momg.cavity_context(M, 1, knudsen=0.1, lid=0.0)
c, p = c5_field(n, n, M, seed=1)
f = momg.CellField.from_host(g, M, c, p)
momg.fast_sweep_step(f, None, ctx)
L = momg.lib()
cap = 200000
L.momg_debug_trace(C.c_longlong(cap))
momg.fast_sweep_step(f, None, ctx)
buf = np.zeros((cap, 8), dtype=np.uint64)
got = L.momg_debug_trace_read(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_longlong(cap))
t = buf[:got].astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
wait = t[:, 1] - t[:, 0]
face = t[:, 2] - t[:, 1]
upd = t[:, 3] - t[:, 2]
print(f"items {len(t)}  span {(t[:, 3].max() - t0) / 1e3:.1f} us")
ph0 = t[:, 4] - t[:, 1]; ph12 = t[:, 5] - t[:, 4]; ph3 = t[:, 6] - t[:, 5]; ph4 = t[:, 2] - t[:, 6]
for name, v in (("wait", wait), ("faces", face), ("f.load", ph0), ("f.proj", ph12), ("f.flux", ph3), ("f.back", ph4), ("update", upd)):
    print(f"{name:7s} median {np.median(v) / 1e3:8.2f} us  p10 {np.percentile(v, 10) / 1e3:8.2f}  p90 {np.percentile(v, 90) / 1e3:8.2f}")
# critical path estimate: end-to-start gap between consecutive diagonals
order = np.argsort(t[:, 1])
sys.exit(0)
print("first items (us from start): ready, faces_done, update_done")
for k in order[:12]:
    print(f"  {(t[k, 1] - t0) / 1e3:9.2f} {(t[k, 2] - t0) / 1e3:9.2f} {(t[k, 3] - t0) / 1e3:9.2f}")
