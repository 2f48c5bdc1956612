"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_summary.py LAUNCHES.csv "header comment" > profiles/...txt"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = collections.OrderedDict()
for r in rows:
    if not r:
        continue
    if "Kernel Name" in r:
        h = r
        continue
    if h is None or len(r) < len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values()) or 1.0
print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
print("# gpu__time_duration.sum, --clock-control none; cold-cache serialised times: compare SHARES")
print(f"{'kernel':44s} launches   total_ms per_launch_ms   share")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:44]:44s} {n:8d} {t:10.3f} {t / n:13.3f} {t / tot * 100:6.1f}%")
