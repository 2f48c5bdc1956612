"""Stall-reason breakdown per source file and top source lines of an ncu
report (needs -lineinfo and --import-source on).
usage: python tools/ncu_lines.py REPORT [n_lines] [exclude_regex]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 40
excl = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cur = None
lines = {}
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != '-':
        continue
    key = (cur, int(r[0]), r[1].strip()[:80])
    if excl and excl.search(key[2]):
        continue
    d = lines.setdefault(key, {})
    for i, name in enumerate(hdr):
        if i < len(r) and name.startswith('stall_') and 'Not Issued' not in name:
            try:
                d[name[6:]] = d.get(name[6:], 0) + int(r[i])
            except ValueError:
                pass
tot = sum(sum(d.values()) for d in lines.values()) or 1
files = {}
for (f, _, _), d in lines.items():
    fd = files.setdefault(f, {})
    for k, v in d.items():
        fd[k] = fd.get(k, 0) + v
print(f"stall samples {tot}")
for f, d in sorted(files.items(), key=lambda kv: -sum(kv[1].values())):
    t = sum(d.values())
    if t < tot * 0.01:
        continue
    top = ' '.join(f"{k}:{v / t * 100:.0f}%" for k, v in sorted(d.items(), key=lambda x: -x[1])[:6])
    print(f"{t / tot * 100:5.1f}% {f:22s} {top}")
print()
for key, d in sorted(lines.items(), key=lambda kv: -sum(kv[1].values()))[:nl]:
    t = sum(d.values())
    top = ' '.join(f"{k}:{v / t * 100:.0f}%" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3])
    print(f"{t / tot * 100:5.1f}% {key[0]}:{key[1]} {key[2][:60]:60s} {top}")
