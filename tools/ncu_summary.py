"""Summaries of an ncu report: key metrics per kernel and the top source lines
by executed instructions (needs -lineinfo + --import-source on)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
WANT = ('Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Compute (SM) Throughput', 'DRAM Throughput', 'Executed Ipc Active', 'Issue Slots Busy',
        'L2 Hit Rate', 'Eligible Warps Per Scheduler', 'Executed Instructions',
        'Warp Cycles Per Issued Instruction', 'Dynamic Shared Memory Per Block',
        'Block Limit Registers', 'Block Limit Shared Mem')
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
seen = set()
for r in rows[1:]:
    if r[mi] in WANT and (r[ki], r[mi]) not in seen:
        seen.add((r[ki], r[mi]))
        print(f"{r[ki][:42]:42s} | {r[mi]:36s} = {r[vi]} {r[ui]}")
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass']
                     + (['--kernel-name', f'regex:{kern}'] if kern else []), capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if r[0] == 'Function Name' or hdr is None or len(r) < 8 or r[2] != '-':
        continue
    try:
        n = int(r[7]); s = int(r[4])
    except ValueError:
        continue
    key = (cur, int(r[0]), r[1].strip()[:80])
    a = agg.setdefault(key, [0, 0]); a[0] += n; a[1] += s
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"\nsource lines ({kern or 'all kernels'}): total instructions {tot}, stall samples {tots}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{v[0]/tot*100:5.1f}% inst {v[1]/tots*100:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
