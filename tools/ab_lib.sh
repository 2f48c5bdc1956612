#!/bin/bash
# A/B: default library vs paper_2206_13164_b200/_lib_b (bench FS at 2048^2 + band trace at 1024^2)
for L in "" "$PWD/paper_2206_13164_b200/_lib_b/libmomg_gpu.so"; do
  echo "== lib ${L:-default}"
  MOMG_GPU_LIB=$L timeout 300 python bench.py --no-cpu --no-e2e --no-nmg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['breakdown_ms'])"
  MOMG_GPU_LIB=$L timeout 200 python tools/trace_band.py ${N:-1024} 5 2>&1 | sed -n 2,4p
done
