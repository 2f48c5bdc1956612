#!/bin/bash
# A/B of library variants under paper_2206_13164_b200/_lib/var*/ against the default build:
# bench FS + residual at 2048^2, band trace at 2048^2, and the k8 parity tests
for L in "" $(ls -d $PWD/paper_2206_13164_b200/_lib/var*/libmomg_gpu.so 2>/dev/null); do
  echo "== lib ${L:-default}"
  MOMG_GPU_LIB=$L timeout 300 python bench.py --no-cpu --no-e2e --no-nmg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['breakdown_ms'])"
  MOMG_GPU_LIB=$L timeout 300 python tools/trace_band.py ${N:-2048} 5 2>&1 | sed -n 1,9p
  if [ -n "$L" ]; then MOMG_GPU_LIB=$L timeout 600 python -m pytest tests/test_gpu_rb.py -x -q -m gpu 2>&1 | tail -2; fi
done
