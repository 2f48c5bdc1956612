#!/bin/bash
# Resident-CTA cap of the register-resident band sweeps (rb_grid_cap, MOMG_RB_GRID
# override): fused FS + residual time at several grid sizes and caps.
for NX in ${SIZES:-1024 2048 4096}; do
  for G in ${GRIDS:-0 148 96 64 48}; do
    echo "== nx $NX cap ${G} (0 = default rule 1.5 nk)"
    MOMG_RB_GRID=$G timeout 600 python bench.py --nx $NX --no-cpu --no-e2e --no-nmg --no-trace 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['breakdown_ms'])"
  done
done
