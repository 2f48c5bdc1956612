#!/bin/bash
# ncu evidence for one round (run under gpurun; one GPU).  Usage: tools/profile.sh TAG
set -e
TAG=${1:-r1}
mkdir -p gpurun_out
# 1) the bench's launch list (short run, no NMG/e2e/cpu legs), plain run first
python bench.py --steps 2 --warmup 1 --no-nmg --no-e2e --no-cpu --nx ${NX:-1024} > gpurun_out/plain_bench_${TAG}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-nmg --no-e2e --no-cpu --nx ${NX:-1024} > gpurun_out/ncu_bench_${TAG}.log 2>&1
# 2) full capture of the top kernels on a small fixed case
python tools/prof_case.py > gpurun_out/plain_case_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_residual|k_sweep_persistent" -s 1 -c 2 \
    -o gpurun_out/prof_${TAG} -f python tools/prof_case.py > gpurun_out/ncu_case_${TAG}.log 2>&1
echo profile done
