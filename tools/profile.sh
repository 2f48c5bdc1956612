#!/bin/bash
# ncu evidence for one round (run under gpurun; one GPU).  Usage: tools/profile.sh TAG
# Each ncu command runs only after the same command exited 0 without ncu.
set -e
TAG=${1:-r1}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-nmg --no-e2e --no-cpu"
# 1) the bench's launch list (C5 2048^2 step), plain run first
$B > gpurun_out/plain_bench_${TAG}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    $B > gpurun_out/ncu_bench_${TAG}.log 2>&1
# 1b) DRAM traffic of one bench-size band sweep launch (roofline "traffic")
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k5_band" -c 1 \
    --csv --log-file gpurun_out/traffic_${TAG}.csv $B > gpurun_out/ncu_traffic_${TAG}.log 2>&1
# 2) full capture of the band sweep on one 32-column band (every warp on the step loop)
python tools/prof_band.py > gpurun_out/plain_band_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k5_band" -c 1 \
    -o /tmp/band_${TAG} -f python tools/prof_band.py > gpurun_out/ncu_band_${TAG}.log 2>&1
# 3) full capture of the residual (512^2) and the band sweep at 256^2 (traffic per launch)
python tools/prof_case.py > gpurun_out/plain_case_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k3_residual|k5_band" -s 1 -c 2 \
    -o gpurun_out/case_${TAG} -f python tools/prof_case.py > gpurun_out/ncu_case_${TAG}.log 2>&1

python tools/ncu_summary.py /tmp/band_${TAG}.ncu-rep k5_band 40 > gpurun_out/band_${TAG}_summary.txt 2>&1
python tools/ncu_lines.py /tmp/band_${TAG}.ncu-rep 60 > gpurun_out/band_${TAG}_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/case_${TAG}.ncu-rep "" 30 > gpurun_out/case_${TAG}_summary.txt 2>&1
echo profile done
