#!/bin/bash
# Round-2 ncu evidence (run under gpurun; one GPU).  Every ncu command runs
# only after the same command exited 0 without ncu.  Outputs: gpurun_out/*_r2*
set -e
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-nmg --no-e2e --no-cpu --no-trace"
$B > gpurun_out/plain_bench_r2.log 2>&1
# 1) launch list of the bench step (C5 2048^2)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
    $B > gpurun_out/ncu_bench_r2.log 2>&1
python tools/launch_summary.py gpurun_out/launches_r2.csv \
  "# ncu launch list, round 2 ($B; C5 2048^2; k5_band = fused FS iteration + residual, xf_* = register-resident transfer operators)" \
  > gpurun_out/r2_launches_summary.txt
# 2) DRAM traffic per launch of the band sweep and the transfer kernels
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k5_band|xf_" -c 4 --csv --log-file gpurun_out/traffic_r2.csv $B > gpurun_out/ncu_traffic_r2.log 2>&1
# 3) full capture of the transfer kernels at C5 size
ncu --set full --clock-control none --import-source on -k regex:"xf_" -c 3 \
    -o gpurun_out/xf_r2 -f $B > gpurun_out/ncu_xf_r2.log 2>&1
python tools/ncu_summary.py gpurun_out/xf_r2.ncu-rep "" 20 > gpurun_out/r2_ncu_xf_summary.txt 2>&1
# 4) full capture of the band sweep, one 32-column band (every warp on the step loop)
python tools/prof_band.py > gpurun_out/plain_band_r2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k5_band" -c 1 \
    -o /tmp/band_r2 -f python tools/prof_band.py > gpurun_out/ncu_band_r2.log 2>&1
python tools/ncu_summary.py /tmp/band_r2.ncu-rep k5_band 40 > gpurun_out/r2_ncu_band_summary.txt 2>&1
python tools/ncu_lines.py /tmp/band_r2.ncu-rep 60 > gpurun_out/r2_ncu_band_lines.txt 2>&1
# 5) band step trace at 2048^2 (per-phase %globaltimer stamps, not timed)
python tools/trace_band.py 2048 > gpurun_out/r2_band_trace_2048.txt 2>&1
echo profile done
