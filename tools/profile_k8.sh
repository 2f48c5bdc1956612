#!/bin/bash
# Round-2 ncu evidence for the register-resident band kernel rb::k8_band (run
# under gpurun; one GPU).  Every ncu command runs only after the same command
# exited 0 without ncu.  Outputs under gpurun_out/ (copied to profiles/ by hand).
set -e
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-nmg --no-e2e --no-cpu --no-trace"
$B > gpurun_out/plain_bench_k8.log 2>&1
# 1) launch list of the bench step (C5 2048^2)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_k8_launches.csv \
    $B > gpurun_out/ncu_bench_k8.log 2>&1
python tools/launch_summary.py gpurun_out/r2_k8_launches.csv \
  "# ncu launch list, round 2 final ($B; C5 2048^2; k8_band = fused FS iteration + residual (register-resident band kernel), xf_* = transfer operators)" \
  > gpurun_out/r2_k8_launches_summary.txt
# 2) DRAM traffic per launch of the band sweep
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k8_band" -c 2 --csv --log-file gpurun_out/r2_k8_traffic.csv $B > gpurun_out/ncu_traffic_k8.log 2>&1
# 3) full capture of one 32-column band (every warp on the step loop)
python tools/prof_band.py > gpurun_out/plain_band_k8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k8_band" -c 1 \
    -o /tmp/band_k8 -f python tools/prof_band.py > gpurun_out/ncu_band_k8.log 2>&1
python tools/ncu_summary.py /tmp/band_k8.ncu-rep k8_band 40 > gpurun_out/r2_ncu_k8_summary.txt 2>&1
python tools/ncu_lines.py /tmp/band_k8.ncu-rep 70 > gpurun_out/r2_ncu_k8_lines.txt 2>&1
# 3b) the same for the second-order kernel (k9_band), and the launch list of C2 NMG V-cycles
python tools/prof_band.py --order 2 > gpurun_out/plain_band_k9.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k9_band" -c 1 \
    -o /tmp/band_k9 -f python tools/prof_band.py --order 2 > gpurun_out/ncu_band_k9.log 2>&1
python tools/ncu_summary.py /tmp/band_k9.ncu-rep k9_band 40 > gpurun_out/r2_ncu_k9_summary.txt 2>&1
python tools/ncu_lines.py /tmp/band_k9.ncu-rep 50 > gpurun_out/r2_ncu_k9_lines.txt 2>&1
python tools/prof_nmg.py > gpurun_out/plain_nmg_k9.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_k9_nmg_launches.csv \
    python tools/prof_nmg.py > gpurun_out/ncu_nmg_k9.log 2>&1
python tools/launch_summary.py gpurun_out/r2_k9_nmg_launches.csv \
  "# ncu launch list, C2 NMG V-cycles (tools/prof_nmg.py; k9_band = second-order / rhs register-resident band sweep)" \
  > gpurun_out/r2_k9_nmg_launches_summary.txt
python tools/trace_band.py 128 5 2 > gpurun_out/r2_k9_trace_128.txt 2>&1
# 3c) M = 6 (k9_band<6,16>, BASELINE C4's order): one 16-column band, and the step trace at 512^2
python tools/prof_band.py --M 6 --order 2 --nx 16 --ny 512 > gpurun_out/plain_band_k9m6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k9_band" -c 1 \
    -o /tmp/band_k9m6 -f python tools/prof_band.py --M 6 --order 2 --nx 16 --ny 512 > gpurun_out/ncu_band_k9m6.log 2>&1
python tools/ncu_summary.py /tmp/band_k9m6.ncu-rep k9_band 40 > gpurun_out/r2_ncu_k9m6_summary.txt 2>&1
python tools/ncu_lines.py /tmp/band_k9m6.ncu-rep 50 > gpurun_out/r2_ncu_k9m6_lines.txt 2>&1
python tools/trace_band.py 512 6 2 > gpurun_out/r2_k9m6_trace_512.txt 2>&1
# 4) band step trace at 2048^2 (per-phase %globaltimer stamps, not timed)
python tools/trace_band.py 2048 > gpurun_out/r2_k8_trace_2048.txt 2>&1
echo profile done
