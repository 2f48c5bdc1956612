#!/bin/bash
# Experiment build: recompile only runtime.cu and kernels_m${M:-5}.cu (with EXTRA
# flags) into paper_2206_13164_b200/_lib_b, reusing the other orders' objects
# from _lib/obj.  Load it with MOMG_GPU_LIB=$PWD/paper_2206_13164_b200/_lib_b/libmomg_gpu.so
set -e
cd "$(dirname "$0")/../paper_2206_13164_b200/csrc"
M=${M:-5}
mkdir -p ../_lib_b/obj
for o in ../_lib/obj/*.o; do
  b=$(basename $o)
  case $b in runtime.o|kernels_m$M.o|band2_m$M.o) ;; *) cp -p $o ../_lib_b/obj/$b ;; esac
done
make -s -j3 OUT=../_lib_b EXTRA="$EXTRA" ../_lib_b/obj/runtime.o ../_lib_b/obj/kernels_m$M.o ../_lib_b/obj/band2_m$M.o
touch ../_lib_b/obj/*.o
make -s OUT=../_lib_b EXTRA="$EXTRA" ../_lib_b/libmomg_gpu.so
grep -A3 "k5_band" ../_lib_b/obj/kernels_m$M.ptxas.log | grep -E "registers|spill" | head -4
