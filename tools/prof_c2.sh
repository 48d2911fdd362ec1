#!/bin/bash
# ncu full capture of the culled C2 stage-1 kernel (second call) -> gpurun_out/tile_c2_$1.ncu-rep
mkdir -p gpurun_out
DS_DENSE=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:eps_unit_kernel' -s 1 -c 1 -o gpurun_out/tile_c2_$1 python tools/prof_unit.py > gpurun_out/prof_c2_$1.log 2>&1
