#!/bin/bash
# ncu full captures of the stage-1 kernel: C2 culled + C2 dense, C4 culled.
#   bash tools/prof_tile.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
K='regex:eps_unit_kernel'
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -c 2 \
  -o gpurun_out/tile_c2_${TAG} python tools/prof_unit.py > gpurun_out/prof_c2_${TAG}.log 2>&1
DS_CONFIG=C4 DS_DENSE=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -c 1 \
  -o gpurun_out/tile_c4_${TAG} python tools/prof_unit.py > gpurun_out/prof_c4_${TAG}.log 2>&1
echo done
