#!/bin/bash
mkdir -p gpurun_out
for v in "8 3" "4 3" "16 3" "8 2" "16 2"; do
  set -- $v
  touch paper_1506_02226_b200/csrc/ds_tile.cu
  make -s -C paper_1506_02226_b200/csrc EXTRA="-DDS_UNROLL_WIDE=$1 -DDS_MINB16=$2" > /dev/null 2>&1
  echo "unroll=$1 minb=$2" >> gpurun_out/c4sweep.log
  python tools/tile_bench.py --configs C4 --dense "" --reps 3 >> gpurun_out/c4sweep.log 2>&1
done
