#!/bin/bash
mkdir -p gpurun_out
for v in 1 2 4; do
  touch paper_1506_02226_b200/csrc/ds_tile.cu
  make -s -C paper_1506_02226_b200/csrc EXTRA="-DDS_BATCH_MIN=$v" > /dev/null 2>&1
  echo "batch_min=$v" >> gpurun_out/bsweep.log
  python tools/tile_bench.py --configs C1,C2,C3,C5 --dense "" --reps 5 >> gpurun_out/bsweep.log 2>&1
done
