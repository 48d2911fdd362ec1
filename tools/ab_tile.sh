#!/bin/bash
# A/B the stage-1 kernel of variants/*.so: tools/tile_bench.py per variant, interleaved twice.
#   bash tools/ab_tile.sh [configs] [variants...]  -> stdout lines "variant {json}"
CFG=${1:-C2,C3,C5}; shift
VARS=${@:-$(ls variants/*.so)}
L=paper_1506_02226_b200/libdensescan_b200.so
cp $L /tmp/ab_keep.so
for r in 1 2; do
  for v in $VARS; do
    cp $v $L
    python tools/tile_bench.py --configs $CFG --dense "" --reps ${REPS:-7} 2>/dev/null | sed "s|^|$(basename $v .so) |"
  done
done
cp /tmp/ab_keep.so $L
