#!/bin/bash
# A/B the built libraries in variants/*.so on the GPU: for each, run_configs on the
# given configs (default C2,C3,C5), interleaved twice.
#   bash tools/ab.sh [configs] [variants...]
CFG=${1:-C2,C3,C5}; shift
VARS=${@:-$(ls variants/*.so)}
L=paper_1506_02226_b200/libdensescan_b200.so
cp $L /tmp/ab_keep.so
for r in 1 2; do
  for v in $VARS; do
    cp $v $L
    python tools/run_configs.py --configs $CFG --reps ${REPS:-7} 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print('$v', d['config'], 'total %.4f fused %.4f merge %.4f tile %.4f' % (d['total_ms'], d['fused_ms'], d['merge_ms'], d['tile_ms']))"
  done
done
cp /tmp/ab_keep.so $L
