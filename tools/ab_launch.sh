#!/bin/bash
# Launch lists (ncu gpu__time_duration) of the C2 bench per variant: gpurun_out/ab_launch_<variant>.csv
L=paper_1506_02226_b200/libdensescan_b200.so
cp $L /tmp/ab_keep.so
for v in ${@:-$(ls variants/*.so)}; do
  cp $v $L
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ab_launch_$(basename $v .so).csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dense > /dev/null 2>&1
done
cp /tmp/ab_keep.so $L
