#!/bin/bash
# Full ncu capture of one kernel (regex) during the C2 bench: bash tools/gpu_prof_kernel.sh <regex> <name>
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s 1 -c 1 -o gpurun_out/prof_$2 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_$2.log 2>&1
tail -3 gpurun_out/ncu_$2.log
