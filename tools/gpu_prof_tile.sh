#!/bin/bash
# Profile the C2 eps-tile kernel (full set) and the union kernels; launch list.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:eps_tile_kernelILi2ELi1ELb1E -s 1 -c 1 -o gpurun_out/prof_tile python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_tile.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_chunks -s 2 -c 2 -o gpurun_out/prof_union python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_union.log 2>&1
