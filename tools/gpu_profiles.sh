#!/bin/bash
# Round profiling evidence: C2 launch list of the bench command + full captures of the
# top kernels (C2) and of the 16-D tile kernel (C4). Outputs land in gpurun_out/.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:eps_tile_kernelILi2ELi1ELb1E -s 1 -c 1 -o gpurun_out/prof_tile_c2 $B > gpurun_out/ncu_t.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:union_diag -s 1 -c 1 -o gpurun_out/prof_diag_c2 $B > gpurun_out/ncu_d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:union_pair -s 1 -c 1 -o gpurun_out/prof_pair_c2 $B > gpurun_out/ncu_p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:eps_tile_kernelILi16ELi1ELb1E -s 1 -c 1 -o gpurun_out/prof_tile_c4 python tools/run_configs.py --configs C4 --reps 1 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out
