#!/bin/bash
# Full GPU iteration: smoke, GPU parity tests, bench (C2) + reference arm, all configs,
# ncu launch list of the bench command and full captures of the top kernels.
#   bash tools/gpu_round.sh [tag]
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 900 python tools/run_configs.py --configs C1,C2,C3,C4,C5 --reps 5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-dense > gpurun_out/ncu_launch.log 2>&1
# second call of tools/prof_unit.py (the graph-recorded one) for each kernel
DS_DENSE=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:eps_unit_kernel' -s 1 -c 1 -o gpurun_out/prof_tile_c2_${TAG} python tools/prof_unit.py > gpurun_out/ncu_tile.log 2>&1
DS_CONFIG=C4 DS_DENSE=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:eps_unit_kernel' -s 1 -c 1 -o gpurun_out/prof_tile_c4_${TAG} python tools/prof_unit.py > gpurun_out/ncu_tile_c4.log 2>&1
DS_DENSE=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:union_|scan_lookback|unit_list|roots' -s 6 -c 6 -o gpurun_out/prof_merge_${TAG} python tools/prof_unit.py > gpurun_out/ncu_merge.log 2>&1
echo done
