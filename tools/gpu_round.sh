#!/bin/bash
# Full GPU iteration: smoke, GPU parity tests, bench (C2), all configs, ncu launch list + full captures.
#   bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 900 python tools/run_configs.py --configs C1,C2,C3,C4,C5 --reps 5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eps_unit -s 3 -c 1 -o gpurun_out/prof_tile_${TAG} python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_tile.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_ -s 6 -c 2 -o gpurun_out/prof_union_${TAG} python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_union.log 2>&1
echo done
