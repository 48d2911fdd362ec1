#!/bin/bash
# Iteration check: GPU tests, C2 bench (no CPU leg), host overhead, all-config stage times.
#   bash tools/gpu_iter2.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu --no-dense > gpurun_out/bench_${TAG}.log 2>&1
timeout 300 python tools/host_overhead.py > gpurun_out/host_${TAG}.log 2>&1
timeout 600 python tools/run_configs.py --configs C1,C2,C3,C5 --reps 5 > gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/configs_${TAG}.err
