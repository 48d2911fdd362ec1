#!/bin/bash
# Quick GPU check: stage timings (all configs), GPU parity tests, ncu launch list of the C2 bench.
#   bash tools/gpu_check.sh TAG [configs]
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python tools/tile_bench.py --configs ${2:-C1,C2,C3,C4,C5} > gpurun_out/tile_bench_${TAG}.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_${TAG}.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-dense > gpurun_out/ncu_launch_${TAG}.log 2>&1
