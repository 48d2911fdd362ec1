#!/bin/bash
# One GPU iteration: build checks, microbench, parity tests, bench, optional ncu.
#   bash tools/gpu_iter.sh [ncu]
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/fp32_microbench tools/fp32_microbench.cu \
  && timeout 120 /tmp/fp32_microbench > gpurun_out/microbench.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
if [ "$1" == "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_chunks -s 2 -c 2 -o gpurun_out/prof_union python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_union.log 2>&1
fi
