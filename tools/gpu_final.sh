#!/bin/bash
# Round-end evidence: tools/gpu_round.sh, then kernel timelines (C2, C4, C5) from the
# tools/kt_patch.py build (variants/kt.so, copied over the product library last).
TAG=${1:-r02}
bash tools/gpu_round.sh $TAG
cp variants/kt.so paper_1506_02226_b200/libdensescan_b200.so
for C in C2 C4 C5; do
  DS_CONFIG=$C DS_KT_OUT=gpurun_out/kt_${C}_${TAG}.txt DS_RUNS=4 timeout 300 python tools/one_run.py > gpurun_out/kt_${C}.log 2>&1
done
echo final_done
