#!/bin/bash
# ncu capture of the stage-1 kernel: DS_CONFIG=C4 DS_DENSE=0 bash tools/gpu_prof_unit.sh <name>
mkdir -p gpurun_out
python tools/prof_unit.py > gpurun_out/prof_unit_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eps_unit -c ${COUNT:-4} -o gpurun_out/prof_${1:-unit} python tools/prof_unit.py > gpurun_out/ncu_unit.log 2>&1
tail -3 gpurun_out/ncu_unit.log
