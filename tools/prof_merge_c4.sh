mkdir -p gpurun_out
DS_CONFIG=C4 DS_DENSE=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:union_' -s 2 -c 2 -o gpurun_out/prof_merge_c4 python tools/prof_unit.py > gpurun_out/ncu_merge_c4.log 2>&1
