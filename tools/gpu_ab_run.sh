mkdir -p gpurun_out
REPS=3 timeout 900 bash tools/ab.sh C4 variants/a_base.so variants/w256.so variants/w512.so > gpurun_out/ab25.log 2>&1
