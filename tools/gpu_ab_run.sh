mkdir -p gpurun_out
REPS=5 timeout 900 bash tools/ab.sh C2,C3,C5 variants/a_base.so variants/x_minb5.so > gpurun_out/ab19.log 2>&1
