mkdir -p gpurun_out
REPS=5 timeout 900 bash tools/ab.sh C3,C5 variants/y_b64.so variants/b32.so variants/b128.so > gpurun_out/ab21.log 2>&1
