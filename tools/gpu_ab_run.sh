mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_big.py -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
REPS=7 timeout 900 bash tools/ab.sh C2,C3,C5 variants/a_base.so variants/r_swap.so > gpurun_out/ab13.log 2>&1
