mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
REPS=3 timeout 900 bash tools/ab.sh C4 variants/a_base.so variants/ca.so > gpurun_out/ab29.log 2>&1
REPS=3 timeout 900 bash tools/ab.sh C2 variants/a_base.so variants/ca.so > gpurun_out/ab30.log 2>&1
