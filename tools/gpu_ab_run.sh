mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
REPS=5 timeout 900 bash tools/ab.sh C3,C5,C2 variants/a_base.so variants/dt.so > gpurun_out/ab22.log 2>&1
REPS=3 timeout 900 bash tools/ab.sh C4 variants/a_base.so variants/dt.so > gpurun_out/ab23.log 2>&1
