mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
REPS=7 timeout 900 bash tools/ab.sh C3,C5,C2 variants/a_base.so variants/ul.so > gpurun_out/ab24.log 2>&1
