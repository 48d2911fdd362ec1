mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
REPS=5 timeout 900 bash tools/ab.sh C2,C3,C5 variants/a_base.so variants/v_group4.so variants/w_group2.so > gpurun_out/ab17.log 2>&1
REPS=3 timeout 900 bash tools/ab.sh C4 variants/a_base.so variants/v_group4.so variants/w_group2.so > gpurun_out/ab18.log 2>&1
