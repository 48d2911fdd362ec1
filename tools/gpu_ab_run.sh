mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
REPS=7 timeout 900 bash tools/ab.sh C2,C3,C5 variants/a_base.so variants/pb.so > gpurun_out/ab27.log 2>&1
REPS=3 timeout 900 bash tools/ab.sh C4 variants/a_base.so variants/pb.so > gpurun_out/ab28.log 2>&1
