mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$? >> gpurun_out/pytest_new.log
REPS=3 timeout 900 bash tools/ab.sh C4 variants/a_base.so variants/pp.so > gpurun_out/ab26.log 2>&1
cp variants/pp.so paper_1506_02226_b200/libdensescan_b200.so
DS_CONFIG=C4 DS_KT_OUT=gpurun_out/kt_C4_pp.txt DS_RUNS=3 timeout 300 python tools/one_run.py > /dev/null 2>&1 || true
