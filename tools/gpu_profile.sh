mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:eps_tile_kernelILi2ELi1ELb1E -s 1 -c 1 -o gpurun_out/prof_tile python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_tile.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_words -s 1 -c 1 -o gpurun_out/prof_union python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_union.log 2>&1
ls -la gpurun_out
