#!/bin/bash
# All five configurations on one GPU, C oracle parity where it finishes in minutes.
mkdir -p gpurun_out
make -s -C oracle
timeout 2400 python tools/run_configs.py --configs ${CONFIGS:-C1,C2,C3,C4,C5} --oracle ${ORACLE:-C1,C2,C3,C4} --reps 5 ${DENSE:+--dense} > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
tail -5 gpurun_out/configs.err
