#!/bin/bash
# config 4 (dense eps-SVR, 1M x 500): timed solves, launch list of one solve, ncu --set full of the q-space Gram
mkdir -p gpurun_out
timeout 600 python scripts/run_config.py 4 1 2 > gpurun_out/c4_run.json 2> gpurun_out/c4_run.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/c4_launches.csv python scripts/run_config.py 4 1 1 > gpurun_out/c4_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gram_kernel" --launch-skip 10 --launch-count 1 \
  -o gpurun_out/c4_gram_kernel -f python scripts/run_config.py 4 1 1 > gpurun_out/c4_full_gram.log 2>&1
