#!/bin/bash
# warm-cache launch windows inside the CG phase of configs 2 and 3 (run under gpurun)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --launch-skip 3000 --launch-count 600 --csv \
  --log-file gpurun_out/s2w_launches.csv python scripts/prof_sparse.py 2 2 > gpurun_out/s2w_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --launch-skip 3000 --launch-count 600 --csv \
  --log-file gpurun_out/s3w_launches.csv python scripts/prof_sparse.py 3 1 > gpurun_out/s3w_ncu.log 2>&1
