#!/bin/bash
# Sparse configs (run under gpurun): plain timed solves, then ncu launch windows in the CG phase.
mkdir -p gpurun_out
timeout 300 python scripts/prof_sparse.py 2 > gpurun_out/s2_plain.log 2>&1
timeout 600 python scripts/prof_sparse.py 3 3 > gpurun_out/s3_plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 --launch-count 700 --csv \
  --log-file gpurun_out/s2_launches.csv python scripts/prof_sparse.py 2 2 > gpurun_out/s2_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 --launch-count 700 --csv \
  --log-file gpurun_out/s3_launches.csv python scripts/prof_sparse.py 3 1 > gpurun_out/s3_ncu.log 2>&1
