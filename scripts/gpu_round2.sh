#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sharded.py -x -q > gpurun_out/t_kern.log 2>&1; echo EXIT $? >> gpurun_out/t_kern.log
timeout 900 python -m pytest tests/test_gpu_solver.py -x -q -k sparse > gpurun_out/t_sparse.log 2>&1; echo EXIT $? >> gpurun_out/t_sparse.log
timeout 300 python scripts/prof_sparse.py 2 > gpurun_out/s2_plain.log 2>&1
timeout 900 python scripts/prof_sparse.py 3 > gpurun_out/s3_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 --launch-count 700 --csv \
  --log-file gpurun_out/s3_launches.csv python scripts/prof_sparse.py 3 1 > gpurun_out/s3_ncu.log 2>&1
