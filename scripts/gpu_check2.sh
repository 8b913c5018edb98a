#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo EXIT $? >> gpurun_out/t_all.log
timeout 300 python scripts/prof_sparse.py 2 > gpurun_out/s2_plain.log 2>&1
timeout 900 python scripts/prof_sparse.py 3 > gpurun_out/s3_plain.log 2>&1
