#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSSNAL_CHOL_TIMING -o /tmp/chol_probe scripts/chol_probe.cu && /tmp/chol_probe 500 > gpurun_out/chol_probe.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/bench_proj.py > gpurun_out/proj_probe.txt 2>&1
