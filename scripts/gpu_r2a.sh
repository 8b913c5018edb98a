#!/bin/bash
# round 2 first look: FP64 tensor peak, config 4 timings and launch list at HEAD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_peak scripts/dmma_peak.cu && timeout 120 /tmp/dmma_peak > gpurun_out/dmma_peak.txt 2>&1
timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/c4_run.json 2> gpurun_out/c4_run.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c4_launches.csv python scripts/run_config.py 4 1 1 > gpurun_out/c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/c4_launches.csv > gpurun_out/c4_launches.txt
