#!/bin/bash
# Config-1 profiling pass (run under gpurun): launch list of one solve and full ncu
# captures of the top kernels (each command has already run clean without ncu).
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 430 --launch-count 430 --csv \
  --log-file gpurun_out/c1_launches.csv python scripts/profile_solve.py 1 2 > gpurun_out/c1_ncu.log 2>&1
for k in stream_xd_kernel proj_cluster_kernel chol_tc_kernel accept_q_kernel hs_finish_dots_kernel; do
  f=$(echo "$k" | tr -d '<')
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip 20 --launch-count 1 \
    -o "gpurun_out/c1_$f" -f python scripts/profile_solve.py 1 2 > "gpurun_out/c1_full_$f.log" 2>&1
done
