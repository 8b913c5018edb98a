#!/bin/bash
# Config-1 profiling pass at HEAD (run under gpurun): launch list of one warm solve
# (534 launches) and full ncu captures of the two top kernels.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 534 --launch-count 534 --csv \
  --log-file gpurun_out/c1_launches.csv python scripts/profile_solve.py 1 2 > gpurun_out/c1_ncu.log 2>&1
for k in proj_cluster_kernel chol_tc_kernel stream_xd_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip 20 --launch-count 1 \
    -o "gpurun_out/c1_$k" -f python scripts/profile_solve.py 1 2 > "gpurun_out/c1_full_$k.log" 2>&1
done
