#!/bin/bash
# Config-1 profiling pass (run under gpurun): projection pass counts, launch list of one
# solve, full ncu captures of the top kernels.
set -x
mkdir -p gpurun_out
SSNAL_DEBUG_PROJ=1 SSNAL_DEBUG_CG=1 timeout 120 python scripts/profile_solve.py 1 1 > gpurun_out/c1_dbg.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 700 --launch-count 700 --csv \
  --log-file gpurun_out/c1_launches.csv python scripts/profile_solve.py 1 2 > gpurun_out/c1_ncu.log 2>&1
for k in proj_cluster_kernel chol_tc_kernel stream_xd_kernel proj_fused_kernel rows_gram_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 20 --launch-count 1 \
    -o gpurun_out/c1_$k -f python scripts/profile_solve.py 1 2 > gpurun_out/c1_full_$k.log 2>&1
done
