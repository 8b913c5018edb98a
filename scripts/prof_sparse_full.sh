#!/bin/bash
# ncu --set full captures of the sparse CG kernels (config 2 and 3, inside the CG phase)
mkdir -p gpurun_out
for k in csr_xd_kernel cscj_xt_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip 400 --launch-count 1 \
    -o "gpurun_out/s2_$k" -f python scripts/prof_sparse.py 2 2 > "gpurun_out/s2_full_$k.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip 400 --launch-count 1 \
    -o "gpurun_out/s3_$k" -f python scripts/prof_sparse.py 3 1 > "gpurun_out/s3_full_$k.log" 2>&1
done
