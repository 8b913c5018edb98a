#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sk_build.log 2>&1
for che in 8 16 32; do
SSNAL_CSCJ_CHE=$che timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/sk_launches_che$che.csv python scripts/prof_sparse_kernels.py 2 > gpurun_out/sk_che$che.log 2>&1
python scripts/launch_summary.py gpurun_out/sk_launches_che$che.csv > gpurun_out/sk_launches_che$che.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cscj_xt_kernel|csr_xd_kernel" --launch-skip 2 --launch-count 2 \
  -o gpurun_out/sk_full python scripts/prof_sparse_kernels.py 2 > gpurun_out/sk_full.log 2>&1
