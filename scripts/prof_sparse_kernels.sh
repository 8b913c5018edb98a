#!/bin/bash
# per-kernel times (ncu launch list) and full captures of the CG products on config-3 data
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sk_build.log 2>&1
T=${1:-sk}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python scripts/prof_sparse_kernels.py 2 > gpurun_out/${T}.log 2>&1
python scripts/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cscj_xt_kernel|csrj_xd_dot" --launch-skip 2 --launch-count 2 \
  -o gpurun_out/${T}_full python scripts/prof_sparse_kernels.py 2 > gpurun_out/${T}_full.log 2>&1
