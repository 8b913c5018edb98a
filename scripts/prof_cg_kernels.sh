#!/bin/bash
# config 3 (CSR Zipf 4M x 1M): ncu --set full of the CG phase's kernels inside a real solve
# (launch 3000 of each, sigma = 125..625) and a 600-launch window of the CG phase
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cgk_build.log 2>&1
for k in cscj_xt_kernel csrj_xd_dot_kernel cg_update_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3000 --launch-count 1 \
    -f -o gpurun_out/c3_$k python scripts/prof_sparse.py 3 6 > gpurun_out/cgk_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 30000 --launch-count 600 --csv \
  --log-file gpurun_out/c3_cg_window.csv python scripts/prof_sparse.py 3 6 > gpurun_out/cgk_window.log 2>&1
python scripts/launch_summary.py gpurun_out/c3_cg_window.csv > gpurun_out/c3_cg_window.txt
