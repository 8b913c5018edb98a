timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g2_tests.log 2>&1
timeout 120 python scripts/time_solve.py 1 20 > gpurun_out/g2_time.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:chol_tc_kernel -s 10 -c 1 -o gpurun_out/g2_chol python scripts/profile_solve.py 1 2 > gpurun_out/g2_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:proj_cluster_kernel -s 20 -c 1 -o gpurun_out/g2_proj python scripts/profile_solve.py 1 2 >> gpurun_out/g2_ncu.log 2>&1
