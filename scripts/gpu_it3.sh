#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/it3_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "cholesky or gram or large_n" > gpurun_out/it3_tests.log 2>&1
timeout 600 python scripts/run_config.py 4 1 2 > gpurun_out/it3_c4.json 2> gpurun_out/it3_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/it3_c4_launches.csv python scripts/run_config.py 4 1 1 > gpurun_out/it3_c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/it3_c4_launches.csv > gpurun_out/it3_c4_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:proj_multi_kernel" --launch-skip 30 --launch-count 1 \
  -o gpurun_out/it3_proj_multi -f python scripts/run_config.py 4 1 1 > gpurun_out/it3_ncu_proj.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:chol_cluster" --launch-skip 30 --launch-count 1 \
  -o gpurun_out/it3_chol_cluster -f python scripts/run_config.py 4 1 1 > gpurun_out/it3_ncu_chol.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gram_kernel" --launch-skip 3 --launch-count 1 \
  -o gpurun_out/it3_gram -f python scripts/run_config.py 4 1 1 > gpurun_out/it3_ncu_gram.log 2>&1
