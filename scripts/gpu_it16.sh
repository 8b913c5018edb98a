#!/bin/bash
mkdir -p gpurun_out
T=${1:-it16}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSSNAL_CHOL_TIMING -o /tmp/chol_probe scripts/chol_probe.cu && /tmp/chol_probe 500 > gpurun_out/${T}_chol_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "cholesky or gram or config4 or svr or golden" > gpurun_out/${T}_tests.log 2>&1
timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_c4_launches.csv python scripts/run_config.py 4 1 1 > gpurun_out/${T}_c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/${T}_c4_launches.csv > gpurun_out/${T}_c4_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gram_kernel" --launch-skip 0 --launch-count 1 \
  -o gpurun_out/${T}_c4_gram -f python scripts/run_config.py 4 1 1 > gpurun_out/${T}_ncu_gram.log 2>&1
