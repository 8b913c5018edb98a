#!/bin/bash
mkdir -p gpurun_out
T=${1:-it10}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "projection or config4 or svr or gram or solver" > gpurun_out/${T}_tests.log 2>&1
timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_c4_launches.csv python scripts/run_config.py 4 1 1 > gpurun_out/${T}_c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/${T}_c4_launches.csv > gpurun_out/${T}_c4_launches.txt
SSNAL_CG_ETA_CAP=1e-2 timeout 900 python scripts/run_config.py 2 1 1 > gpurun_out/${T}_c2_eta2.json 2>&1
SSNAL_CG_ETA_CAP=1e-2 timeout 1200 python scripts/run_config.py 3 1 1 > gpurun_out/${T}_c3_eta2.json 2>&1
