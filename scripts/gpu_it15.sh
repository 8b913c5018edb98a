#!/bin/bash
mkdir -p gpurun_out
T=${1:-it15}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "cholesky or pspace or config1 or golden or native" > gpurun_out/${T}_tests.log 2>&1
timeout 600 python scripts/run_config.py 1 1 5 > gpurun_out/${T}_c1.json 2> gpurun_out/${T}_c1.err
timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/${T}_c4_fb2.json 2> gpurun_out/${T}_c4_fb2.err
SSNAL_FIRST_BATCH=4 timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/${T}_c4_fb4.json 2> gpurun_out/${T}_c4_fb4.err
SSNAL_FIRST_BATCH=3 timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/${T}_c4_fb3.json 2> gpurun_out/${T}_c4_fb3.err
SSNAL_FIRST_BATCH=1 timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/${T}_c4_fb1.json 2> gpurun_out/${T}_c4_fb1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_c1_launches.csv python scripts/run_config.py 1 1 2 > gpurun_out/${T}_c1_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/${T}_c1_launches.csv > gpurun_out/${T}_c1_launches.txt
