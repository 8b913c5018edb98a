#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/it2_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "solver or gram or newton" > gpurun_out/it2_tests.log 2>&1
SSNAL_DEBUG_PROJ=1 timeout 600 python scripts/run_config.py 4 1 1 > gpurun_out/it2_c4dbg.json 2> gpurun_out/it2_c4dbg.err
timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/it2_c4.json 2> gpurun_out/it2_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/it2_c4_launches.csv python scripts/run_config.py 4 1 1 > gpurun_out/it2_c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/it2_c4_launches.csv > gpurun_out/it2_c4_launches.txt
