#!/bin/bash
# iteration check: selected GPU tests, config-4 timings and launch list
# usage: bash scripts/gpu_iter.sh "<pytest -k expr>" <tag>
mkdir -p gpurun_out
K="$1"; TAG="${2:-it}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_tests.log 2>&1
fi
timeout 600 python scripts/run_config.py 4 1 3 > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_c4_launches.csv python scripts/run_config.py 4 1 1 > gpurun_out/${TAG}_c4_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_c4_launches.csv > gpurun_out/${TAG}_c4_launches.txt
