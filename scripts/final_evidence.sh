#!/bin/bash
# Round-end style evidence at HEAD: GPU tests, smoke, default bench (config 4), reference arm,
# the other configs, the sharded driver at N = 1, launch lists of configs 4 and 1.
mkdir -p gpurun_out
T=${1:-fin}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/${T}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench_config4.json 2> gpurun_out/${T}_bench_config4.err
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_reference_config4.json 2> gpurun_out/${T}_bench_reference_config4.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_config1.json 2>/dev/null
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/${T}_bench_config2.json 2>/dev/null
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 > gpurun_out/${T}_bench_config3.json 2>/dev/null
timeout 300 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_config4_sharded_n1.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_config4.csv \
  python scripts/run_config.py 4 1 1 > gpurun_out/${T}_ncu4.log 2>&1
python scripts/launch_summary.py gpurun_out/${T}_launches_config4.csv > gpurun_out/${T}_launches_config4_solve.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_config1.csv \
  python scripts/run_config.py 1 1 1 > gpurun_out/${T}_ncu1.log 2>&1
python scripts/launch_summary.py gpurun_out/${T}_launches_config1.csv > gpurun_out/${T}_launches_config1_solve.txt
