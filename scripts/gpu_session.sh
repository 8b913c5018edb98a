#!/bin/bash
# One gpurun session: build, GPU tests, default bench (optionally a tag and a pytest -k filter)
mkdir -p gpurun_out
T=${1:-s}
K=${2:-}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${T}_tests.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1
fi
echo "EXIT $?" >> gpurun_out/${T}_tests.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "EXIT $?" >> gpurun_out/${T}_bench.err
