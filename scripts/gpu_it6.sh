#!/bin/bash
mkdir -p gpurun_out
T=${1:-it6}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "api or cholesky or config4" > gpurun_out/${T}_tests.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "config2 or config3" --durations=5 > gpurun_out/${T}_tests_sparse.log 2>&1
