#!/bin/bash
# round-end style evidence: full GPU tests, smoke, bench (ours + reference arm)
mkdir -p gpurun_out
T=${1:-full}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${T}_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
nproc > gpurun_out/${T}_nproc.txt
