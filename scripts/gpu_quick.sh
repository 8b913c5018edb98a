#!/bin/bash
# gpurun helper: build, then one pytest selection (args: tag, pytest args...)
mkdir -p gpurun_out
T=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 python -m pytest "$@" > gpurun_out/${T}_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/${T}_tests.log
