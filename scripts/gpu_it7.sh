#!/bin/bash
mkdir -p gpurun_out
T=${1:-it7}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${T}_tests.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --sharded --steps 2 --warmup 1 > gpurun_out/${T}_bench_sharded.json 2> gpurun_out/${T}_bench_sharded.err
