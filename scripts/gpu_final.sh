#!/bin/bash
# round-end evidence pass: GPU tests, bench (ours + reference arm), configs 2-4, config-1 launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "csr" > gpurun_out/t_csr.log 2>&1; echo EXIT $? >> gpurun_out/t_csr.log
grep -q "EXIT 0" gpurun_out/t_csr.log || exit 1
timeout 300 python -m pytest tests/test_gpu_solver.py -x -q -k "sparse_config_shapes and cg" > gpurun_out/t_cg.log 2>&1; echo EXIT $? >> gpurun_out/t_cg.log
grep -q "EXIT 0" gpurun_out/t_cg.log || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo EXIT $? >> gpurun_out/t_all.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 300 python scripts/prof_sparse.py 2 > gpurun_out/s2_plain.log 2>&1
timeout 600 python scripts/run_config.py 4 1 2 > gpurun_out/c4_run.json 2> gpurun_out/c4_run.err
timeout 900 python scripts/prof_sparse.py 3 > gpurun_out/s3_plain.log 2>&1
