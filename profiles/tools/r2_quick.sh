#!/bin/bash
# quick GPU pass: build check, small parity tests, bench at 128K and 1M
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/q_gpu.txt 2>&1
python __graft_entry__.py smoke > gpurun_out/q_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/q_smoke.log
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_dense.py -x -q > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests.log
timeout 400 python bench.py --workload 1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/q_bench_w1.json 2> gpurun_out/q_bench_w1.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/q_bench_w4.json 2> gpurun_out/q_bench_w4.err
