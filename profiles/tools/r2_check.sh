#!/bin/bash
# build + quick parity + bench lines (+ optional full-size parity)
cd $GRAFT_REPO_ROOT
python __graft_entry__.py > gpurun_out/c_build.log 2>&1
python __graft_entry__.py smoke > gpurun_out/c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/c_smoke.log
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_dense.py -x -q > gpurun_out/c_tests.log 2>&1; rc=$?; echo "tests rc=$rc" >> gpurun_out/c_tests.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 400 python bench.py --workload 1 --steps 5 --warmup 3 --no-cpu --no-e2e --dense 0 > gpurun_out/c_bench_w1.json 2> gpurun_out/c_bench_w1.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --dense 0 > gpurun_out/c_bench_w4.json 2> gpurun_out/c_bench_w4.err
if [ "$1" == "full" ]; then
  ( time timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -rA --durations=0 ) > gpurun_out/c_full.log 2>&1; echo "rc=$?" >> gpurun_out/c_full.log
fi
