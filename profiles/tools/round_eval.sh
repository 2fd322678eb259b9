#!/bin/bash
# full evaluation pass on the GPU box: tests, bench lines, launch list, ncu sections
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
for w in 2 3 4; do timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err; done
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --dense 0 > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy --section WarpStateStats --section SchedulerStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:'attn_kernel|merge_kernel|slab_kernel|grid_acc|gather_rows' -c 7 -o gpurun_out/sections python profiles/tools/prof_sparse.py 1 > gpurun_out/ncu_sections.log 2>&1
