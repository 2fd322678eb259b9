#!/bin/bash
# round-2 (second session) evaluation pass on one B200: smoke, full GPU tests, bench lines (all workloads), reference
# arm, f1/f3 measurement lines, launch list, ncu sections of the hot kernels (compute-sanitizer is closed on this pool)
cd $GRAFT_REPO_ROOT
O=gpurun_out
python __graft_entry__.py > $O/e_build.log 2>&1
python __graft_entry__.py smoke > $O/e_smoke.log 2>&1; echo "smoke rc=$?" >> $O/e_smoke.log
timeout 600 python bench.py > $O/e_bench_default.json 2> $O/e_bench_default.err
for w in 1 2 3 5 6; do timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $O/e_bench_w$w.json 2> $O/e_bench_w$w.err; done
timeout 500 python bench.py --impl reference --steps 3 --warmup 1 > $O/e_bench_ref.json 2> $O/e_bench_ref.err
timeout 600 python profiles/tools/analysis_bench.py > $O/e_analysis.json 2> $O/e_analysis.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e_launches_1m.csv python profiles/tools/prof_sparse.py 4 > $O/e_ncu_l.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e_launches_128k.csv python profiles/tools/prof_sparse.py 1 > $O/e_ncu_l2.log 2>&1
SEC="--section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy --section WarpStateStats --section SchedulerStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active"
timeout 900 ncu $SEC --clock-control none -k regex:'attn_kernel|slab_tc|grid_acc|gather_rows|merge' -s 21 -c 7 -o $O/e_sections_1m python profiles/tools/prof_sparse.py 4 > $O/e_ncu_s1.log 2>&1
timeout 600 ncu $SEC --clock-control none -k regex:'attn_kernel|slab_tc|grid_acc|gather_rows|merge' -s 21 -c 7 -o $O/e_sections_128k python profiles/tools/prof_sparse.py 1 > $O/e_ncu_s2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=0 > $O/e_gpu_tests.log 2>&1; echo "rc=$?" >> $O/e_gpu_tests.log
