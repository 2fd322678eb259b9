#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the whole hot path on the tiny config and a
# 3.3K multi-pattern config; logs under gpurun_out/ (copied to profiles/)
cd $GRAFT_REPO_ROOT
python __graft_entry__.py > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
# memcheck on every config; the slower tools on the tiny config
timeout 900 $CS --tool memcheck --print-limit 20 --error-exitcode 99 python profiles/tools/sanitize_run.py > gpurun_out/sanitize_memcheck.log 2>&1
echo "tool=memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
for tool in racecheck synccheck initcheck; do
  timeout 600 $CS --tool $tool --print-limit 20 --error-exitcode 99 python profiles/tools/sanitize_run.py tiny > gpurun_out/sanitize_$tool.log 2>&1
  echo "tool=$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
