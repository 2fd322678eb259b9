#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the whole hot path on the tiny config and a
# 3.3K multi-pattern config; logs under gpurun_out/ (copied to profiles/)
cd $GRAFT_REPO_ROOT
python __graft_entry__.py > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 99 python profiles/tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "tool=$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
