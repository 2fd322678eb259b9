#!/bin/bash
cd $GRAFT_REPO_ROOT
python __graft_entry__.py > /dev/null 2>&1
( time timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=0 ) > gpurun_out/ft_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ft_tests.log
