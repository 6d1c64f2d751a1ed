#!/bin/bash
# Two-pass phase B: grid GPU tests, C5 traces with the split on (default) / off.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grid.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1l_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1l_tests.log
export MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
timeout 600 python scripts/c5_run.py > gpurun_out/l_c5_split.log 2>&1
MPAX_GRID_SPLIT=0 timeout 600 python scripts/c5_run.py > gpurun_out/l_c5_nosplit.log 2>&1
