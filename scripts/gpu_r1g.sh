#!/bin/bash
# GPU tests, C5 trace (dyn = 2 default vs 3), bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1g_tests.log
export MPAX_LIB_TRACE=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
for d in 2 3; do
  MPAX_LIB=$MPAX_LIB_TRACE MPAX_GRID_DYN=$d timeout 600 python scripts/c5_run.py > gpurun_out/g_c5_dyn$d.log 2>&1
done
timeout 900 python bench.py > gpurun_out/r1g_bench.json 2> gpurun_out/r1g_bench.err
echo "bench rc=$?" >> gpurun_out/r1g_bench.err
