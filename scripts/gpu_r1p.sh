#!/bin/bash
# Global dynamic phase A: grid tests, C5 / C4 traces at dyn = 2 / 6.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grid.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1p_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1p_tests.log
export MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
for d in 2 6; do
  MPAX_GRID_DYN=$d timeout 600 python scripts/c5_run.py > gpurun_out/p_c5_dyn$d.log 2>&1
  MPAX_GRID_DYN=$d MPAX_GRID_GT=1 PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/p_c4_dyn$d.log 2>&1
done
