#!/bin/bash
# C5 / C4 per-phase timings (trace library): contiguous vs interleaved tile distribution.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
for td in 0 1; do
  MPAX_GRID_TDIST=$td timeout 600 python scripts/c5_run.py > gpurun_out/td_c5_$td.log 2>&1
  MPAX_GRID_TDIST=$td PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/td_c4_$td.log 2>&1
done
