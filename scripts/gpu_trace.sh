#!/bin/bash
# Per-phase timings of the grid kernel (trace library), C5 and C4, both SpMV mappings.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
tag=${TRACE_TAG:-t}
timeout 600 python scripts/c5_run.py > gpurun_out/${tag}_c5_tile.log 2>&1
MPAX_GRID_G=4 MPAX_GRID_GT=2 timeout 600 python scripts/c5_run.py > gpurun_out/${tag}_c5_glanes.log 2>&1
PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/${tag}_c4_tile.log 2>&1
MPAX_GRID_G=4 MPAX_GRID_GT=2 PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/${tag}_c4_glanes.log 2>&1
