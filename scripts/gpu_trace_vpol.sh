#!/bin/bash
# C5 per-phase timings (trace library) for the vector L2 policies MPAX_GRID_VPOL=0/1/2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
for v in 0 1 2; do
  MPAX_GRID_VPOL=$v timeout 600 python scripts/c5_run.py > gpurun_out/v_c5_vpol$v.log 2>&1
done
