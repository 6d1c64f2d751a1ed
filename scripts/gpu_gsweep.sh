#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/gsweep.log
for g in 2 4 8; do for gt in 1 2 4; do
  echo "G=$g GT=$gt" >> gpurun_out/gsweep.log
  MPAX_GRID_G=$g MPAX_GRID_GT=$gt PROF_M=1000000 PROF_K=128 timeout 120 python scripts/prof_grid.py 2>&1 | grep "^1 " >> gpurun_out/gsweep.log
done; done
