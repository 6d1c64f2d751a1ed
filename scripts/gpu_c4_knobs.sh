#!/bin/bash
# C4 attempt time under the grid kernel's experiment knobs (256 accepted raPDHG steps).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "MPAX_GRID_GT=1" "MPAX_GRID_GT=4" "MPAX_GRID_GT=8" "MPAX_GRID_G=2" "MPAX_GRID_G=4" "MPAX_GRID_MINB=2" \
           "MPAX_GRID_DYN=3" "MPAX_GRID_DYN=0" "MPAX_GRID_LEAN=0" "MPAX_GRID_LEAN=1" "MPAX_GRID_GT=1 MPAX_GRID_DYN=3"; do
  echo "== $cfg" >> gpurun_out/c4_knobs.log
  env $cfg PROF_K=256 timeout 300 python scripts/prof_grid.py 2>&1 | grep "^1 " >> gpurun_out/c4_knobs.log
done
