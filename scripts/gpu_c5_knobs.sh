#!/bin/bash
# C5 attempt time under the grid kernel's experiment knobs (fixed 256 accepted steps, raPDHG).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "MPAX_GRID_DYN=3" "MPAX_GRID_DYN=6" "MPAX_GRID_VPOL=1" "MPAX_GRID_VPOL=2" "MPAX_GRID_TDIST=1" \
           "MPAX_GRID_LEAN=1" "MPAX_GRID_LEAN=2" "MPAX_GRID_LEAN=7" "MPAX_GRID_GT=2" "MPAX_GRID_SPLIT=0"; do
  echo "== $cfg" >> gpurun_out/c5_knobs.log
  env $cfg C5_ALGS=ra C5_LIMIT=256 C5_REPS=2 timeout 300 python scripts/c5_run.py 2>&1 | grep "ra fp64" >> gpurun_out/c5_knobs.log
done
