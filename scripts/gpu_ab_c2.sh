#!/bin/bash
# C2 A/B of two library builds (alternating, 3 rounds each).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in base exp; do
    MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_$v.so timeout 300 python scripts/c2_time.py >> gpurun_out/ab_c2.log 2>&1
  done
done
