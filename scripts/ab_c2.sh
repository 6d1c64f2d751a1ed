#!/bin/bash
# A/B of C2 step timing across libraries: bash scripts/ab_c2.sh ab/a.so ab/b.so ... (alternating, 3 rounds)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3; do
  for lib in "$@"; do
    for alg in ${C2_ALGS:-ra}; do
      MPAX_LIB=$PWD/$lib C2_ALG=$alg timeout 300 python scripts/c2_time.py 2>&1 | tail -1
    done
  done
done
