#!/bin/bash
# A/B of the C5 grid attempt across libraries (ab/*.so): PROF_K accepted steps, raPDHG (+ r2 with PROF_ALGS)
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
  echo "== $lib"
  MPAX_LIB=$PWD/$lib PROF_K=${PROF_K:-128} timeout 900 python scripts/c5_variants.py 2>&1 | grep round
done
