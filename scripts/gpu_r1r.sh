#!/bin/bash
# Batched create uploads: C2 breakdown, full GPU tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/c2_breakdown.py > gpurun_out/r1r_breakdown.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1r_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1r_tests.log
