#!/bin/bash
# DMMA prefetch A/B: C3 with the previous and the new library, DMMA GPU tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_prev.so C3_PATHS=3 timeout 300 python scripts/c3_bench.py > gpurun_out/k_c3_prev.log 2>&1
C3_PATHS=3 timeout 300 python scripts/c3_bench.py > gpurun_out/k_c3_new.log 2>&1
MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_prev.so C3_PATHS=3 timeout 300 python scripts/c3_bench.py > gpurun_out/k_c3_prev2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dmma.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1k_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1k_tests.log
