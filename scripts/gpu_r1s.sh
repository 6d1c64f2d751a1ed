#!/bin/bash
# setup_small: unrolled finiteness checks -- C2 breakdown and the validation / parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/c2_breakdown.py > gpurun_out/r1s_breakdown.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_library.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1s_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1s_tests.log
