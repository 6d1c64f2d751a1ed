#!/bin/bash
# Sharded tile mapping: sharded + grid GPU tests, bench with the 1-rank sharded C5 leg.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_grid.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1h_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1h_tests.log
timeout 1200 python bench.py --c5-sharded > gpurun_out/r1h_bench.json 2> gpurun_out/r1h_bench.err
echo "bench rc=$?" >> gpurun_out/r1h_bench.err
