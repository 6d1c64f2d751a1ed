#!/bin/bash
# Sharded two-pass rows step: sharded GPU tests, 1-rank sharded C5 bench leg.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1q_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1q_tests.log
timeout 1200 python bench.py --c5-sharded --no-large --no-dense --no-spo --no-cpu-baseline > gpurun_out/r1q_bench.json 2> gpurun_out/r1q_bench.err
echo "bench rc=$?" >> gpurun_out/r1q_bench.err
