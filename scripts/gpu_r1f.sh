#!/bin/bash
# Dynamic tile driver: GPU tests, C5/C4 traces, C5 full runs, bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1f_tests.log
TRACE_TAG=f bash scripts/gpu_trace.sh
timeout 900 python bench.py > gpurun_out/r1f_bench.json 2> gpurun_out/r1f_bench.err
echo "bench rc=$?" >> gpurun_out/r1f_bench.err
