#!/bin/bash
# Session check: gather microbenchmark, GPU tests, default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1d_smi.txt 2>&1
timeout 300 scripts/micro/gather_bench > gpurun_out/r1d_gather.jsonl 2>&1
echo "gather rc=$?" >> gpurun_out/r1d_gather.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1d_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1d_tests.log
timeout 900 python bench.py > gpurun_out/r1d_bench.json 2> gpurun_out/r1d_bench.err
echo "bench rc=$?" >> gpurun_out/r1d_bench.err
