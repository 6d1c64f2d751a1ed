#!/bin/bash
# GPU tests + bench after the in-place device SpMV diagnostic.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1o_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1o_tests.log
timeout 900 python bench.py > gpurun_out/r1o_bench.json 2> gpurun_out/r1o_bench.err
echo "bench rc=$?" >> gpurun_out/r1o_bench.err
