#!/bin/bash
# Round check on one GPU: tests, smoke, the default bench line, then the profiling pass.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rs > gpurun_out/round_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/round_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/round_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/round_smoke.log
timeout 900 python bench.py > gpurun_out/round_bench.json 2> gpurun_out/round_bench.err
echo "bench rc=$?" >> gpurun_out/round_bench.err
timeout 1500 bash scripts/gpu_profile_all.sh > gpurun_out/round_profile.log 2>&1
echo "profile rc=$?" >> gpurun_out/round_profile.log
