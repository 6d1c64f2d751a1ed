#!/bin/bash
# GPU tests + smoke + short bench + ncu launch list + one full capture of the instance kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh "$1"
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$PROFILE" ]; then bash scripts/gpu_profile.sh; fi
