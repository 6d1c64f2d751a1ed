#!/bin/bash
# Tile-mapping A/B: GPU tests, C5 with the new (default) and the old (G lanes) mapping, bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1e_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1e_tests.log
timeout 600 python scripts/c5_run.py > gpurun_out/r1e_c5_tile.log 2>&1
MPAX_GRID_G=4 MPAX_GRID_GT=2 timeout 600 python scripts/c5_run.py > gpurun_out/r1e_c5_glanes.log 2>&1
timeout 900 python bench.py > gpurun_out/r1e_bench.json 2> gpurun_out/r1e_bench.err
echo "bench rc=$?" >> gpurun_out/r1e_bench.err
