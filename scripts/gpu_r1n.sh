#!/bin/bash
# C4 phase-A mapping: trace default (G lanes for few column tiles) vs the tile mapping; grid tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/n_c4_default.log 2>&1
MPAX_GRID_GT=1 PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/n_c4_tile.log 2>&1
PROF_K=256 PROF_ALG=r2 timeout 300 python scripts/prof_grid.py > gpurun_out/n_c4_default_r2.log 2>&1
MPAX_GRID_GT=1 PROF_K=256 PROF_ALG=r2 timeout 300 python scripts/prof_grid.py > gpurun_out/n_c4_tile_r2.log 2>&1
unset MPAX_LIB
timeout 900 python -m pytest tests/test_gpu_grid.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1n_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1n_tests.log
