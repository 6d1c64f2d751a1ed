#!/bin/bash
# quick timing of the grid path on C4 (and optionally a bench run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PROF_SHARDED=1 PROF_K=256 python scripts/prof_grid.py > gpurun_out/quick_grid.log 2>&1
PROF_K=256 PROF_ALG=r2 python scripts/prof_grid.py >> gpurun_out/quick_grid.log 2>&1
echo "--- MINB=1" >> gpurun_out/quick_grid.log
MPAX_GRID_MINB=1 PROF_K=256 python scripts/prof_grid.py >> gpurun_out/quick_grid.log 2>&1
echo "--- C5-like 1e6 x 2e6" >> gpurun_out/quick_grid.log
PROF_SHARDED=1 PROF_M=1000000 PROF_K=128 python scripts/prof_grid.py >> gpurun_out/quick_grid.log 2>&1
MPAX_GRID_MINB=1 PROF_M=1000000 PROF_K=128 python scripts/prof_grid.py >> gpurun_out/quick_grid.log 2>&1
if [ -n "$BENCH" ]; then timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.log 2>&1; fi
if [ -n "$TESTS" ]; then bash scripts/gpu_tests.sh "$TESTS"; fi
echo done
