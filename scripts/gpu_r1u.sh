#!/bin/bash
# C4: 1 vs 2 CTAs per SM (trace build).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so
PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/u_c4_minb2.log 2>&1
MPAX_GRID_MINB=1 PROF_K=256 timeout 300 python scripts/prof_grid.py > gpurun_out/u_c4_minb1.log 2>&1
PROF_K=256 PROF_ALG=r2 timeout 300 python scripts/prof_grid.py > gpurun_out/u_c4_minb2_r2.log 2>&1
MPAX_GRID_MINB=1 PROF_K=256 PROF_ALG=r2 timeout 300 python scripts/prof_grid.py > gpurun_out/u_c4_minb1_r2.log 2>&1
