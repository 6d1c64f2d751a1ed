#!/bin/bash
# C5 grid kernel: trace timings at MINB=1/2, then one ncu --set full capture (source-level).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so MPAX_GRID_MINB=1 PROF_M=5000000 PROF_K=64 \
  timeout 300 python scripts/prof_grid.py > gpurun_out/p_c5_minb1.log 2>&1
MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so PROF_M=5000000 PROF_K=64 \
  timeout 300 python scripts/prof_grid.py > gpurun_out/p_c5_minb2.log 2>&1
PROF_M=5000000 PROF_K=16 timeout 300 python scripts/prof_grid.py > gpurun_out/p_c5_plain.log 2>&1 || exit 1
PROF_M=5000000 PROF_K=16 timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -c 1 \
  -o gpurun_out/p_c5_grid python scripts/prof_grid.py > gpurun_out/p_c5_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p_c5_ncu.log
