#!/bin/bash
# ncu full capture (source-level) of the C5 grid kernel, after a plain run exits 0.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PROF_M=5000000 PROF_K=16 timeout 600 python scripts/prof_grid.py > gpurun_out/prof_c5_plain.log 2>&1 || { echo "plain failed"; exit 1; }
PROF_M=5000000 PROF_K=16 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 1 -c 1 \
  -o gpurun_out/prof_grid_c5${1:+_$1} python scripts/prof_grid.py > gpurun_out/ncu_grid_c5.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_grid_c5.log
