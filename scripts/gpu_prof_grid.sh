#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/micro/barrier_bench > gpurun_out/barrier.log 2>&1
python scripts/prof_grid.py > gpurun_out/prof_grid_plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:grid_kernel -c 1 -o gpurun_out/prof_grid python scripts/prof_grid.py > gpurun_out/ncu_grid.log 2>&1
echo done
