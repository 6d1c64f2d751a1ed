#!/bin/bash
# Profiling pass (one ncu session per call): plain runs first, then the launch list of a
# short bench and full captures of the three solver kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary-steps 1 --no-c5"
$BENCH > gpurun_out/prof_plain.log 2>&1 || { echo "plain bench failed"; exit 1; }
python scripts/prof_grid.py > gpurun_out/prof_grid_plain.log 2>&1 || { echo "plain grid failed"; exit 1; }
C3_PATHS=3 python scripts/c3_bench.py > gpurun_out/prof_c3_plain.log 2>&1 || { echo "plain c3 failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $BENCH > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 2 -c 1 -o gpurun_out/prof_tiny $BENCH > gpurun_out/ncu_tiny.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:grid_kernel -c 1 -o gpurun_out/prof_grid python scripts/prof_grid.py > gpurun_out/ncu_grid.log 2>&1
C3_PATHS=3 ncu --set full --clock-control none --import-source on -k regex:dmma_kernel -c 1 -o gpurun_out/prof_dmma python scripts/c3_bench.py > gpurun_out/ncu_dmma.log 2>&1
PROF_M=5000000 PROF_K=16 python scripts/prof_grid.py > gpurun_out/prof_grid_c5_plain.log 2>&1 && \
  PROF_M=5000000 PROF_K=16 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 1 -c 1 \
  -o gpurun_out/prof_grid_c5 python scripts/prof_grid.py > gpurun_out/ncu_grid_c5.log 2>&1
echo done
