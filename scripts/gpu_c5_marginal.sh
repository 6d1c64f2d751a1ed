#!/bin/bash
# Marginal DRAM traffic per attempt of the C5 grid kernel: two launches limited to K = 16 and 32
# accepted steps (same init, check and output), so (T32 - T16) / (att32 - att16) excludes them.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none"
for prec in fp64 fp32; do
  for K in 16 32; do
    PROF_PREC=$prec PROF_M=5000000 PROF_K=$K ncu $M -k regex:grid_kernel -s 1 -c 1 --csv \
      python scripts/prof_grid.py > gpurun_out/c5m_${prec}_$K.csv 2>&1
  done
done
