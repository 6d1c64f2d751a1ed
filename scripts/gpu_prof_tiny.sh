#!/bin/bash
# ncu source-level capture of the C2 register kernel (after a plain run exits 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C2_REPS=20 python scripts/c2_time.py > gpurun_out/prof_tiny_plain.log 2>&1 || { echo "plain failed"; exit 1; }
C2_REPS=2 ncu --set full --clock-control none --import-source on -k regex:tiny_kernel -s 3 -c 1 \
  -o gpurun_out/prof_tiny${1:+_$1} python scripts/c2_time.py > gpurun_out/ncu_tiny.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_tiny.log
