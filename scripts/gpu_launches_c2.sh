#!/bin/bash
# Launch list (per-kernel durations) of a few C2 steps, after a plain run.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C2_REPS=5 python scripts/c2_time.py > gpurun_out/launch_plain.log 2>&1 || exit 1
C2_REPS=3 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \
  python scripts/c2_time.py > gpurun_out/c2_launches.log 2>&1
