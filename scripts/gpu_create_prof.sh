#!/bin/bash
# Where the C2 create goes: host marks (MPAX_HOST_TRACE) and the device durations of its kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MPAX_HOST_TRACE=1 python scripts/create_time.py > gpurun_out/create_trace.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,launch__grid_size --clock-control none -c 40 --csv \
  python scripts/create_time.py > gpurun_out/create_ncu.csv 2>/dev/null
