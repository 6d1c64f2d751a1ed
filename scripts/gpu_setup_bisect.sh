#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for st in 0 1 2 3 9; do echo "== stop $st"; MPAX_SETUP_STOP=$st MPAX_HOST_TRACE=1 python scripts/create_time.py 2>&1 | grep "create device" | tail -3; done
