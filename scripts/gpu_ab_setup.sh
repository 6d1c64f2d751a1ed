#!/bin/bash
# A/B of the C2 create and step across libraries (ab/*.so), plus a launch list of the setup kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for lib in "$@"; do MPAX_LIB=$PWD/$lib python scripts/create_time.py 2>&1 | tail -1; done; done
for lib in "$@"; do MPAX_LIB=$PWD/$lib C2_REPS=3 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:setup \
  --csv python scripts/c2_time.py 2>/dev/null | grep -E '"setup' | tail -2; done
