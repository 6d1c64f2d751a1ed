#!/bin/bash
# C5 per-phase timings (trace library) in fp64 and fp32 storage (fp32 also with the forced
# column split), the cuSPARSE SpMV-pair yardstick, and a short bench that exercises every leg.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-f32}
MPAX_LIB=$PWD/paper_2412_09734_b200/libmpax_b200_trace.so C5_REPS=2 C5_PREC=fp64,fp32 C5_LIMIT=256 \
  timeout 600 python scripts/c5_run.py > gpurun_out/${T}_trace.log 2>&1
MPAX_GRID_SPLIT=1 MPAX_LIB=$PWD/paper_2412_09734_b200/libmpax_b200_trace.so C5_REPS=2 C5_PREC=fp32 C5_LIMIT=256 \
  timeout 600 python scripts/c5_run.py > gpurun_out/${T}_trace_split.log 2>&1
timeout 300 python scripts/c5_yard.py > gpurun_out/${T}_yard.json 2> gpurun_out/${T}_yard.err
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-spo --secondary-steps 1 \
  > gpurun_out/${T}_bench_short.json 2> gpurun_out/${T}_bench_short.err
echo "bench rc=$?" >> gpurun_out/${T}_bench_short.err
