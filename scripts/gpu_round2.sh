#!/bin/bash
# Round-2 evidence pass on one GPU, in two parts so that each call's gpurun_out/ stays under the
# 64 MiB copy-back limit.  PART=A: the default bench line, the ncu launch list of a short bench,
# full captures of the C2 register kernel and the C4 grid kernel.  PART=B: full captures of the
# C5 grid kernel (fp64 and fp32 storage) and the C3 DMMA kernel.  Every capture runs only after
# its plain run exits 0.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r02}
NCU="ncu --set full --clock-control none --import-source on"
if [ "${PART:-A}" = "A" ]; then
  timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
  echo "bench rc=$?" >> gpurun_out/${T}_bench.err
  SHORT="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary-steps 1 --no-c5 --no-spo"
  $SHORT > gpurun_out/${T}_short.json 2>&1 || echo "short bench failed" >> gpurun_out/${T}_bench.err
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${T}_launches.csv \
    $SHORT > gpurun_out/${T}_ncu_launches.log 2>&1
  C2_REPS=2 $NCU -k regex:tiny_kernel -s 3 -c 1 -o gpurun_out/${T}_tiny python scripts/c2_time.py \
    > gpurun_out/${T}_ncu_tiny.log 2>&1
  PROF_K=64 python scripts/prof_grid.py > gpurun_out/${T}_c4_plain.log 2>&1 && \
    PROF_K=64 $NCU -k regex:grid_kernel -s 1 -c 1 -o gpurun_out/${T}_grid_c4 python scripts/prof_grid.py \
    > gpurun_out/${T}_ncu_c4.log 2>&1
else
  PROF_M=5000000 PROF_K=16 python scripts/prof_grid.py > gpurun_out/${T}_c5_plain.log 2>&1 && \
    PROF_M=5000000 PROF_K=16 $NCU -k regex:grid_kernel -s 1 -c 1 -o gpurun_out/${T}_grid_c5 python scripts/prof_grid.py \
    > gpurun_out/${T}_ncu_c5.log 2>&1
  PROF_PREC=fp32 PROF_M=5000000 PROF_K=16 python scripts/prof_grid.py > gpurun_out/${T}_c5f_plain.log 2>&1 && \
    PROF_PREC=fp32 PROF_M=5000000 PROF_K=16 $NCU -k regex:grid_kernel -s 1 -c 1 -o gpurun_out/${T}_grid_c5f \
    python scripts/prof_grid.py > gpurun_out/${T}_ncu_c5f.log 2>&1
  C3_PATHS=3 python scripts/c3_bench.py > gpurun_out/${T}_c3_plain.log 2>&1 && \
    C3_PATHS=3 $NCU -k regex:dmma_kernel -c 1 -o gpurun_out/${T}_dmma python scripts/c3_bench.py \
    > gpurun_out/${T}_ncu_dmma.log 2>&1
fi
echo done
