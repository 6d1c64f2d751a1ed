#!/bin/bash
# GPU-box profiling pass: plain bench run, then the ncu launch list and one full
# capture of the per-instance kernel (only after the plain run exited 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --secondary-steps 1"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tiny_kernel|instance_kernel" -s 2 -c 1 -o gpurun_out/prof_instance $CMD > gpurun_out/ncu_full.log 2>&1
echo done
