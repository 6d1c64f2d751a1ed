mkdir -p gpurun_out
for ax in rows cols; do
  SG_AXIS=$ax SG_K=64 timeout 600 python scripts/prof_sharded.py > gpurun_out/ps_$ax.log 2>&1
  SG_AXIS=$ax SG_K=16 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/ps_${ax}_launches.csv python scripts/prof_sharded.py > gpurun_out/ps_${ax}_ncu.log 2>&1
done
