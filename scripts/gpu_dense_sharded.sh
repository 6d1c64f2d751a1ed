cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 --no-large --no-c5 --no-spo --no-cpu-baseline > gpurun_out/ds_bench.json 2> gpurun_out/ds_bench.err; echo bench rc=$?
for ax in rows cols; do
  SG_AXIS=$ax SG_K=16 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/r02h_sharded_${ax}_launches.csv python scripts/prof_sharded.py > gpurun_out/ps2_${ax}_ncu.log 2>&1
done
