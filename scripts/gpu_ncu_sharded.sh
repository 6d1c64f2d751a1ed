# one --set full capture of each sharded step kernel (C5, rows, 1 NCCL rank), read with ncu -i
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SG_AXIS=rows SG_K=2 timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_cols_spmv|k_rows_left|k_rows|k_cols" --launch-skip 8 --launch-count 8 \
  -o gpurun_out/r02j_sharded python scripts/prof_sharded.py > gpurun_out/r02j_ncu_sharded.log 2>&1
echo rc=$?
ncu -i gpurun_out/r02j_sharded.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/r02j_sharded_raw.csv 2>&1
echo rc=$?
