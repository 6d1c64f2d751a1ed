mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_polish.py tests/test_gpu_determinism.py tests/test_gpu_infeasibility.py tests/test_gpu_const_step.py tests/test_gpu_reflection.py -q -x > gpurun_out/shc_tests.log 2>&1; tail -3 gpurun_out/shc_tests.log
for ax in rows cols; do SG_AXIS=$ax SG_K=64 timeout 600 python scripts/prof_sharded.py 2>&1 | tail -1; done
SG_M=100000 timeout 600 python scripts/sharded_graph_time.py
