cd $GRAFT_REPO_ROOT
bash scripts/gpu_tests.sh
tail -3 gpurun_out/gputests.log; tail -4 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err; echo bench rc=$?
tail -c 600 gpurun_out/r02l_bench.json
