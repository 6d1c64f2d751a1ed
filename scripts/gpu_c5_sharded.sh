set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5s_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/c5s_tests.log 2>&1; tail -3 gpurun_out/c5s_tests.log
for ax in rows cols; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-large --no-dense --no-spo --no-cpu-baseline --c5-sharded --c5-axis $ax > gpurun_out/c5s_$ax.json 2> gpurun_out/c5s_$ax.err; tail -2 gpurun_out/c5s_$ax.err
done
