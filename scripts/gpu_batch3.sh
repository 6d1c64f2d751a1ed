#!/bin/bash
# Round-2 batch: new parity tests (decision log, skewed rows, sharded graph), the skew and
# sharded-graph timings (old library ab/cta2.so beside the current one), then the full GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MPAX_PARITY_LOG=$PWD/gpurun_out/parity_b3.jsonl
rm -f $MPAX_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_decision_log.py tests/test_gpu_grid.py tests/test_gpu_fp32.py \
  tests/test_gpu_sharded.py -q -m gpu -p no:cacheprovider > gpurun_out/b3_tests.log 2>&1
echo "rc=$?" >> gpurun_out/b3_tests.log
for l in ab/cta2.so paper_2412_09734_b200/libmpax_b200.so; do
  echo "== $l" >> gpurun_out/b3_skew.log
  MPAX_LIB=$PWD/$l timeout 600 python scripts/skew_time.py >> gpurun_out/b3_skew.log 2>&1
done
timeout 600 python scripts/sharded_graph_time.py > gpurun_out/b3_graph.log 2>&1
bash scripts/gpu_tests.sh
