#!/bin/bash
# div_rn_fast bitwise check, full GPU tests, C5 trace, bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 scripts/micro/div_check > gpurun_out/r1j_div.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r1j_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1j_tests.log
MPAX_LIB=$GRAFT_REPO_ROOT/paper_2412_09734_b200/libmpax_b200_trace.so timeout 600 python scripts/c5_run.py > gpurun_out/j_c5.log 2>&1
timeout 900 python bench.py > gpurun_out/r1j_bench.json 2> gpurun_out/r1j_bench.err
echo "bench rc=$?" >> gpurun_out/r1j_bench.err
