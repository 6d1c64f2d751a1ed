#!/bin/bash
# Run the GPU tests (optionally those matching the pattern in $1) and smoke() on the GPU box;
# logs, and the per-test parity counts (MPAX_PARITY_LOG), go under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/parity_counts.jsonl
MPAX_PARITY_LOG=$PWD/gpurun_out/parity_counts.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 900 \
  -p no:cacheprovider ${1:+-k "$1"} -rs > gpurun_out/gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
