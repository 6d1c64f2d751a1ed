#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over every kernel path (scripts/sanitize.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/sanitize.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain failed"; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
