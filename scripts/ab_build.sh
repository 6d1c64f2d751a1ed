#!/bin/bash
# Build the library of git revision $1 into ab/$2.so (A/B timing with MPAX_LIB=ab/$2.so; ab/ is
# git-ignored but travels to the GPU box with gpurun).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REV=$1; NAME=$2
WT=/tmp/ab_wt_$NAME
rm -rf $WT
git -C $ROOT worktree add -f --detach $WT $REV >/dev/null 2>&1
(cd $WT && python -c "import sys; sys.path.insert(0,'.'); from paper_2412_09734_b200 import _build; _build.build(force=True)")
mkdir -p $ROOT/ab
cp $WT/paper_2412_09734_b200/libmpax_b200.so $ROOT/ab/$NAME.so
git -C $ROOT worktree remove --force $WT
echo "ab/$NAME.so"
