#!/bin/bash
# A/B variants of one source file: recompile csrc/$2.cu with extra -D flags and relink
# with the current build's other objects into ab/$1.so (experiments).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; SRC=$2; shift 2
B=$ROOT/paper_2412_09734_b200/build
NCCL=$(python -c "from paper_2412_09734_b200 import _build; i,l=_build._nccl_dirs(); print(i or '', l or '')")
NI=$(echo $NCCL | cut -d' ' -f1); NL=$(echo $NCCL | cut -d' ' -f2)
mkdir -p /tmp/abg_$NAME $ROOT/ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -fmad=true -prec-div=true -prec-sqrt=true -ftz=false -DMPAX_HAVE_NCCL=1 "$@" -I$ROOT/include \
  -I$ROOT/paper_2412_09734_b200/csrc -I$NI -c $ROOT/paper_2412_09734_b200/csrc/$SRC.cu -o /tmp/abg_$NAME/obj.o
objs=$(ls $B/*.o | grep -v "/$SRC.cu.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/ab/$NAME.so $objs /tmp/abg_$NAME/obj.o -lcudart \
  -L $NL -l:libnccl.so.2 -Xlinker -rpath=$NL
echo ab/$NAME.so
