#!/bin/bash
# SASS of the kernels in build/$1.cu.o whose mangled name contains $2 (e.g. Lb0ELb0ELi1ELi2ELi4ELi2E)
OBJ=$(dirname "$0")/../paper_2412_09734_b200/build/$1.cu.o
for f in $(cuobjdump -sass "$OBJ" | grep "Function :" | awk '{print $3}' | grep -- "$2"); do
  cuobjdump -sass -fun "$f" "$OBJ" | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed 's@ */\* 0x.*@@'
done
