#!/bin/bash
# Build a variant of libsrj.so with extra -D flags on one source (A/B tuning):
#   tools/variant.sh NAME srj_tbs.cu -DSRJ_TBS_ILP8=false
# Links build/release/*.o (run build() first) with the variant object into
# paper_2011_06636_b200/libsrj_NAME.so; select it with SRJ_LIBRARY=<path>.
set -eu
name=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/build/variants"
obj="$root/build/variants/${name}_${src%.cu}.o"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v -Xcompiler -fPIC \
    "$@" -c -o "$obj" "$root/paper_2011_06636_b200/csrc/$src" 2>&1 | grep -E "error|spill" | sort | uniq -c || true
others=$(ls "$root"/build/release/*.o | grep -v "/${src%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/paper_2011_06636_b200/libsrj_${name}.so" $others "$obj" -ldl
echo "built libsrj_${name}.so"
