#!/bin/bash
# Build an A/B variant of libpmagraph_cuda.so with extra nvcc defines:
#   tools/build_variant.sh NAME -DFOO=1 ...   -> paper_1709_05061_b200/build/NAME.so
# (load it with GPMA_LIB=paper_1709_05061_b200/build/NAME.so)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_1709_05061_b200/build/var_$name
mkdir -p $out
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC -cudart static -Iinclude"
objs=""
for f in paper_1709_05061_b200/csrc/*.cu; do
  o=$out/$(basename $f).o
  /usr/local/cuda/bin/nvcc $FLAGS "$@" -c $f -o $o &
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static $objs -ldl -o paper_1709_05061_b200/build/$name.so
echo paper_1709_05061_b200/build/$name.so
