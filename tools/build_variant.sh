#!/bin/bash
# Scratch: builds an instrumented copy of the library into build/<name>/libcqp_b200.so
#   tools/build_variant.sh trace -DCQP_TRACE
# Use it with CQP_B200_LIB=build/<name>/libcqp_b200.so (paper_2311_18056_b200/_lib.py).
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_2311_18056_b200/csrc
out=$root/build/$name
mkdir -p $out
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
pids=()
for f in cqp_single cqp_cluster cqp_capi cqp_setup cqp_batch; do
  if [ -n "$ONLY" ] && [[ " $ONLY " != *" $f "* ]] && [ -f $root/paper_2311_18056_b200/csrc/$f.o ]; then
    cp $src/$f.o $out/$f.o; continue
  fi
  $NVCC "$@" -std=c++17 -O3 -lineinfo $ARCH -Xcompiler -fPIC,-fvisibility=hidden -I$root/include -I$src -c $src/$f.cu -o $out/$f.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
$NVCC -shared $ARCH -o $out/libcqp_b200.so $out/*.o
echo built $out/libcqp_b200.so
