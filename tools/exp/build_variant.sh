#!/bin/bash
# build_variant.sh NAME "-DFOO=1 ..." : library variant into tools/exp/libNAME.so (git-ignored)
set -e
name=$1; shift
mkdir -p build/var_$name
for f in paper_2512_24449_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $f -o build/var_$name/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/exp/lib$name.so build/var_$name/*.o -lcudart
