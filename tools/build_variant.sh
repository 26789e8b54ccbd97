#!/bin/bash
# build a variant of libpvo_b200.so with extra nvcc defines: tools/build_variant.sh <name> -DFOO=1 ...
set -e
name=$1; shift
out=build/variants/$name; rm -rf $out; mkdir -p $out
for s in corr corr_tma ba ba_large measure dgraph features capi_core capi_window capi_provider capi_batch capi_dgraph; do
  extra=""; { [ $s = measure ] || [ $s = features ]; } && extra="--fmad=false"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC -I include $extra "$@" -c paper_2208_04726_b200/csrc/$s.cu -o $out/$s.o &
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I include -c paper_2208_04726_b200/csrc/graph.cpp -o $out/graph.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/lib_$name.so $out/*.o -lcudart_static -lrt -ldl -lpthread
echo tools/lib_$name.so
