#!/bin/bash
# Build libantkv_b200.so with extra -D flags into $1 (experiments; select it
# at run time with ANTKV_LIB=$1/libantkv_b200.so).  Usage: build_variant.sh DIR -DFOO ...
set -e
out=$1; shift
cd "$(dirname "$0")/../paper_2506_19505_b200/csrc"
mkdir -p "$out/obj"
for f in runtime prefill prefill_mma prefill_tc select cache encode_mma encode_tc encode_tc5 decode decode_fast decode_tc decode_mha kmeans evaluate; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c $f.cu -o "$out/obj/$f.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libantkv_b200.so" "$out"/obj/*.o -cudart static
