#!/bin/bash
# build a variant of libgraphlb_b200.so with extra nvcc flags into _exp/<name>.so
name=$1; shift
out=_exp/$name; mkdir -p $out
for f in glb_memory glb_graph glb_driver glb_gen glb_peak; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 20054 "$@" -c paper_1711_00231_b200/csrc/$f.cu -o $out/$f.o &
done
wait
g++ -O3 -mavx2 -fPIC -std=c++17 -c paper_1711_00231_b200/csrc/glb_host_simd.cpp -o $out/glb_host_simd.o
g++ -O3 -fPIC -std=c++17 -c paper_1711_00231_b200/csrc/glb_io.cpp -o $out/glb_io.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o _exp/$name.so $out/*.o -lpthread
