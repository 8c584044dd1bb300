#!/bin/bash
# Build an A/B variant of the library from a modified spmv.cu:
#   scripts/ab_build.sh NAME path/to/spmv_variant.cu
# -> build/ab_NAME/paper_2303_05098_b200 (package copy whose lib uses the variant);
#    run with AB_ROOT=build/ab_NAME python scripts/ab_spmv.py ...
set -e
name=$1; src=$2
out=build/ab_$name
rm -rf $out; mkdir -p $out
cp -r paper_2303_05098_b200 $out/
rm -rf $out/paper_2303_05098_b200/lib/obj
mkdir -p $out/obj
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Iinclude \
  -Ipaper_2303_05098_b200/csrc --expt-relaxed-constexpr -c $src -o $out/obj/spmv.o
objs=$(ls paper_2303_05098_b200/lib/obj/*.o | grep -v '/spmv.o' | grep -v '/cpp_')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/paper_2303_05098_b200/lib/libsparseoracle_b200.so $objs $out/obj/spmv.o
echo built $out
