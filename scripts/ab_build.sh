#!/bin/bash
# Build an A/B variant of the library with one translation unit replaced:
#   scripts/ab_build.sh NAME path/to/variant.cu [OBJ=spmv] [extra nvcc flags...]
# -> build/ab_NAME/paper_2303_05098_b200 (package copy whose lib uses the variant);
#    run with AB_ROOT=build/ab_NAME python scripts/ab_spmv.py ...
set -e
name=$1; src=$2; obj=${3:-spmv}; shift 3 || shift $#
out=build/ab_$name
rm -rf $out; mkdir -p $out
cp -r paper_2303_05098_b200 $out/
rm -rf $out/paper_2303_05098_b200/lib/obj
mkdir -p $out/obj
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Iinclude \
  -Ipaper_2303_05098_b200/csrc --expt-relaxed-constexpr "$@" -c $src -o $out/obj/$obj.o
objs=$(ls paper_2303_05098_b200/lib/obj/*.o | grep -v "/$obj.o" | grep -v '/cpp_')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/paper_2303_05098_b200/lib/libsparseoracle_b200.so $objs $out/obj/$obj.o
echo built $out
