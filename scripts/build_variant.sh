#!/bin/bash
# A/B builds: recompile one fitness kernel source with extra -D flags and link
# a fitness-only library copy libhga_<name>.so next to libhga.so (selected at
# run time with HGA_LIB_VARIANT=<name>; symbols outside fitness are absent).  Usage: scripts/build_variant.sh NAME SOURCE "FLAGS"
set -e
name=$1; src=$2; flags=$3
D=paper_2208_14961_b200
mkdir -p $D/build/var_$name
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
$NV $flags -c $D/csrc/$src.cu -o $D/build/var_$name/$src.o
# only the fitness objects (keeps the copy small enough for the gpurun snapshot)
objs=$(ls $D/build/fitness.o $D/build/fitness_tc.o $D/build/fitness_tc2.o $D/build/fit_m*.o $D/build/probe.o | grep -v "/$src.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libhga_$name.so $objs $D/build/var_$name/$src.o -lcudart
echo built $D/libhga_$name.so
