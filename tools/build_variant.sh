#!/bin/bash
# Experiment build: recompile one unit (default the fp32 r=1 2D K1) with extra
# nvcc flags and link a separate library build/var_<name>/libso2dr_b200.so
# (load it with SO2DR_LIB=...).
# Usage: bash tools/build_variant.sh <name> "<nvcc flags>" [unit, e.g. k1_3d]
set -e
cd "$(dirname "$0")/.."
make -s -j8 >/dev/null
NAME=$1; FLAGS=$2; UNIT=${3:-k1_2d_f32_r1}
D=build/var_$NAME; mkdir -p $D
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++20 -ccbin /usr/bin/g++ -Xcompiler -fPIC -Iinclude -Ipaper_2309_08864_b200/csrc --expt-relaxed-constexpr"
$NV $FLAGS -c paper_2309_08864_b200/csrc/$UNIT.cu -o $D/$UNIT.o
OBJS=$(ls build/obj/*.o | grep -v "/$UNIT.o")
$NV -shared -o $D/libso2dr_b200.so $D/$UNIT.o $OBJS -L/usr/local/cuda/lib64 -L/usr/local/cuda/lib64/stubs -lcudart_static -ldl -lrt -lpthread
echo built $D/libso2dr_b200.so
