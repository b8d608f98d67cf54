#!/bin/bash
# Dev A/B: build libltlgrid_gpu.so with extra nvcc -D flags into
# paper_1810_02612_b200/_lib/var_<name>/ (load it with LTLG_DEV_SO=<path>).
#   tools/build_variant.sh u6b5 -DWM1_U=6 -DWM1_MINB=5
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1810_02612_b200/csrc; L=$ROOT/paper_1810_02612_b200/_lib; O=$L/var_$name
mkdir -p $O
SRC=${SRC:-$C/kernels.cu}  # (SRC=<file>: another kernels.cu, e.g. git show HEAD:... > /tmp/k.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --fmad=false -Xptxas -v \
    -I$C -I$ROOT/include "$@" -c $SRC -o $O/kernels.o 2> $O/ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $O/libltlgrid_gpu.so $O/kernels.o $L/sweep.o $L/tc_i8.o \
    $L/api.o $L/loader.o -lcudart_static -ldl -lpthread -lrt
grep -A3 "Compiling entry function .*label_wm1_kernelImLi2" $O/ptxas.log | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | tr "\n" " "; echo " -> $O"
