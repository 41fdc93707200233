#!/bin/bash
# usage: mkvar.sh name src.cu "-DFLAGS"
set -e
cd /root/repo
name=$1; src=$2; flags=$3
d=build/var_$name; rm -rf $d; mkdir -p $d; cp build/obj/*.o $d/
base=$(basename $src .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills -I include $flags -c paper_2603_15603_b200/csrc/$src -o $d/$base.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_15603_b200/lib/libfsb_$name.so $d/*.o -lcuda
echo built $name
