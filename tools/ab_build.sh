#!/bin/bash
# Build an A/B variant of liblz.so whose gemm.cu is taken from a git revision or file:
#   tools/ab_build.sh <name> <git-rev | path/to/gemm.cu>
# -> build/ab/liblz_<name>.so ; select it with LZ_LIB_PATH=build/ab/liblz_<name>.so
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2
mkdir -p build/ab
if [ -f "$src" ]; then cp "$src" build/ab/gemm_$name.cu
else git show "$src":paper_2407_04656_b200/csrc/gemm.cu > build/ab/gemm_$name.cu; fi
python -m paper_2407_04656_b200.build > /dev/null
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -Ipaper_2407_04656_b200/csrc"
nvcc $F -c build/ab/gemm_$name.cu -o build/ab/gemm_$name.o
objs=$(ls build/lz/*.o | grep -v gemm.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/liblz_$name.so $objs build/ab/gemm_$name.o -lcudart_static -ldl -lrt -lpthread
echo build/ab/liblz_$name.so
