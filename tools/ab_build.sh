#!/bin/bash
# Build an A/B variant of liblz.so with one CUDA source replaced by a git revision or a file:
#   tools/ab_build.sh <name> <git-rev | path/to/file.cu> [source-name, default gemm.cu]
# -> build/ab/liblz_<name>.so ; select it with LZ_LIB_PATH=build/ab/liblz_<name>.so
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; which=${3:-gemm.cu}
mkdir -p build/ab
if [ -f "$src" ]; then cp "$src" build/ab/${which%.cu}_$name.cu
else git show "$src":paper_2407_04656_b200/csrc/$which > build/ab/${which%.cu}_$name.cu; fi
python -m paper_2407_04656_b200.build > /dev/null
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -Ipaper_2407_04656_b200/csrc"
nvcc $F -c build/ab/${which%.cu}_$name.cu -o build/ab/${which%.cu}_$name.o
objs=$(ls build/lz/*.o | grep -v "/${which%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/liblz_$name.so $objs build/ab/${which%.cu}_$name.o -lcudart_static -ldl -lrt -lpthread
echo build/ab/liblz_$name.so
