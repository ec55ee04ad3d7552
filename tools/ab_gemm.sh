#!/bin/bash
# Interleaved A/B of GEMM builds with a cooldown before every measurement (equal power state):
#   bash tools/ab_gemm.sh "<kinds>" <shape> <rounds> build/ab/liblz_a.so build/ab/liblz_b.so ...
kinds=$1; shape=$2; rounds=$3; shift 3
for i in $(seq 1 $rounds); do
  for lib in "$@"; do
    sleep 3
    LZ_LIB_PATH=$lib python tools/gemm_one.py --shape $shape --time --kinds $kinds 2>&1 | sed "s#^#$(basename $lib) #"
  done
done
