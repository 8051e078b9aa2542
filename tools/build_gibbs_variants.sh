#!/bin/bash
# Variant libraries differing only in the Gibbs element kernel's occupancy
# target (tools/_build/variants/gibbs_m<N>/; select with CS_LIB_PATH).
set -e
cd "$(dirname "$0")/.."
B=paper_2508_18413_b200/_build
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
OBJS=$(ls $B/*.o | grep -v cs_gibbs.o)
build() {
  name=$1; shift
  d=tools/_build/variants/$name; mkdir -p $d
  $NVCC $FL "$@" -Xptxas -v -c paper_2508_18413_b200/csrc/cs_gibbs.cu -o $d/cs_gibbs.o 2> $d/ptxas.txt
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $d/libchainscan_b200.so $OBJS $d/cs_gibbs.o -cudart static -Xlinker -rpath=/usr/local/cuda/lib64
  echo built $name
}
build gibbs_m3 -DCS_GIBBS_MINB=3 &
build gibbs_m4 -DCS_GIBBS_MINB=4 &
build gibbs_m5 -DCS_GIBBS_MINB=5 &
wait
