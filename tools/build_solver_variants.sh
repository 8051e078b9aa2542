#!/bin/bash
# Variant libraries differing only in the fused solver's occupancy target for the
# headline system (HMC Rosenbrock; tools/_build/variants/solve_m<N>/; select
# with CS_LIB_PATH).
set -e
cd "$(dirname "$0")/.."
B=paper_2508_18413_b200/_build
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
OBJS=$(ls $B/*.o | grep -v gen_hmc_rosen.o)
build() {
  name=$1; shift
  d=tools/_build/variants/$name; mkdir -p $d
  $NVCC $FL "$@" -Xptxas -v -c paper_2508_18413_b200/csrc/gen_hmc_rosen.cu -o $d/gen_hmc_rosen.o 2> $d/ptxas.txt
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $d/libchainscan_b200.so $OBJS $d/gen_hmc_rosen.o -cudart static -lcublas -Xlinker -rpath=/usr/local/cuda/lib64
  echo built $name
}
build solve_m2 -DCS_SOLVE_MIN_BLOCKS=2 &
build solve_m3 -DCS_SOLVE_MIN_BLOCKS=3 &
build solve_m4 -DCS_SOLVE_MIN_BLOCKS=4 &
wait
