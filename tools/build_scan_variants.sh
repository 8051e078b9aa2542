#!/bin/bash
# Build variant libraries that differ only in the row-scan compile-time tuning
# (tools/_build/variants/<name>/libchainscan_b200.so; select with CS_LIB_PATH).
set -e
cd "$(dirname "$0")/.."
B=paper_2508_18413_b200/_build
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
OBJS=$(ls $B/*.o | grep -v cs_scan.o)
build() {
  name=$1; shift
  d=tools/_build/variants/$name; mkdir -p $d
  $NVCC $FL "$@" -c paper_2508_18413_b200/csrc/cs_scan.cu -o $d/cs_scan.o
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $d/libchainscan_b200.so $OBJS $d/cs_scan.o -cudart static -lcublas -Xlinker -rpath=/usr/local/cuda/lib64
  echo built $name
}
build kr16_m3 -DCS_ROWS_DIAG_KR=16 -DCS_ROWS_DIAG_MINB=3 &
build kr20_m2 -DCS_ROWS_DIAG_KR=20 -DCS_ROWS_DIAG_MINB=2 &
build kr24_m2 -DCS_ROWS_DIAG_KR=24 -DCS_ROWS_DIAG_MINB=2 &
build kr28_m2 -DCS_ROWS_DIAG_KR=28 -DCS_ROWS_DIAG_MINB=2 &
build kr32_m2 -DCS_ROWS_DIAG_KR=32 -DCS_ROWS_DIAG_MINB=2 &
wait
