#!/bin/bash
# Plain diag row scan: rows per thread x CTAs per SM with the balanced partition
# (variant libraries from tools/build_scan_variants.sh).
for v in kr16_m3 kr20_m2 kr24_m2 kr28_m2 kr32_m2; do
  L=tools/_build/variants/$v/libchainscan_b200.so
  for T in 4194304 16777216; do
    echo "$v $(CS_LIB_PATH=$L python tools/probe_scan.py --T $T --D 18 --reps 10)"
  done
  echo "$v $(CS_LIB_PATH=$L python tools/probe_scan.py --T 33554432 --D 2 --reps 8)"
done
