#!/bin/bash
# Sweep the opt-in look-back-warp row scan (CS_SCAN_LBW=1) against the default
# chained-chunk scan at SURVEY 8d's large synthetic (diag fp32, T=2^24, D=18).
T=${T:-16777216}
echo "default: $(python tools/probe_scan.py --T $T --D 18 --reps 8)"
for kb in 16384 32768 49152 65536; do
  for lag in 1 2 3; do
    echo "LBW round_kb=$kb lag=$lag: $(CS_SCAN_LBW=1 CS_SCAN_ROUND_KB=$kb CS_SCAN_LAG=$lag python tools/probe_scan.py --T $T --D 18 --reps 8)"
  done
done
