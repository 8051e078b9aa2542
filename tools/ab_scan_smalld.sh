#!/bin/bash
# Small-D diag row scan: parity suites, then throughput at D = 1, 2, 4 (8, 18 unaffected).
timeout 600 python -m pytest tests/test_pscan_api.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for D in 1 2 4 8 18; do python tools/probe_scan.py --T 33554432 --D $D --reps 8; done
python tools/probe_scan.py --T 1000003 --D 2 --reps 8
