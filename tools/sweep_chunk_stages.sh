#!/bin/bash
# Row-scan chunk length (stages per chunk, CS_SCAN_CHUNK_STAGES) with the balanced partition.
for cs in 48 64 96 128 192 256; do
  echo "cs=$cs $(CS_SCAN_CHUNK_STAGES=$cs python tools/probe_scan.py --T 16777216 --D 18 --reps 10)"
done
for cs in 48 64 96 128; do
  echo "cs=$cs $(CS_SCAN_CHUNK_STAGES=$cs python tools/probe_scan.py --mode block --T 16777216 --D 18 --reps 6)"
  echo "cs=$cs $(CS_SCAN_CHUNK_STAGES=$cs python tools/probe_scan.py --T 16777216 --D 64 --reps 6)"
  echo "cs=$cs $(CS_SCAN_CHUNK_STAGES=$cs python tools/probe_scan.py --T 16777216 --D 18 --dtype f64 --reps 6)"
done
