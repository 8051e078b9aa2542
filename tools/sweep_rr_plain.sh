# plain diag scans: default selection vs reduce-then-replay across T (D = 18)
for T in 131072 262144 524288 1048576 2097152 4194304 16777216; do
  python tools/scan_sweep.py diag $T 18 | sed "s/^/dflt /"
  CS_SCAN_RR_PLAIN_MAX_T=1000000000 python tools/scan_sweep.py diag $T 18 | sed "s/^/rr   /"
done
