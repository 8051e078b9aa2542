timeout 600 python -m pytest tests/test_pscan_api.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for T in 4194304 16777216; do
 for b in 0 1; do echo "bal=$b $(CS_SCAN_BALANCED=$b python tools/probe_scan.py --T $T --D 18 --reps 10)"; done
 for b in 0 1; do echo "bal=$b $(CS_SCAN_BALANCED=$b python tools/probe_scan.py --mode block --T $T --D 18 --reps 10)"; done
done
for b in 0 1; do echo "bal=$b $(CS_SCAN_BALANCED=$b python tools/probe_scan.py --T 1000000 --D 18 --reps 10)"; done
for b in 0 1; do echo "bal=$b $(CS_SCAN_BALANCED=$b python tools/probe_scan.py --T 4194304 --D 18 --dtype f64 --reps 10)"; done
