for sl in 2 3 4; do for kb in 16384 32768 65536; do
echo "slots=$sl kb=$kb"; CS_SCAN_SLOTS=$sl CS_SCAN_ROUND_KB=$kb timeout 60 python tools/probe_scan.py --mode diag --D 18 --T 4194304
done; done
timeout 300 python -m pytest tests -m gpu -x -q -k "scan or deer" 2>&1 | tail -2
