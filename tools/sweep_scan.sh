timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in 64 128 256; do CS_DENSE_CHUNK=$c timeout 120 python tools/probe_scan.py --mode dense --D 100 --T 100000 --reps 3; done
timeout 120 python tools/probe_scan.py --mode dense --D 100 --T 100000 --reps 3 --dtype f64
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dense -c 6 python tools/probe_scan.py --mode dense --D 100 --T 100000 --reps 1 2>&1 | grep -E "k_dense|gpu__time"
