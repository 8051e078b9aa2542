timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for T in 4194304 16777216; do timeout 60 python tools/probe_scan.py --mode diag --D 18 --T $T; done
timeout 60 python tools/probe_scan.py --mode block --D 18 --T 4194304
timeout 60 python tools/probe_scan.py --mode diag --D 2 --T 16777216
timeout 600 python tools/bench_configs.py 5 2>&1 | tail -1 | cut -c1-120
timeout 600 python tools/bench_configs.py 2 2>&1 | tail -1 | cut -c1-120
