timeout 600 python -m pytest tests -m gpu -x -q -k "dense or blr" 2>&1 | tail -2
timeout 120 python tools/probe_scan.py --mode dense --D 100 --T 100000 --reps 3
timeout 900 python tools/bench_configs.py 3d 2>&1 | tail -1 | cut -c1-140
