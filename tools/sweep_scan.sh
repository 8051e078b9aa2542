timeout 900 python -m pytest tests -m gpu -x -q -k "wide_short or leapfrog or wide or scan" 2>&1 | tail -3
timeout 600 python tools/bench_configs.py 4 2>&1 | tail -1 | cut -c1-160
