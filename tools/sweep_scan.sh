timeout 900 python -m pytest tests -m gpu -x -q -k "streamed or leapfrog or gibbs or blr or engines" 2>&1 | tail -2
timeout 600 python tools/bench_configs.py 4 5 3 2>&1 | grep config | cut -c1-140
