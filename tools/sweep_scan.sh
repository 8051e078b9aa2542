timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench=$?
timeout 900 python tools/bench_configs.py 1 1r 2 3 3d 4 5 2>&1 | grep config | cut -c1-170
