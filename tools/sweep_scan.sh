# round-end check: GPU suite, smoke, bench, the BASELINE config table, bench launch list
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py > gpurun_out/bench12.json 2> gpurun_out/bench12.err; echo bench=$?
timeout 900 python tools/bench_configs.py 1 1r 2 3 3d 4 5 2>&1 | grep config | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01_final.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/ncu_final.log 2>&1; echo ncu=$?
