timeout 900 python -m pytest tests -m gpu -x -q -k "run_deer or engines or fused or smoke or deer_api or gibbs or mala or hmc" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
cd tools && timeout 300 python probe_phases.py hmc 100000 | head -8 && cd ..
for i in 1 2; do timeout 300 python bench.py --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['value'])"; done
timeout 600 python tools/bench_configs.py 1 1r 2 2>&1 | grep config | cut -c1-120
