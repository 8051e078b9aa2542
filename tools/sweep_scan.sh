timeout 600 python -m pytest tests -m gpu -x -q -k "dense or blr or gram" 2>&1 | tail -2
timeout 900 python tools/bench_configs.py 3d 2>&1 | tail -1 | cut -c1-140
timeout 120 python tools/probe_scan.py --mode dense --D 100 --T 100000 --reps 3
timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_bd_final -c 1 python tools/bench_configs.py 3d 2>&1 | grep -E "duration|warps_active"
