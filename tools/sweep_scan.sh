timeout 600 python -m pytest tests -m gpu -x -q -k "blr or dense" 2>&1 | tail -3
timeout 900 python tools/bench_configs.py 3d 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/cfg3d_launches_v4.csv python tools/bench_configs.py 3d > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/cfg3d_launches_v4.csv > gpurun_out/cfg3d_v4_summary.txt
