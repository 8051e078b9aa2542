timeout 600 python -m pytest tests -m gpu -x -q -k "blr or dense or gram" 2>&1 | tail -3
timeout 900 python tools/bench_configs.py 3d 2>&1 | tail -1
CS_BLR_DENSE_TC=1 timeout 900 python tools/bench_configs.py 3d 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/cfg3d_launches_v5.csv python tools/bench_configs.py 3d > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/cfg3d_launches_v5.csv > gpurun_out/cfg3d_v5_summary.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bd_final -c 1 -o gpurun_out/prof_bd_final_umma -f python tools/bench_configs.py 3d10k > gpurun_out/ncu_bd2.log 2>&1; echo ncu=$?
