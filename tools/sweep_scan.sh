timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dense_tc_launches.csv python tools/probe_scan.py --mode dense --D 100 --T 100000 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/dense_tc_launches.csv
CS_DENSE_TC=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dense_simt_launches.csv python tools/probe_scan.py --mode dense --D 100 --T 100000 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/dense_simt_launches.csv
