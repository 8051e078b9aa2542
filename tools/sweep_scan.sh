for i in 1 2 3; do timeout 900 python tools/bench_configs.py 3d 2>&1 | tail -1 | cut -c1-110; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
