# bench + scan probes + one ncu capture of the 2^24 diag row scan
timeout 300 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench=$?
for m in diag block; do timeout 120 python tools/probe_scan.py --mode $m --T 4194304 --D 18 --reps 20 2>&1 | tail -1; done
timeout 120 python tools/probe_scan.py --mode diag --T 16777216 --D 18 --reps 20 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "scan" 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_rows -s 2 -c 1 -o gpurun_out/scan24 -f \
  python tools/probe_scan.py --mode diag --T 16777216 --D 18 --reps 2 > gpurun_out/ncu24.log 2>&1; echo ncu=$?
