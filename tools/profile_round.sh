#!/bin/bash
# Round-2 evidence under profiles/: launch list of the bench step, ncu --set full
# of the headline solver, the row scan at T=2^24 and the fused BLR builder.
set -x
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_bench.csv \
    python bench.py --steps 3 --warmup 2 --no-extras > gpurun_out/prof/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:deer_persistent -s 3 -c 1 -o gpurun_out/prof/solver \
    python tools/one_solve.py 2 > gpurun_out/prof/ncu_solver.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:scan_rows -s 3 -c 1 -o gpurun_out/prof/scan \
    python tools/scan_sweep.py diag > gpurun_out/prof/ncu_scan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_blr_fused -c 1 -o gpurun_out/prof/blr \
    python tools/one_blr.py 40000 f64 > gpurun_out/prof/ncu_blr.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/prof/launches_cfg3.csv python tools/one_blr.py 100000 f64 > gpurun_out/prof/ncu_cfg3.log 2>&1
