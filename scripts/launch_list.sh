#!/bin/bash
# launch list of the default N=1 bench command (after it exits 0 without ncu)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 1 > gpurun_out/ll_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench_n1.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ll_ncu.log 2>&1
echo "ncu rc=$?"
