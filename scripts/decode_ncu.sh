#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for b in 1 64; do python scripts/decode_probe.py $b; BZ_PDL=0 python scripts/decode_probe.py $b; done
for b in 1 64; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 60 --csv --log-file gpurun_out/decode_launch_b$b.csv python scripts/decode_probe.py $b > /dev/null 2>&1
done
echo done
