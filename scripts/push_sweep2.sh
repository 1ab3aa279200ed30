#!/bin/bash
# 7B NVLink hop (N=2) vs push engine and CTA count: per-destination GB/s
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
X="--gpus 2 --no-e2e --no-c3 --no-coop --no-live --no-realclock --no-cpu --steps 5 --warmup 3"
port=29700
for cfg in "vector 48" "vector 64" "vector 96" "vec256 32" "vec256 48" "vec256 64" "vec256 96" "tma 48" "tma 96" "tma 148"; do
  set -- $cfg; port=$((port+1))
  timeout 200 $R --master-port $port bench.py $X --engine $1 --nctas $2 > gpurun_out/ps_$1_$2.log 2>&1
  echo "$1 nctas=$2 rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/ps_$1_$2.log | head -1) $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/ps_$1_$2.log | head -1)"
done
