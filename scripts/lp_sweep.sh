#!/bin/bash
# live pair (7B, NVLink hop) vs push engine / CTA budget, two repeats each
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=30500
for cfg in "vector 48" "vector 24" "vector 12" "ce 48"; do
  set -- $cfg
  for rep in 1 2; do
    port=$((port+1))
    BZ_MODE=nvlink BZ_ENGINE=$1 BZ_NCTAS=$2 timeout 200 $R2 --master-port $port scripts/live_pair.py > gpurun_out/lps_$1_$2_$rep.log 2>&1
    echo "$1 nctas=$2 rep=$rep: $(grep -o '"avg_latency_ms": {[^}]*' gpurun_out/lps_$1_$2_$rep.log | cut -c1-160) load=$(grep -o '"weights_load_ms": [0-9.]*' gpurun_out/lps_$1_$2_$rep.log)"
  done
done
