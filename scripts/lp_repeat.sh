#!/bin/bash
# live pair (7B, NVLink hop) repeated: run-to-run spread of the ZigZag latency
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for rep in 1 2 3 4; do
  BZ_MODE=nvlink timeout 200 $R2 --master-port $((30600+rep)) scripts/live_pair.py > gpurun_out/lpr_$rep.log 2>&1
  echo "rep=$rep: $(grep -o '"avg_latency_ms": {[^}]*' gpurun_out/lpr_$rep.log | cut -c1-200)"
done
