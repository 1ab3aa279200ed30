#!/bin/bash
# 4-GPU parity + tuning sweep of the scale-up movers (run on the GPU box)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29520 scripts/mgpu_check.py > gpurun_out/mgpu4.log 2>&1; echo "mgpu4 rc=$?"
BZ_ARCH=llama2-7b BZ_TILE_KIB=1024 timeout 400 $R --master-port 29521 scripts/mgpu_check.py > gpurun_out/mgpu4_7b.log 2>&1; echo "mgpu4_7b rc=$?"
P=29530
for args in "--nctas 32" "--nctas 16" "--nctas 64" "--engine tma --nctas 32" "--engine tma --nctas 64" "--nctas 32 --tile-kib 4096" "--no-group --nctas 32" "--fanout chain --nctas 32"; do
  P=$((P+1))
  timeout 200 $R --master-port $P bench.py --gpus 4 --steps 3 --warmup 2 --no-e2e --no-cpu --watchdog-s 180 $args > gpurun_out/sweep_$P.log 2>&1
  echo "$args -> $(grep -o '"value": [0-9.]*' gpurun_out/sweep_$P.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/sweep_$P.log | head -1)"
done
