#!/bin/bash
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29620 scripts/mgpu_check.py > gpurun_out/mgpu4.log 2>&1; echo "mgpu4 rc=$?"; grep -o '"case": "[a-z-]*", [^,]*, [^,]*, "ok": [a-z]*, "max_ms": [0-9.]*' gpurun_out/mgpu4.log
P=29630
for args in "--fanout nvls --nctas 32" "--fanout nvls --nctas 64" "--fanout nvls --nctas 16" "--fanout chain --nctas 32" "--fanout chain --nctas 64" "--no-group --nctas 48" "--fanout nvls --nctas 32 --tile-kib 512"; do
  P=$((P+1))
  timeout 200 $R --master-port $P bench.py --gpus 4 --steps 3 --warmup 2 --no-e2e --no-cpu --watchdog-s 180 $args > gpurun_out/sweep_$P.log 2>&1
  echo "$args -> $(grep -o '"value": [0-9.]*' gpurun_out/sweep_$P.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/sweep_$P.log | head -1) $(grep -o '"first_layer_ms": [0-9.]*' gpurun_out/sweep_$P.log | head -1)"
done
