#!/bin/bash
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29800
for args in "--fanout nvls --nctas 96" "--fanout nvls --nctas 128" "--fanout nvls --nctas 64 --tile-kib 4096" "--fanout star --nctas 64" "--fanout chain --nctas 96"; do
  P=$((P+1))
  timeout 200 $R --master-port $P bench.py --gpus 4 --steps 3 --warmup 2 --no-e2e --no-cpu --no-c3 --no-coop --watchdog-s 180 $args > gpurun_out/nv_$P.log 2>&1
  echo "$args -> $(grep -o '"value": [0-9.]*' gpurun_out/nv_$P.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/nv_$P.log | head -1)"
done
free -g | head -2
timeout 900 $R --master-port 29850 bench.py --gpus 4 --arch llama2-70b --tp 4 --steps 2 --warmup 1 --no-c3 --no-coop --cpu-sample-units 2 --watchdog-s 850 > gpurun_out/c5_70b_tp4.log 2>&1; echo "c5 rc=$?"; grep '^{' gpurun_out/c5_70b_tp4.log | cut -c1-900; grep "bench r0" gpurun_out/c5_70b_tp4.log | tail -5
