#!/bin/bash
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=30100
for args in "--nctas 48" "--nctas 48 --tile-kib 2048" "--nctas 64 --tile-kib 4096" "--nctas 96 --tile-kib 2048" "--nctas 32 --tile-kib 512" "--nctas 48 --engine vec256 --tile-kib 2048"; do
  P=$((P+1))
  timeout 150 $R --master-port $P bench.py --gpus 2 --steps 4 --warmup 2 --no-e2e --no-cpu --no-c3 --no-coop --no-live --watchdog-s 140 $args > gpurun_out/s2_$P.log 2>&1
  echo "$args -> $(grep -o '"value": [0-9.]*' gpurun_out/s2_$P.log | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/s2_$P.log | head -1)"
done
s=$(date +%s); timeout 600 $R --master-port 30120 bench.py --gpus 2 > gpurun_out/def_n2.log 2>&1; echo "default n2 rc=$? $(( $(date +%s)-s ))s"
grep '^{' gpurun_out/def_n2.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['live_pair']['avg_latency_ms'] if d.get('live_pair') else None, d['roofline']['frac'])"
