#!/bin/bash
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 120 python -m pytest tests/test_dataplane_gpu.py -q -x > gpurun_out/dp.log 2>&1; echo "dataplane tests rc=$? $(tail -1 gpurun_out/dp.log)"
for e in vector ce; do timeout 150 $R4 --master-port 3040${#e} bench.py --gpus 4 --steps 3 --warmup 2 --no-e2e --no-cpu --no-c3 --no-coop --no-live --engine $e > gpurun_out/ce4_$e.log 2>&1; echo "n4 $e -> $(grep -o '"value": [0-9.]*' gpurun_out/ce4_$e.log | head -1) bit_exact $(grep -o '"bit_exact": [a-z]*' gpurun_out/ce4_$e.log | head -1)"; done
for e in vector ce; do BZ_MODE=nvlink BZ_ENGINE=$e timeout 150 $R2 --master-port 3041${#e} scripts/live_pair.py > gpurun_out/lpce_$e.log 2>&1; echo "live pair $e: $(grep -o 'avg_latency_ms[^}]*' gpurun_out/lpce_$e.log)"; done
