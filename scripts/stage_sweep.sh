#!/bin/bash
# N=1 host-cache staging variants (copy-engine chunk size, zero-copy kernel)
for args in "--tiles-per-copy 8" "--tiles-per-copy 32" "--tiles-per-copy 128" "--stage-engine sm --nctas 16" "--stage-engine sm --nctas 48" "--tile-kib 4096 --tiles-per-copy 8"; do
  timeout 200 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-c3 --no-coop --watchdog-s 180 $args > gpurun_out/stage.log 2>&1
  echo "$args -> $(grep -o '"value": [0-9.]*' gpurun_out/stage.log | head -1) first_layer $(grep -o '"first_layer_ms": [0-9.]*' gpurun_out/stage.log | head -1)"
done
python scripts/profile_single.py gemm > gpurun_out/prof_gemm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16 -s 1 -c 2 -o gpurun_out/prof_gemm_pair \
    python scripts/profile_single.py gemm > gpurun_out/ncu_gemm_pair.log 2>&1
echo "gemm pair ncu rc=$?"
