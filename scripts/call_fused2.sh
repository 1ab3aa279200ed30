timeout 900 python -m pytest tests/test_decode_fused_gpu.py tests/test_decode_gpu.py tests/test_coop_gpu.py -q -rf -p no:cacheprovider --timeout 300 2>&1 | grep -E "^FAILED|passed|failed" | head -20
BZ_DECODE_FUSED=1 timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_coop_gpu.py tests/test_realclock_gpu.py -q -rf -p no:cacheprovider --timeout 300 2>&1 | grep -E "^FAILED|passed|failed" | head -20
for b in 1 2 4; do
  echo -n "fused "; BZ_DECODE_FUSED=1 timeout 300 python scripts/decode_breakdown.py $b
  echo -n "per-block "; timeout 300 python scripts/decode_breakdown.py $b
done 2>&1 | tee gpurun_out/fused_mma.log
BZ_DECODE_FUSED=1 timeout 300 python scripts/fused_trace.py 1 2>&1 | tee gpurun_out/fused_mma_trace.log | grep -v producer | head -20
BZ_DECODE_FUSED=1 timeout 300 python scripts/fused_trace.py 4 2>&1 | tee -a gpurun_out/fused_mma_trace.log | grep -v producer | head -20
