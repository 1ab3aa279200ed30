# fused small-batch decode: GPU tests, then step times fused vs per-block kernels, then a phase trace
timeout 900 python -m pytest tests/test_decode_fused_gpu.py tests/test_decode_gpu.py tests/test_coop_gpu.py -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_fused.log
for b in 1 2; do
  echo -n "fused "; timeout 300 python scripts/decode_breakdown.py $b
  echo -n "per-block "; BZ_DECODE_FUSED=0 timeout 300 python scripts/decode_breakdown.py $b
done 2>&1 | tee gpurun_out/fused_bd.log
timeout 300 python scripts/fused_trace.py 1 2>&1 | tee gpurun_out/fused_trace.log
