# K-chunked decode GEMM (BZ_GEMM_KC=1, default) vs the stream-K skinny path (BZ_GEMM_KC=0)
for kc in 1 0; do echo "== KC=$kc"; BZ_GEMM_KC=$kc timeout 300 python scripts/skinny_bench.py 1 8 16; done 2>&1 | tee gpurun_out/kc_skinny.log
for b in 1 4 16; do
  for kc in 1 0; do echo -n "kc=$kc "; BZ_GEMM_KC=$kc timeout 300 python scripts/decode_breakdown.py $b; done
done 2>&1 | tee gpurun_out/kc_decode.log
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_decode_gpu.py tests/test_coop_gpu.py tests/test_decode_fused_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_kc.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" gpurun_out/pytest_kc.log | tail -15
