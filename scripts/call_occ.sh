# skinny GEMM with 1 vs 2 CTAs per SM: decode step times, then the GEMM/decode tests on each
for b in 1 4 16 64; do
  for occ in 1 2; do echo -n "occ=$occ "; BZ_GEMM_OCC=$occ timeout 300 python scripts/decode_breakdown.py $b; done
done 2>&1 | tee gpurun_out/occ.log
for occ in 1 2; do
  BZ_GEMM_OCC=$occ timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_decode_gpu.py tests/test_coop_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_occ$occ.log 2>&1; echo "occ=$occ rc=$?"; grep -E "passed|failed" gpurun_out/pytest_occ$occ.log
done
