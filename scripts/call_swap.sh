# swapped-operand decode GEMM (BZ_GEMM_SWAP=1, default) vs previous paths; tests
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_swap_gemm.log 2>&1; echo "gemm tests rc=$?"; tail -5 gpurun_out/pytest_swap_gemm.log
for sw in 1 0; do echo "== SWAP=$sw"; BZ_GEMM_SWAP=$sw timeout 300 python scripts/skinny_bench.py 1 8 16 | cut -c1-100; done 2>&1 | tee gpurun_out/swap_skinny.log
for b in 1 4 16; do
  for sw in 1 0; do echo -n "swap=$sw "; BZ_GEMM_SWAP=$sw timeout 300 python scripts/decode_breakdown.py $b; done
done 2>&1 | tee gpurun_out/swap_decode.log
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_coop_gpu.py tests/test_decode_fused_gpu.py tests/test_coop_7b_gpu.py tests/test_attention_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_swap.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" gpurun_out/pytest_swap.log | tail -15
