timeout 600 python -m pytest tests/test_attention_gpu.py -v -rs -p no:cacheprovider --timeout 60 -o timeout_method=thread > gpurun_out/pytest_attn12.log 2>&1; echo "pytest rc=$?"
grep -E "PASSED|FAILED|Timeout|passed|failed" gpurun_out/pytest_attn12.log | head -10
if grep -q "6 passed" gpurun_out/pytest_attn12.log; then
timeout 300 python scripts/attn_bench.py > gpurun_out/attn_bench12.jsonl 2> gpurun_out/attn_bench12.err; echo "bench rc=$?"
cat gpurun_out/attn_bench12.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flash_prefill -s 3 -c 1 -o gpurun_out/prof_attn12 python scripts/attn_bench.py > gpurun_out/ncu_attn12.log 2>&1; echo "ncu rc=$?"
fi
