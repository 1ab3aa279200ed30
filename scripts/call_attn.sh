timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_coop_gpu.py tests/test_coop_7b_gpu.py tests/test_decode_gpu.py -q -rs -s -p no:cacheprovider > gpurun_out/pytest_attn.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_attn.log | tail -3
timeout 300 python scripts/attn_bench.py > gpurun_out/attn_bench.jsonl 2> gpurun_out/attn_bench.err; echo "bench rc=$?"
cat gpurun_out/attn_bench.jsonl
timeout 300 python scripts/attn_bench.py > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flash_prefill -s 3 -c 1 -o gpurun_out/prof_attn python scripts/attn_bench.py > gpurun_out/ncu_attn.log 2>&1; echo "ncu rc=$?"
