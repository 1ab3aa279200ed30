timeout 600 python -m pytest tests/test_attention_gpu.py -q -rs -s -p no:cacheprovider > gpurun_out/pytest_attn2.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|assert" gpurun_out/pytest_attn2.log | tail -8
timeout 300 python scripts/attn_bench.py > gpurun_out/attn_bench2.jsonl 2> gpurun_out/attn_bench2.err; echo "bench rc=$?"
cat gpurun_out/attn_bench2.jsonl; tail -3 gpurun_out/attn_bench2.err
