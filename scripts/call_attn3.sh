timeout 900 python -m pytest tests/test_attention_gpu.py -v -rs -p no:cacheprovider --timeout 45 -o timeout_method=thread > gpurun_out/pytest_attn3.log 2>&1; echo "pytest rc=$?"
grep -E "PASSED|FAILED|Timeout|ERROR" gpurun_out/pytest_attn3.log | head -20
