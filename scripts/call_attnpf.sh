# decode attention: K/V chunk prefetched into L2 before the grid dependency (rope_append triggers first)
for b in 1 4 16; do timeout 300 python scripts/decode_breakdown.py $b; done 2>&1 | tee gpurun_out/attnpf_decode.log
for c in 256 4096; do echo "ctx=$c"; done
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_coop_gpu.py tests/test_decode_fused_gpu.py tests/test_coop_7b_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_attnpf.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" gpurun_out/pytest_attnpf.log | tail -15
