#!/bin/bash
# decode path: parity tests + the measured 7B decode line
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_coop_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/decode_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/decode_tests.log)"
grep -E "Error|assert|FAILED" gpurun_out/decode_tests.log | head -20
timeout 300 python - <<'PY' 2>&1 | tail -5
import json, torch
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.calibrate import measure_decode
for arch in (S.LLAMA2_7B,):
    d = measure_decode(arch)
    wb = arch.total_bytes() - arch.embed_bytes()
    print(json.dumps({"arch": arch.name, "decode_ms": d, "b1_weight_GBps": wb / (d[1] / 1e3) / 1e9}))
PY
