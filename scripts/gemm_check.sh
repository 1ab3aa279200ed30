#!/bin/bash
for bn in 128 192 256; do BZ_GEMM_BN=$bn timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/gemm_bn$bn.log 2>&1; echo "bn=$bn tests rc=$? $(tail -1 gpurun_out/gemm_bn$bn.log)"; done
for bn in 0 128 192 256; do echo "== BZ_GEMM_BN=$bn"; BZ_GEMM_BN=$bn python scripts/gemm_bench.py 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=list(d)[0]; v=d[k]; print(f'{k:14s} {v[\"tflops\"]:7.1f} TF  cublas {v[\"cublas_tflops\"]:7.1f}  err {v[\"max_rel_err\"]:.1e}')
"; done
timeout 300 python -m pytest tests/test_coop_gpu.py -q -x > gpurun_out/coop.log 2>&1; echo "coop rc=$? $(tail -1 gpurun_out/coop.log)"
timeout 400 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_n1_coop.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench_n1_coop.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps(d['coop_c1'])); print(json.dumps(d['decisions']))"
