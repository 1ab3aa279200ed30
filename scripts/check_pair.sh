#!/bin/bash
for bn in 128 192 256; do BZ_GEMM_PAIR=1 BZ_GEMM_BN=$bn timeout 120 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/gemm_pair_bn$bn.log 2>&1; echo "pair bn=$bn rc=$? $(tail -1 gpurun_out/gemm_pair_bn$bn.log)"; done
for pr in 0 1; do echo "== BZ_GEMM_PAIR=$pr"; BZ_GEMM_PAIR=$pr timeout 120 python scripts/gemm_bench.py 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=list(d)[0]; v=d[k]; print(f'{k:14s} {v[\"tflops\"]:7.1f} TF  cublas {v[\"cublas_tflops\"]:7.1f}  err {v[\"max_rel_err\"]:.1e}')
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])
"; done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
BZ_MODE=host timeout 150 $R --master-port 29952 scripts/live_pair.py > gpurun_out/lp_7b_host.log 2>&1; echo "7b host rc=$?"; grep '^{' gpurun_out/lp_7b_host.log | cut -c1-1200
