#!/bin/bash
# short-prompt prefill GEMMs (o, down at M = 256..512) under pinned schedules
for cfg in "" "BZ_GEMM_PAIR=0 BZ_GEMM_BN=128" "BZ_GEMM_PAIR=0 BZ_GEMM_BN=256" "BZ_GEMM_PAIR=0 BZ_GEMM_BN=192" \
           "BZ_GEMM_PAIR=1 BZ_GEMM_BN=128 BZ_GEMM_PAIR_SPLIT=1" "BZ_GEMM_PAIR=1 BZ_GEMM_BN=128 BZ_GEMM_PAIR_SPLIT=2" \
           "BZ_GEMM_PAIR=1 BZ_GEMM_BN=256 BZ_GEMM_NSUB=1 BZ_GEMM_PAIR_SPLIT=1" "BZ_GEMM_PAIR=1 BZ_GEMM_BN=256 BZ_GEMM_NSUB=1 BZ_GEMM_PAIR_SPLIT=2" \
           "BZ_GEMM_PAIR=1 BZ_GEMM_BN=256 BZ_GEMM_NSUB=1 BZ_GEMM_PAIR_SPLIT=3" "BZ_GEMM_PAIR=1 BZ_GEMM_BN=256 BZ_GEMM_NSUB=1 BZ_GEMM_PAIR_SPLIT=4" \
           "BZ_GEMM_PAIR=1 BZ_GEMM_BN=192 BZ_GEMM_NSUB=1 BZ_GEMM_PAIR_SPLIT=2" "BZ_GEMM_PAIR=1 BZ_GEMM_BN=128 BZ_GEMM_PAIR_SPLIT=4"; do
  echo "== ${cfg:-model}"
  env $cfg BZ_MS=256,384,512 python scripts/gemm_msweep.py 2>&1 | grep '^{' | grep -v '"qkv"\|gate_up' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"  m={d['m']} {d['shape']:5s} ctas {d['ctas']:4d} ours {d['ours_tf']:7.1f} cublas {d['cublas_tf']:7.1f} ratio {d['ratio']:.3f} err {d['err']:.1e}\")"
done
