#!/bin/bash
# decode GEMMs (batch 1 and 8) under pinned skinny schedules: tile width x stream-K
for cfg in "" "BZ_GEMM_STREAMK=0" "BZ_GEMM_STREAMK=1" "BZ_GEMM_BN=32 BZ_GEMM_STREAMK=0" "BZ_GEMM_BN=64 BZ_GEMM_STREAMK=0" \
           "BZ_GEMM_BN=128 BZ_GEMM_STREAMK=0" "BZ_GEMM_BN=64 BZ_GEMM_STREAMK=1" "BZ_GEMM_BN=128 BZ_GEMM_STREAMK=1" \
           "BZ_GEMM_BN=256 BZ_GEMM_STREAMK=1"; do
  echo "== ${cfg:-model}"
  env $cfg python scripts/skinny_bench.py 1 8 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"  m={d['m']} {d['shape']:8s} ctas {d['ctas']:4d} ours {d['ours']['us']:7.2f} us {d['ours']['GBps']:7.1f} GB/s  cublas {d['cublas']['us']:7.2f}\")"
done
