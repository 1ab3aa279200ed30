#!/bin/bash
# prefill GEMMs vs cuBLAS at short prompts: twice, then forced tile configs at M=1024
python scripts/gemm_msweep.py 2>&1 | grep '^{' > gpurun_out/ms1.jsonl
python scripts/gemm_msweep.py 2>&1 | grep '^{' > gpurun_out/ms2.jsonl
for cfg in "BZ_GEMM_BN=256 BZ_GEMM_NSUB=1" "BZ_GEMM_BN=240 BZ_GEMM_NSUB=1" "BZ_GEMM_BN=256 BZ_GEMM_NSUB=2" "BZ_GEMM_PAIR=0" "BZ_GEMM_BN=192 BZ_GEMM_NSUB=2"; do
  echo "== $cfg"; env $cfg BZ_MS=1024 python scripts/gemm_msweep.py 2>&1 | grep '^{' | grep gate_up
done
