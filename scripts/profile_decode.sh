#!/bin/bash
# ncu --set full of one 7B decode block's attention (batch 64, 1024 cached tokens) and
# its first skinny GEMM (batch 1), each after a clean run of the same command
mkdir -p gpurun_out
export PYTHONPATH=$PWD
python scripts/decode_probe.py 64 > gpurun_out/pd_plain64.log 2>&1 || { echo "plain 64 failed"; exit 1; }
python scripts/decode_probe.py 1 > gpurun_out/pd_plain1.log 2>&1 || { echo "plain 1 failed"; exit 1; }
ncu --set full --clock-control none -k regex:k_decode_partial -s 5 -c 1 -o gpurun_out/prof_decode_attn_b64 \
    python scripts/decode_probe.py 64 > gpurun_out/ncu_pd64.log 2>&1; echo "attn rc=$?"
ncu --set full --clock-control none -k regex:k_gemm_bf16 -s 8 -c 4 -o gpurun_out/prof_decode_gemm_b1 \
    python scripts/decode_probe.py 1 > gpurun_out/ncu_pd1.log 2>&1; echo "gemm rc=$?"
for f in prof_decode_attn_b64 prof_decode_gemm_b1; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
done
ls -la gpurun_out/prof_decode_*
