#!/bin/bash
# ncu --set full of the prefill GEMM (qkv @ 2000 tokens, 2nd launch) after a clean run
mkdir -p gpurun_out
python scripts/profile_single.py gemm > gpurun_out/prof_gemm_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16 -s 1 -c 1 -o gpurun_out/prof_gemm_r1b \
    python scripts/profile_single.py gemm > gpurun_out/ncu_gemm.log 2>&1
echo "gemm full rc=$?"
ncu -i gpurun_out/prof_gemm_r1b.ncu-rep --page raw --csv > gpurun_out/prof_gemm_r1b_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_gemm_r1b.ncu-rep --page details --csv > gpurun_out/prof_gemm_r1b_details.csv 2>/dev/null
ls -la gpurun_out/prof_gemm_r1b*
