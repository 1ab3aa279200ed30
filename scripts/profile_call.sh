#!/bin/bash
# one-GPU ncu evidence: launch list of the bench command + full captures of the top kernels
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n1.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_n1.log 2>&1
echo "launch list rc=$?"
python scripts/profile_single.py push gemm block > gpurun_out/prof_single_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_single.csv \
    python scripts/profile_single.py push gemm block > gpurun_out/ncu_single.log 2>&1
echo "single launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16 -s 1 -c 2 -o gpurun_out/prof_gemm \
    python scripts/profile_single.py gemm > gpurun_out/ncu_gemm.log 2>&1
echo "gemm full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_push_tiles -s 1 -c 1 -o gpurun_out/prof_push \
    python scripts/profile_single.py push > gpurun_out/ncu_push.log 2>&1
echo "push full rc=$?"
python scripts/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1; echo "gemm bench rc=$?"; cat gpurun_out/gemm_bench.log
