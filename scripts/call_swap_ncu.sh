# launch list of one graph-replayed batch-1 decode step (8 x 7B blocks) and a full capture of the swapped decode GEMM
timeout 300 python scripts/decode_breakdown.py 1 > gpurun_out/swap_bd.log 2>&1; echo "bd rc=$?"; cat gpurun_out/swap_bd.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --graph-profiling node -s 400 -c 120 --csv --log-file gpurun_out/ncu_swap_bd.csv python scripts/decode_breakdown.py 1 > gpurun_out/ncu_swap_bd.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_swap -s 6 -c 2 -o gpurun_out/ncu_swap_full python scripts/skinny_bench.py 1 > gpurun_out/ncu_swap_full.log 2>&1; echo "ncu full rc=$?"
