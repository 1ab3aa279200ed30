# full ncu captures of the two other decode GEMM kernels (gate/up K-chunked BN=160, down swapped S=4), M = 1
timeout 300 python scripts/skinny_bench.py 1 > gpurun_out/sk1.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_skinny_kc -s 4 -c 1 -o gpurun_out/ncu_kc160 python scripts/skinny_bench.py 1 > gpurun_out/ncu_kc160.log 2>&1; echo "ncu kc rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_swap -s 30 -c 1 -o gpurun_out/ncu_swap4 python scripts/skinny_bench.py 1 > gpurun_out/ncu_swap4.log 2>&1; echo "ncu swap rc=$?"
