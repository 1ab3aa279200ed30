# K-chunked kernel: forced tile widths, with and without the MMAs (TMA stream rate vs MMA rate)
for bn in 32 64 128 256; do for nm in 0 1; do echo "== BN=$bn NOMMA=$nm"; BZ_GEMM_KC_BN=$bn BZ_GEMM_KC_NOMMA=$nm timeout 120 python scripts/skinny_bench.py 1 | cut -c1-90; done; done 2>&1 | tee gpurun_out/kc2.log
