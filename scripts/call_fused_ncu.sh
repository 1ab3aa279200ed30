timeout 300 python scripts/fused_once.py 1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decode_fused -s 3 -c 1 -o gpurun_out/fused_b1 -f python scripts/fused_once.py 1 > gpurun_out/fused_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/fused_ncu.log
