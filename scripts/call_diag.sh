timeout 600 python scripts/coop_diag.py > gpurun_out/coop_diag.log 2>&1; echo rc=$?
BZ_GEMM_PAIR=0 timeout 600 python scripts/coop_diag.py > gpurun_out/coop_diag_nopair.log 2>&1; echo rc=$?
B=1 SEQ=256 timeout 600 python scripts/coop_diag.py > gpurun_out/coop_diag_b1.log 2>&1; echo rc=$?
tail -4 gpurun_out/coop_diag*.log
