timeout 300 python scripts/decode_breakdown.py 1 > gpurun_out/decode_bd2.log 2>&1; BZ_GEMV=0 python scripts/decode_breakdown.py 1 >> gpurun_out/decode_bd2.log 2>&1; cat gpurun_out/decode_bd2.log
