timeout 600 python scripts/fused_debug2.py 2>&1 | tail -20
