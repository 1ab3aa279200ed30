for c in 64 256 1024 4096; do echo "== ctx $c"; BZ_DECODE_FUSED=1 timeout 300 python scripts/fused_trace.py 1 $c 2>&1 | grep -E "step|bar1->attn|attn ->bar2|bar2->comb|a_q|a_s|a_pv" | head -8; done
