"""Phase timeline of the fused decode kernel (bz_decode_fused_set_trace): 8 distinct
7B blocks at batch B, KV at 1024 tokens; prints per-phase median / max over CTAs (us)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights

EV = ["start", "norm1", "qkv", "bar1", "attn", "bar2", "comb", "o", "bar3", "norm2", "gu", "bar4", "act", "down",
      "p_qkv", "p_o", "p_gu", "p_down", "a_q", "a_s", "a_sm", "a_pv"]
nl, B = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
a = S.LLAMA2_7B
probe = S.LlamaArch("probe", a.d_model, nl, a.n_heads, a.n_kv_heads, a.ffn, a.vocab)
lay = S.SlabLayout.for_arch(probe)
slab = DeviceSlab(lay, 0)
w = SlabWeights(probe, lay, slab.data)
w.init_random(seed=0)
ex = LlamaExecutor(w, max_tokens=8, device="cuda:0")
kv = KVCache(probe, B, ctx + 64, "cuda:0")
kv.length = ctx
x = torch.randn(B, a.d_model, device="cuda").to(torch.bfloat16)
for _ in range(3):
    ex.decode_blocks(0, nl, x, kv)
sms = torch.cuda.get_device_properties(0).multi_processor_count
buf = torch.zeros(sms * nl * len(EV), dtype=torch.int64, device="cuda")
ex.lib.bz_decode_fused_set_trace(buf.data_ptr(), buf.numel() * 8)
ex.decode_blocks(0, nl, x, kv)
torch.cuda.synchronize()
ex.lib.bz_decode_fused_set_trace(None, 0)
t = buf.view(sms, nl, len(EV)).double().cpu()
t0 = t[:, 0, 0].min()
t = (t - t0) / 1e3
total = (t[:, -1, EV.index("down")].max()).item()
print(f"B={B}: step {total:.1f} us for {nl} blocks = {total / nl:.1f} us per block")
for l in (1, nl - 1):
    print(f"block {l}: start median {t[:, l, 0].median():.1f}")
    prev = "start"
    for e in EV[1:14]:
        d = t[:, l, EV.index(e)] - t[:, l, EV.index(prev)]
        print(f"  {prev:>6s}->{e:<6s} median {d.median():7.2f}  max {d.max():7.2f}  min {d.min():7.2f}")
        prev = e
    prev = "bar1"
    for e in EV[18:]:
        d = t[:, l, EV.index(e)] - t[:, l, EV.index(prev)]
        ok = t[:, l, EV.index(e)] > 0
        print(f"  attn {prev:>5s}->{e:<5s} median {d[ok].median():7.2f}  max {d[ok].max():7.2f}")
        prev = e
    for e in EV[14:18]:
        d = t[:, l, EV.index(e)] - t[:, l, 0]
        print(f"  producer {e:<7s} done at +{d.median():7.2f} (max {d.max():7.2f}) after block start")
