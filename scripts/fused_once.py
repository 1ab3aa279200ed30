"""One eager fused decode step over 8 distinct 7B blocks at batch B (ncu target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights

nl, ctx, B = 8, 1024, int(sys.argv[1]) if len(sys.argv) > 1 else 1
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
for _ in range(4):
    ex.decode_blocks(0, nl, x, kv)
torch.cuda.synchronize()
print("ok")
