"""One batch-1 decode step of 8 distinct 7B blocks (KV at 1024 tokens), graph-replayed:
per-kernel device times come from ncu (--graph-profiling node); this script alone prints
the CUDA-event step time and the weight bandwidth."""
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
ex = LlamaExecutor(w, max_tokens=max(B, 8), device="cuda:0")
kv = KVCache(probe, B, ctx + 64, "cuda:0")
for t in list(kv.k.values()) + list(kv.v.values()):
    t.normal_(0, 1)
kv.length = ctx
g = ex.decode_graph(kv, 0, nl, hidden_in=True, head=False)
g.hidden.normal_(0, 1)
for _ in range(5):
    g()
torch.cuda.synchronize()
kv.length = ctx
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    g()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 20
wbytes = nl * a.block_bytes()
print(f"B={B}: {ms * 1e3 / nl:.1f} us per block, weights {wbytes / (ms / 1e3) / 1e9:.0f} GB/s")
