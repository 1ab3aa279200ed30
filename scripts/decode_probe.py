"""One Llama-2 7B block decode step (B sequences, 1024 cached tokens), eager, for
ncu launch lists: python scripts/decode_probe.py [B]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200.dataplane import DeviceSlab  # noqa: E402
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
a = S.LLAMA2_7B
probe = S.LlamaArch("probe", a.d_model, 1, a.n_heads, a.n_kv_heads, a.ffn)
lay = S.SlabLayout.for_arch(probe)
slab = DeviceSlab(lay, 0)
w = SlabWeights(probe, lay, slab.data)
w.init_random(0)
ex = LlamaExecutor(w, max_tokens=max(B, 8), device="cuda")
kv = KVCache(probe, B, 1100, "cuda")
kv.length = 1024
x = torch.randn(B, a.d_model, device="cuda").to(torch.bfloat16)
for _ in range(3):
    ex.decode_block(0, x, kv)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    ex.decode_block(0, x, kv)
ev[1].record()
torch.cuda.synchronize()
print(f"B={B} eager block step {ev[0].elapsed_time(ev[1]) / 20 * 1e3:.1f} us")
