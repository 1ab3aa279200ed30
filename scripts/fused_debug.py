"""Fused vs per-block decode, one step, several shapes (debug aid)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2412_17246_b200 import llama as LL
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights

def run(arch, B, nl_note=""):
    lay = S.SlabLayout.for_arch(arch, tile_bytes=1 << 20)
    slab = DeviceSlab(lay, 0)
    w = SlabWeights(arch, lay, slab.data)
    w.init_random(seed=3)
    ex = LlamaExecutor(w, max_tokens=64, device="cuda")
    x = torch.randn(B, arch.d_model, device="cuda").to(torch.bfloat16)
    outs = {}
    for fused in (True, False):
        LL.FUSED_DECODE = fused
        kv = KVCache(arch, B, 40, "cuda")
        g = torch.Generator(device="cuda").manual_seed(1)
        for l in kv.k:
            kv.k[l].normal_(0, 1, generator=g); kv.v[l].normal_(0, 1, generator=g)
        kv.length = 20
        outs[fused] = ex.decode_blocks(0, 1, x, kv).float()
    torch.cuda.synchronize()
    a, b = outs[True], outs[False]
    rel = ((a - b).abs().max() / b.abs().max()).item()
    rows = [((a[i] - b[i]).abs().max() / b[i].abs().max()).item() for i in range(B)]
    print(f"{arch.name:10s} B={B} rel={rel:.4f} per-row={[round(r, 4) for r in rows]}")
    slab.close()

for (d, H, KV, ffn) in [(1024, 16, 2, 2816), (1024, 16, 16, 2816), (1024, 16, 2, 704), (256, 4, 2, 2816), (512, 8, 2, 1408)]:
    for B in (1, 4):
        run(S.LlamaArch(f"d{d}h{H}k{KV}f{ffn}", d, 1, H, KV, ffn), B)
