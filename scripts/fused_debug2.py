"""Replicates test_fused_decode_matches_per_block_kernels_and_oracle[gqa8-b4] with per-step errors."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2412_17246_b200 import llama as LL
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights

def case(arch, B, nsteps=5, seed=3):
    lay = S.SlabLayout.for_arch(arch, tile_bytes=1 << 20)
    slab = DeviceSlab(lay, 0)
    w = SlabWeights(arch, lay, slab.data)
    w.init_random(seed=seed)
    ex = LlamaExecutor(w, max_tokens=B * 24, device="cuda")
    g = torch.Generator().manual_seed(seed + 1)
    prompt = torch.randint(0, arch.vocab, (B, 24), generator=g).cuda()
    res = {}
    for fused in (True, False):
        LL.FUSED_DECODE = fused
        kv = KVCache(arch, B, 24 + nsteps + 2, "cuda")
        lg = ex.forward(prompt, kv=kv)
        tok = lg.argmax(-1)
        seq = []
        for _ in range(nsteps):
            lg = ex.decode(tok, kv)
            seq.append(lg.float().clone())
            tok = lg.argmax(-1)
        res[fused] = seq
    torch.cuda.synchronize()
    for i, (a, b) in enumerate(zip(res[True], res[False])):
        rel = ((a - b).abs().max() / b.abs().max()).item()
        rows = [round(((a[r] - b[r]).abs().max() / b[r].abs().max()).item(), 4) for r in range(B)]
        print(f"{arch.name} B={B} step {i}: rel {rel:.4f} rows {rows} argmax_eq {torch.equal(a.argmax(-1), b.argmax(-1))}")
    slab.close()

case(S.LlamaArch("gqa8", d_model=1024, n_layers=2, n_heads=16, n_kv_heads=2, ffn=2816), 4)
case(S.LlamaArch("gqa8-1l", d_model=1024, n_layers=1, n_heads=16, n_kv_heads=2, ffn=2816), 4)
case(S.LlamaArch("gqa8", d_model=1024, n_layers=2, n_heads=16, n_kv_heads=2, ffn=2816), 1)
