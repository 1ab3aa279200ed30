"""Diagnose cooperative execution at 7B shapes on one GPU: the split prefill (and
decode) must equal the unsplit forward bit for bit (same kernels, same M)."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.coop import CooperativePair
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights

ARCH = S.LlamaArch("llama2-7b-l3", 4096, 3, 32, 32, 11008)
B, SEQ, n = int(os.environ.get("B", 4)), int(os.environ.get("SEQ", 64)), 4
lay = S.SlabLayout.for_arch(ARCH)
src, tgt = DeviceSlab(lay, 0), DeviceSlab(lay, 0)
w = SlabWeights(ARCH, lay, src.data); w.init_random(seed=0)
tgt.data.copy_(src.data); tgt.loaded.fill_(ARCH.n_layers)
torch.cuda.synchronize()
g = torch.Generator().manual_seed(11)
batches = [torch.randint(0, ARCH.vocab, (B, SEQ), generator=g).cuda() for _ in range(n)]
ref_ex = LlamaExecutor(w, max_tokens=B * SEQ, device="cuda")
ref_logits, ref_dec = [], []
for b in batches:
    kv = KVCache(ARCH, B, SEQ + 2, "cuda")
    lg = ref_ex.forward(b, kv=kv)
    ref_logits.append(lg)
    ref_dec.append(ref_ex.decode(lg.argmax(-1), kv))
torch.cuda.synchronize()
cfg = ss.configure_pipeline(n, ARCH.n_layers, 0.5)
tl = ss.zigzag_schedule(cfg)
for fused in (True, False):
    pair = CooperativePair(LlamaExecutor(w, max_tokens=B * SEQ, device="cuda"),
                           LlamaExecutor(SlabWeights(ARCH, lay, tgt.data), max_tokens=B * SEQ, device="cuda"),
                           tgt.loaded, fused_handoff=fused)
    caches = pair.make_caches(batches, cfg, max_new_tokens=2)
    res = pair.run(batches, cfg, tl, caches=caches)
    toks = [lg.argmax(-1) for lg in ref_logits]
    dec = pair.decode(toks, cfg, caches)
    out = {"fused": fused, "splits": cfg.splits,
           "prefill_max_abs": [float((a - r).abs().max()) for a, r in zip(res.logits, ref_logits)],
           "decode_max_abs": [float((a - r).abs().max()) for a, r in zip(dec.logits, ref_dec)]}
    print(json.dumps(out), flush=True)
