"""Batch-1 decode step of 8 distinct 7B blocks (KV at 1024), graph-replayed, with parts of
the per-block kernel chain left out (timing only -- the math of a reduced chain is wrong):
how much of the 106 us per block is the four weight GEMMs and how much the glue kernels."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights

nl, ctx = 8, 1024
a = S.LLAMA2_7B
probe = S.LlamaArch("probe", a.d_model, nl, a.n_heads, a.n_kv_heads, a.ffn, a.vocab)
lay = S.SlabLayout.for_arch(probe)
slab = DeviceSlab(lay, 0)
w = SlabWeights(probe, lay, slab.data)
w.init_random(seed=0)
ex = LlamaExecutor(w, max_tokens=8, device="cuda:0")
kv = KVCache(probe, 1, ctx + 64, "cuda:0")
kv.length = ctx
x0 = torch.randn(1, a.d_model, device="cuda").to(torch.bfloat16)


def body(parts):
    x = x0
    s = torch.cuda.current_stream().cuda_stream
    for k in range(nl):
        L = ex.w.layers[k]
        h, qkv, attn, o, gu, act = ex.h[:1], ex.qkv[:1], ex.attn[:1], ex.o[:1], ex.gu[:1], ex.act[:1]
        if "norm" in parts:
            ex._rmsnorm(x, L["attn_norm"], h)
        ex._gemm(h, L["wqkv"], qkv)
        if "rope" in parts:
            ex.lib.bz_rope_append(qkv.data_ptr(), qkv.stride(0), 1, a.n_heads, a.n_kv_heads, a.head_dim, a.rope_theta,
                                  kv.k[k].data_ptr(), kv.v[k].data_ptr(), kv.max_seq, kv.pos_dev.data_ptr(), s)
        if "attn" in parts:
            ex.lib.bz_decode_attention(qkv.data_ptr(), qkv.stride(0), kv.k[k].data_ptr(), kv.v[k].data_ptr(), 1,
                                       a.n_heads, a.n_kv_heads, a.head_dim, kv.max_seq, kv.pos_dev.data_ptr(),
                                       attn.data_ptr(), attn.stride(0), kv.workspace.data_ptr(), kv.workspace.numel(), s)
        ex._gemm(attn, L["wo"], o, residual=x)
        if "norm" in parts:
            ex._rmsnorm(o, L["ffn_norm"], h)
        ex._gemm(h, L["wgu"], gu)
        if "silu" in parts:
            ex.lib.bz_silu_mul(gu.data_ptr(), act.data_ptr(), 1, a.ffn, gu.stride(0), act.stride(0), s)
        out = torch.empty_like(x) if k == nl - 1 else ex.o2 if hasattr(ex, "o2") else torch.empty_like(x)
        ex._gemm(act, L["wdown"], out, residual=o)
        x = out
    return x


for label, parts in (("all", {"norm", "rope", "attn", "silu"}), ("gemms only", set()),
                     ("gemms + attention", {"rope", "attn"}), ("gemms + norms + silu", {"norm", "silu"})):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        body(parts)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            body(parts)
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    e1.synchronize()
    print(f"{label:22s}: {e0.elapsed_time(e1) / 20 * 1e3 / nl:6.1f} us per block")
