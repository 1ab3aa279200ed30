"""Fused small-batch decode (bz_decode_fused: one persistent kernel per step) against
the per-block kernels and the fp32 oracle.

The two GPU paths round to bf16 at the same points, so their step outputs agree to
fp32-summation-order noise; the oracle bar is the decode tests' (max relative error
<= 1e-2 on the logits, greedy tokens equal where the oracle's margin is decisive).
"""

import pytest
import torch

from paper_2412_17246_b200 import llama as LL
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights
from oracle.forward_ref import forward_fp32, weights_to_cpu_fp32

pytestmark = pytest.mark.gpu

# the fused kernel streams 64-wide k tiles: ffn a multiple of 64 (704 = 11 x 64)
FT_MHA = S.LlamaArch("ft-mha", d_model=256, n_layers=4, n_heads=4, n_kv_heads=4, ffn=704)
FT_GQA = S.LlamaArch("ft-gqa", d_model=256, n_layers=4, n_heads=4, n_kv_heads=2, ffn=704)
GQA8 = S.LlamaArch("gqa8", d_model=1024, n_layers=2, n_heads=16, n_kv_heads=2, ffn=2816)
W7B_2L = S.LlamaArch("w7b-2l", d_model=4096, n_layers=2, n_heads=32, n_kv_heads=32, ffn=11008)


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / (b.float().abs().max() + 1e-6)).item()


def _check(got, want):
    got = got.cpu()
    assert _rel(got, want) <= 1e-2
    top2 = want.topk(2, dim=-1).values
    decisive = (top2[:, 0] - top2[:, 1]) > 2e-2 * want.abs().max()
    assert torch.equal(got.argmax(-1)[decisive], want.argmax(-1)[decisive])


def _setup(arch, seed=0):
    lay = S.SlabLayout.for_arch(arch, tile_bytes=1 << 20)
    slab = DeviceSlab(lay, 0)
    w = SlabWeights(arch, lay, slab.data)
    w.init_random(seed=seed)
    torch.cuda.synchronize()
    return slab, w


def _prompt(b, s, seed, vocab):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (b, s), generator=g).cuda()


def _two_paths(monkeypatch, arch, B, S_prompt, steps, seed=3):
    """Decode `steps` tokens with the fused kernel (greedy) and with the per-block kernels
    fed the SAME tokens (a near-tie argmax flip must not fork the inputs); returns both
    logit sequences, both caches and the executor."""
    slab, w = _setup(arch, seed)
    ex = LlamaExecutor(w, max_tokens=B * S_prompt, device="cuda")
    prompt = _prompt(B, S_prompt, seed + 1, arch.vocab)
    out = {}
    fed = []
    for fused in (True, False):
        monkeypatch.setattr(LL, "FUSED_DECODE", fused)
        kv = KVCache(arch, B, S_prompt + steps + 2, "cuda")
        logits = ex.forward(prompt, kv=kv)
        tok = logits.argmax(-1)
        seq = []
        for i in range(steps):
            if fused:
                fed.append(tok)
            logits = ex.decode(fed[i], kv)
            seq.append(logits)
            tok = logits.argmax(-1)
        torch.cuda.synchronize()
        out[fused] = (seq, kv)
    monkeypatch.setattr(LL, "FUSED_DECODE", True)
    assert ex.fused_decode_ok(B, out[True][1], 0, arch.n_layers)
    assert not ex.fused_decode_timed_out(B)
    return out, ex, prompt, w, slab


@pytest.mark.parametrize("arch,B", [(FT_MHA, 1), (FT_MHA, 3), (FT_GQA, 2), (GQA8, 4)],
                         ids=["mha-b1", "mha-b3", "gqa-b2", "gqa8-b4"])
def test_fused_decode_matches_per_block_kernels_and_oracle(monkeypatch, arch, B):
    out, ex, prompt, w, slab = _two_paths(monkeypatch, arch, B, 24, 5)
    (fz, kv_f), (pb, kv_p) = out[True], out[False]
    ref_w = weights_to_cpu_fp32(w)
    seq = prompt.cpu()
    tok = None
    for i in range(5):
        assert _rel(fz[i], pb[i]) < 5e-3, i
        # teacher-forced oracle over the fused path's own greedy tokens
        prev = (ex.forward(prompt) if i == 0 else fz[i - 1]).argmax(-1)
        seq = torch.cat([seq, prev.cpu()[:, None]], 1)
        _check(fz[i], forward_fp32(arch, ref_w, seq))
        tok = fz[i].argmax(-1)
    assert tok is not None
    # the appended keys / values agree with the per-block kernels' (RoPE'd, bf16)
    n = kv_f.length
    assert n == kv_p.length == 24 + 5
    for l in kv_f.k:
        assert _rel(kv_f.k[l][:, :, 24:n], kv_p.k[l][:, :, 24:n]) < 2e-2
        assert _rel(kv_f.v[l][:, :, 24:n], kv_p.v[l][:, :, 24:n]) < 2e-2
    slab.close()


def test_fused_decode_7b_width(monkeypatch):
    """Full Llama-2 7B block width (d 4096, ffn 11008, 32 heads of 128), 2 blocks, batch 1."""
    out, ex, prompt, w, slab = _two_paths(monkeypatch, W7B_2L, 1, 64, 3)
    for a, b in zip(out[True][0], out[False][0]):
        assert _rel(a, b) < 1e-2
        assert torch.equal(a.argmax(-1), b.argmax(-1)) or _rel(a, b) < 5e-3
    slab.close()


def test_fused_decode_per_row_positions_and_small_grid(monkeypatch):
    """Continuous batching (one device position per row) and a grid of fewer CTAs than
    SMs: each row's step equals the per-block kernels' on the same cache."""
    arch = FT_GQA
    slab, w = _setup(arch, seed=11)
    ex = LlamaExecutor(w, max_tokens=64, device="cuda")
    lens = [19, 5, 11, 2]
    caches = {}
    for fused in (True, False):
        monkeypatch.setattr(LL, "FUSED_DECODE", fused)
        kv = KVCache(arch, 4, 32, "cuda", per_row=True)
        g = torch.Generator(device="cuda").manual_seed(7)
        for l in kv.k:
            kv.k[l].normal_(0, 1, generator=g)
            kv.v[l].normal_(0, 1, generator=g)
        kv.pos_dev.copy_(torch.tensor(lens, dtype=torch.int32))
        toks = torch.tensor([3, 14, 15, 92], device="cuda")
        caches[fused] = (ex.decode(toks, kv), kv)
    torch.cuda.synchronize()
    (lf, kf), (lp, kp) = caches[True], caches[False]
    assert _rel(lf, lp) < 5e-3
    assert kf.pos_dev.tolist() == [n + 1 for n in lens]
    for l in kf.k:
        for r, n in enumerate(lens):   # row r wrote exactly its own position n
            assert _rel(kf.k[l][r, :, n], kp.k[l][r, :, n]) < 2e-2
            assert torch.equal(kf.k[l][r, :, :n], kp.k[l][r, :, :n])
    # a 37-CTA grid: same rows per warp (bitwise-equal projections), other attention splits
    x = torch.randn(4, arch.d_model, device="cuda").to(torch.bfloat16)
    kv2 = KVCache(arch, 4, 32, "cuda", per_row=True)
    kv2.pos_dev.copy_(torch.tensor(lens, dtype=torch.int32))
    a = ex.decode_blocks(0, arch.n_layers, x, kv2)
    full = a.clone()
    kv2.pos_dev.copy_(torch.tensor(lens, dtype=torch.int32))
    orig = ex.lib.bz_decode_fused

    def small_grid(*args):
        args = list(args)
        args[-2] = 37
        return orig(*args)

    monkeypatch.setattr(ex.lib, "bz_decode_fused", small_grid, raising=False)
    b = ex.decode_blocks(0, arch.n_layers, x, kv2)
    torch.cuda.synchronize()
    assert _rel(b, full) < 5e-3
    slab.close()


def test_fused_decode_graph_replay_is_identical(monkeypatch):
    """A captured fused step (cooperative kernel inside a CUDA graph) replays bit-exactly."""
    monkeypatch.setattr(LL, "FUSED_DECODE", True)
    arch = FT_MHA
    slab, w = _setup(arch, seed=5)
    ex = LlamaExecutor(w, max_tokens=2 * 16, device="cuda")
    prompt = _prompt(2, 16, 9, arch.vocab)
    kv_e, kv_g = KVCache(arch, 2, 24, "cuda"), KVCache(arch, 2, 24, "cuda")
    first = ex.forward(prompt, kv=kv_e)
    ex.forward(prompt, kv=kv_g)
    graph = ex.decode_graph(kv_g)
    tok = first.argmax(-1)
    for _ in range(4):
        eager = ex.decode(tok, kv_e)
        replay = graph(tok).clone()
        assert torch.equal(eager, replay)
        tok = eager.argmax(-1)
    slab.close()


def test_fused_decode_rejects_unsupported_shapes(monkeypatch):
    """Five sequences (or an ffn that is not a multiple of 64) fall back to the per-block kernels."""
    monkeypatch.setattr(LL, "FUSED_DECODE", True)
    arch = FT_MHA
    slab, w = _setup(arch)
    ex = LlamaExecutor(w, max_tokens=8, device="cuda")
    kv5 = KVCache(arch, 5, 8, "cuda")
    assert not ex.fused_decode_ok(5, kv5, 0, arch.n_layers)
    assert ex.fused_decode_ok(4, kv5, 0, arch.n_layers)
    ex688 = LlamaExecutor(SlabWeights(S.TINY_4L, S.SlabLayout.for_arch(S.TINY_4L), torch.zeros(
        S.SlabLayout.for_arch(S.TINY_4L).data_bytes, dtype=torch.uint8, device="cuda")), max_tokens=8, device="cuda")
    assert not ex688.fused_decode_ok(1, KVCache(S.TINY_4L, 1, 8, "cuda"), 0, 4)
    from paper_2412_17246_b200._native import BlitzError, BzDecodeBlock
    with pytest.raises(BlitzError):
        ex.lib.bz_decode_fused((BzDecodeBlock * 1)(), 1, None, 0, 5, 256, 4, 4, 64, 688, 1e4, 1e-5, 8, None, 0,
                               None, 0, 0, None)
    slab.close()


def test_fused_decode_more_blocks_than_one_launch(monkeypatch):
    """50 blocks: the host runs them as launches of 48 + 2 (tensor maps travel in the
    kernel parameters); the step matches the per-block kernels."""
    arch = S.LlamaArch("ft-deep", d_model=256, n_layers=50, n_heads=4, n_kv_heads=2, ffn=704)
    out, ex, prompt, w, slab = _two_paths(monkeypatch, arch, 2, 16, 2, seed=8)
    for a, b in zip(out[True][0], out[False][0]):
        assert _rel(a, b) < 1e-2
    slab.close()
