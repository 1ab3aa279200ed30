"""Decode (KV-cache) path, prefill->decode mutation on a real instance, and
cooperative decode under a ZigZag split -- all against the fp32 CPU oracle.

Oracle: ``forward_fp32`` over the prompt plus the tokens generated so far
(teacher-forced full recompute), so the incremental KV path is checked against
an independent computation.  Tolerance as for prefill (north star): max
relative error <= 1e-2, identical greedy tokens where the oracle's top-2
margin is decisive.
"""

import pytest
import torch

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.coop import CooperativePair
from paper_2412_17246_b200.dataplane import DeviceSlab, execute_plan_loopback
from paper_2412_17246_b200.instance import ServingInstance
from paper_2412_17246_b200.livescale import ProtocolError, mutate_decode_to_prefill
from paper_2412_17246_b200.llama import KVCache, LlamaExecutor, SlabWeights
from oracle.forward_ref import forward_fp32, weights_to_cpu_fp32

pytestmark = pytest.mark.gpu

TINY_GQA = S.LlamaArch("tiny-gqa", d_model=256, n_layers=4, n_heads=4, n_kv_heads=2, ffn=688)


def _rel(a, b):
    return ((a - b).abs().max() / (b.abs().max() + 1e-6)).item()


def _check(got, want):
    got = got.cpu()
    assert _rel(got, want) <= 1e-2
    top2 = want.topk(2, dim=-1).values
    decisive = (top2[:, 0] - top2[:, 1]) > 2e-2 * want.abs().max()
    assert torch.equal(got.argmax(-1)[decisive], want.argmax(-1)[decisive])


def _slab(arch, seed=0):
    lay = S.SlabLayout.for_arch(arch, tile_bytes=128 * 1024)
    slab = DeviceSlab(lay, 0)
    w = SlabWeights(arch, lay, slab.data)
    w.init_random(seed=seed)
    torch.cuda.synchronize()
    return lay, slab, w


def _prompt(b, s, seed, vocab):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (b, s), generator=g).cuda()


@pytest.mark.parametrize("arch", [S.TINY_4L, TINY_GQA], ids=["mha", "gqa"])
def test_kv_decode_matches_full_recompute(arch):
    lay, slab, w = _slab(arch)
    ref_w = weights_to_cpu_fp32(w)
    ex = LlamaExecutor(w, max_tokens=3 * 24, device="cuda")
    prompt = _prompt(3, 24, 5, arch.vocab)
    kv = KVCache(arch, 3, 24 + 6, "cuda")
    logits = ex.forward(prompt, kv=kv)
    assert kv.length == 24
    seq = prompt.cpu()
    _check(logits, forward_fp32(arch, ref_w, seq))
    tok = logits.argmax(-1)
    for step in range(6):
        seq = torch.cat([seq, tok.cpu()[:, None]], 1)
        logits = ex.decode(tok, kv)
        assert kv.length == 25 + step
        _check(logits, forward_fp32(arch, ref_w, seq))
        tok = logits.argmax(-1)
    full = KVCache(arch, 1, 2, "cuda")
    full.length = 2
    with pytest.raises(ValueError):
        full.advance()
    slab.close()


def test_graph_replayed_decode_is_identical_to_eager():
    """The captured step reads its position from the device: replaying one graph
    for every token gives exactly the eager step's logits."""
    arch = S.TINY_4L
    lay, slab, w = _slab(arch, seed=9)
    ex = LlamaExecutor(w, max_tokens=4 * 40, device="cuda")
    prompt = _prompt(4, 40, 2, arch.vocab)
    kv_e, kv_g = KVCache(arch, 4, 48, "cuda"), KVCache(arch, 4, 48, "cuda")
    first = ex.forward(prompt, kv=kv_e)
    assert torch.equal(first, ex.forward(prompt, kv=kv_g))
    graph = ex.decode_graph(kv_g)
    tok = first.argmax(-1)
    for _ in range(6):
        eager = ex.decode(tok, kv_e)
        replay = graph(tok).clone()
        assert kv_e.length == kv_g.length
        assert torch.equal(eager, replay)
        tok = eager.argmax(-1)
    for l in kv_e.k:
        assert torch.equal(kv_e.k[l][:, :, :kv_e.length], kv_g.k[l][:, :, :kv_g.length])
    slab.close()


def test_prefill_to_decode_mutation_moves_no_bytes():
    """livescale.py:512-544: a fully resident prefill instance flips to decode and
    keeps serving its sequences from the same slab and KV cache."""
    arch = S.TINY_4L
    lay, slab, w = _slab(arch, seed=3)
    ref_w = weights_to_cpu_fp32(w)
    inst = ServingInstance("inst0", arch, slab, role="prefill", max_tokens=64)
    with pytest.raises(ProtocolError):                       # not resident yet
        inst.prefill(_prompt(2, 16, 1, arch.vocab))
    with pytest.raises(ProtocolError):
        ss.mutate_prefill_to_decode(inst)
    inst.mark_resident()
    prompt = _prompt(2, 16, 1, arch.vocab)
    logits, kv = inst.prefill(prompt, max_new_tokens=4)
    with pytest.raises(ProtocolError):                       # prefill role cannot decode
        inst.decode(logits.argmax(-1), kv)
    inst.live_session = object()
    with pytest.raises(ProtocolError):                       # mid-scale
        ss.mutate_prefill_to_decode(inst)
    inst.live_session = None
    ptr_before, kv_ptr = slab.ptr, kv.k[0].data_ptr()
    res = ss.mutate_prefill_to_decode(inst, compensation_count=2)
    assert inst.role == "decode" and res.instance is inst
    assert res.compensation.model == arch.name and res.compensation.count == 2
    toks, step_logits = inst.generate(kv, logits.argmax(-1), 4)
    assert slab.ptr == ptr_before and kv.k[0].data_ptr() == kv_ptr   # nothing moved
    seq = torch.cat([prompt.cpu(), logits.argmax(-1).cpu()[:, None]], 1)
    for t, lg in enumerate(step_logits):
        _check(lg, forward_fp32(arch, ref_w, seq))
        seq = torch.cat([seq, toks[:, t].cpu()[:, None]], 1)
    assert mutate_decode_to_prefill(inst).role == "prefill"
    slab.close()


@pytest.mark.parametrize("n,time_l", [(4, 1.0), (3, 2.0)])
def test_cooperative_decode_keeps_the_split(n, time_l):
    """Prefill under the configure_pipeline split leaves blocks [0, T_i) of batch
    i's KV on the target and [T_i, L) on the source; decode continues with the
    same split, handing [B, d] per step."""
    arch = S.TINY_4L
    lay, src, w = _slab(arch, seed=4)
    ref_w = weights_to_cpu_fp32(w)
    tgt = DeviceSlab(lay, 0)
    topo = ss.load_topology("b200-hgx")
    plan = ss.generate_plan(ss.build_scale_request(S.model_spec_for(arch), ["gpu0"], ["gpu1"], topo,
                                                   ss.FlowSet(topo)), topo, ss.FlowSet(topo))
    execute_plan_loopback(plan, {"gpu0": src, "gpu1": tgt}, epoch=1)
    torch.cuda.synchronize()
    cfg = ss.configure_pipeline(n, arch.n_layers, time_l)
    pair = CooperativePair(LlamaExecutor(w, max_tokens=64, device="cuda"),
                           LlamaExecutor(SlabWeights(arch, lay, tgt.data), max_tokens=64, device="cuda"),
                           tgt.loaded)
    batches = [_prompt(2, 20, 30 + i, arch.vocab) for i in range(n)]
    caches = pair.make_caches(batches, cfg, max_new_tokens=3)
    res = pair.run(batches, cfg, ss.zigzag_schedule(cfg), caches=caches)
    seqs = [b.cpu() for b in batches]
    toks = []
    for i, lg in enumerate(res.logits):
        _check(lg, forward_fp32(arch, ref_w, seqs[i]))
        toks.append(lg.argmax(-1))
    for (t_i, _), (kt, ks) in zip(cfg.splits, caches):
        assert sorted(kt.k) == list(range(t_i)) and sorted(ks.k) == list(range(t_i, arch.n_layers))
    for _ in range(3):
        seqs = [torch.cat([s, t.cpu()[:, None]], 1) for s, t in zip(seqs, toks)]
        step = pair.decode(toks, cfg, caches)
        assert step.handoff_bytes == sum(2 * arch.d_model * 2 for t, _ in cfg.splits if t > 0)
        for i, lg in enumerate(step.logits):
            _check(lg, forward_fp32(arch, ref_w, seqs[i]))
        toks = [lg.argmax(-1) for lg in step.logits]
    tgt.close()
    src.close()


def _attn_ref(q, kc, vc, length, n_heads, n_kv):
    """fp32 softmax attention of q [B, H, hd] over cache[:, :, :length]."""
    B, _, _, hd = kc.shape
    k = kc[:, :, :length].float().repeat_interleave(n_heads // n_kv, dim=1)
    v = vc[:, :, :length].float().repeat_interleave(n_heads // n_kv, dim=1)
    s = torch.einsum("bhd,bhtd->bht", q.float(), k) / hd ** 0.5
    return torch.einsum("bht,bhtd->bhd", torch.softmax(s, -1), v).reshape(B, n_heads * hd)


@pytest.mark.parametrize("rows,H,KV,hd,s_max,pos", [
    (1, 32, 32, 128, 1100, 1023), (2, 8, 2, 64, 700, 650), (16, 32, 32, 128, 600, 300),
    (3, 64, 8, 128, 300, 0), (4, 4, 4, 64, 40, 39), (2, 16, 4, 128, 2048, 1500),
    # long contexts on few kv heads: the chunk may not shrink past the combine's 64 stages
    (1, 8, 1, 128, 16384, 16000), (1, 8, 2, 64, 6000, 5999),
])
def test_decode_attention_kernel_matches_fp32(rows, H, KV, hd, s_max, pos):
    import ctypes
    from paper_2412_17246_b200._native import cuda_lib
    lib = cuda_lib()
    torch.manual_seed(rows * H + pos)
    q = torch.randn(rows, H * hd, device="cuda").to(torch.bfloat16)
    kc = torch.randn(rows, KV, s_max, hd, device="cuda").to(torch.bfloat16)
    vc = torch.randn(rows, KV, s_max, hd, device="cuda").to(torch.bfloat16)
    p = torch.tensor([pos], dtype=torch.int32, device="cuda")
    nbytes = ctypes.c_int64(0)
    lib.bz_decode_workspace_bytes(rows, H, KV, hd, s_max, ctypes.byref(nbytes))
    ws = torch.zeros(nbytes.value, dtype=torch.uint8, device="cuda")
    out = torch.empty(rows, H * hd, dtype=torch.bfloat16, device="cuda")
    lib.bz_decode_attention(q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), rows, H, KV, hd, s_max,
                            p.data_ptr(), out.data_ptr(), out.stride(0), ws.data_ptr(), ws.numel(),
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = _attn_ref(q.view(rows, H, hd), kc, vc, pos + 1, H, KV)
    assert ((out.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2


@pytest.mark.parametrize("H,KV,hd", [(32, 32, 128), (8, 2, 64)])
def test_rope_append_matches_prefill_rope(H, KV, hd):
    """The decode rotation is the prefill rotation (bit-exact), written into the
    cache at the device position; v is copied unchanged."""
    from paper_2412_17246_b200._native import cuda_lib
    lib = cuda_lib()
    rows, s_max, pos = 3, 64, 37
    ld = (H + 2 * KV) * hd
    torch.manual_seed(H + hd)
    qkv = torch.randn(rows, ld, device="cuda").to(torch.bfloat16)
    ref = qkv.clone()
    positions = torch.full((rows,), pos, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    lib.bz_rope(ref.data_ptr(), positions.data_ptr(), rows, H + KV, hd, ld, 10000.0, s)
    kc = torch.zeros(rows, KV, s_max, hd, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    p = torch.tensor([pos], dtype=torch.int32, device="cuda")
    lib.bz_rope_append(qkv.data_ptr(), ld, rows, H, KV, hd, 10000.0, kc.data_ptr(), vc.data_ptr(), s_max,
                       p.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(qkv[:, : H * hd], ref[:, : H * hd])
    assert torch.equal(kc[:, :, pos].reshape(rows, -1), ref[:, H * hd:(H + KV) * hd])
    assert torch.equal(vc[:, :, pos].reshape(rows, -1), ref[:, (H + KV) * hd:])
    assert int(kc[:, :, :pos].abs().sum().item()) == 0


def test_cooperative_decode_graph_matches_eager():
    """The two-stream captured cooperative step gives the eager step's logits
    bit for bit, and keeps both sides' cache positions in step."""
    arch = S.TINY_4L
    lay, src, w = _slab(arch, seed=6)
    tgt = DeviceSlab(lay, 0)
    tgt.data.copy_(src.data)
    tgt.loaded.fill_(arch.n_layers)
    cfg = ss.configure_pipeline(3, arch.n_layers, 1.0)
    batches = [_prompt(2, 24, 50 + i, arch.vocab) for i in range(3)]
    runs = []
    for _ in range(2):
        pair = CooperativePair(LlamaExecutor(w, max_tokens=64, device="cuda"),
                               LlamaExecutor(SlabWeights(arch, lay, tgt.data), max_tokens=64, device="cuda"),
                               tgt.loaded)
        caches = pair.make_caches(batches, cfg, max_new_tokens=4)
        res = pair.run(batches, cfg, ss.zigzag_schedule(cfg), caches=caches)
        runs.append((pair, caches, [lg.argmax(-1) for lg in res.logits]))
    (pe, ce, toks), (pg, cg, toks_g) = runs
    graph = pg.decode_graph(toks_g, cfg, cg)
    for _ in range(3):
        eager = pe.decode(toks, cfg, ce).logits
        replay = [lg.clone() for lg in graph(toks)]
        for a, b in zip(eager, replay):
            assert torch.equal(a, b)
        for (t_i, _), (kt, ks), (kt2, ks2) in zip(cfg.splits, ce, cg):
            assert ks.length == ks2.length and (t_i == 0 or kt.length == kt2.length)
        toks = [lg.argmax(-1) for lg in eager]
    tgt.close()
    src.close()


def test_kv_consolidation_lets_the_target_decode_alone():
    """After a cooperative prefill and two cooperative decode steps, the source's
    KV blocks [T_i, L) move to the target (bz_copy_panels); the target alone then
    decodes with the merged cache, matching the fp32 oracle."""
    arch = S.TINY_4L
    lay, src, w = _slab(arch, seed=8)
    ref_w = weights_to_cpu_fp32(w)
    tgt = DeviceSlab(lay, 0)
    tgt.data.copy_(src.data)
    tgt.loaded.fill_(arch.n_layers)
    cfg = ss.configure_pipeline(3, arch.n_layers, 2.0)
    pair = CooperativePair(LlamaExecutor(w, max_tokens=64, device="cuda"),
                           LlamaExecutor(SlabWeights(arch, lay, tgt.data), max_tokens=64, device="cuda"),
                           tgt.loaded)
    batches = [_prompt(2, 18, 70 + i, arch.vocab) for i in range(3)]
    caches = pair.make_caches(batches, cfg, max_new_tokens=6)
    res = pair.run(batches, cfg, ss.zigzag_schedule(cfg), caches=caches)
    seqs = [b.cpu() for b in batches]
    toks = [lg.argmax(-1) for lg in res.logits]
    for _ in range(2):
        seqs = [torch.cat([s_, t.cpu()[:, None]], 1) for s_, t in zip(seqs, toks)]
        toks = [lg.argmax(-1) for lg in pair.decode(toks, cfg, caches).logits]
    full, nbytes, _ = pair.consolidate(caches)
    hd, kv_heads = arch.head_dim, arch.n_kv_heads
    assert nbytes == sum(2 * (arch.n_layers - t_i) * 2 * kv_heads * 20 * hd * 2 for t_i, _ in cfg.splits)
    for i, kv in enumerate(full):
        assert sorted(kv.k) == list(range(arch.n_layers)) and kv.length == 20
        seq, tok = seqs[i], toks[i]
        for _ in range(2):
            seq = torch.cat([seq, tok.cpu()[:, None]], 1)
            lg = pair.tgt.decode(tok, kv)
            _check(lg, forward_fp32(arch, ref_w, seq))
            tok = lg.argmax(-1)
    tgt.close()
    src.close()


@pytest.mark.multigpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_kv_consolidation_over_nvlink():
    """Source on cuda:0, new instance on cuda:1: the KV hand-over crosses NVLink
    (peer stores from bz_copy_panels) and the new instance decodes alone."""
    from paper_2412_17246_b200._native import cuda_lib
    lib = cuda_lib()
    lib.bz_enable_peer_mesh(0)
    lib.bz_enable_peer_mesh(1)
    arch = S.TINY_4L
    lay, src, w = _slab(arch, seed=9)
    ref_w = weights_to_cpu_fp32(w)
    with torch.cuda.device(1):
        tgt = DeviceSlab(lay, 1)
        tgt.data.copy_(src.data.to("cuda:1"))
        tgt.loaded.fill_(arch.n_layers)
        target = LlamaExecutor(SlabWeights(arch, lay, tgt.data), max_tokens=64, device="cuda:1")
    source = LlamaExecutor(w, max_tokens=64, device="cuda:0")
    cfg = ss.configure_pipeline(2, arch.n_layers, 1.0)
    pair = CooperativePair(source, target, tgt.loaded)
    batches = [_prompt(2, 16, 90 + i, arch.vocab) for i in range(2)]
    caches = pair.make_caches(batches, cfg, max_new_tokens=2)
    res = pair.run(batches, cfg, ss.zigzag_schedule(cfg), caches=caches)
    full, nbytes, ms = pair.consolidate(caches)
    assert nbytes > 0 and all(kv.k[0].device.index == 1 for kv in full)
    for i, kv in enumerate(full):
        tok = res.logits[i].argmax(-1).to("cuda:1")
        seq = torch.cat([batches[i].cpu(), tok.cpu()[:, None]], 1)
        with torch.cuda.device(1):
            lg = target.decode(tok, kv)
        _check(lg, forward_fp32(arch, ref_w, seq))
    tgt.close()
    src.close()


def test_decode_on_full_cache_raises_before_writing():
    """A decode step on a full cache must raise before anything is enqueued, and the
    cache panels (including the next panel in memory) must stay untouched."""
    arch = S.TINY_4L
    lay, slab, w = _slab(arch)
    ex = LlamaExecutor(w, max_tokens=2 * 8, device="cuda")
    prompt = _prompt(2, 8, 3, arch.vocab)
    kv = KVCache(arch, 2, 8, "cuda")          # room for the prompt only
    logits = ex.forward(prompt, kv=kv)
    torch.cuda.synchronize()
    before = {l: (kv.k[l].clone(), kv.v[l].clone()) for l in kv.k}
    with pytest.raises(ValueError, match="full"):
        ex.decode(logits.argmax(-1), kv)
    torch.cuda.synchronize()
    for l, (k0, v0) in before.items():
        assert torch.equal(kv.k[l], k0) and torch.equal(kv.v[l], v0)
    assert kv.length == 8 and int(kv.pos_dev.item()) == 8
    # the device kernels refuse too: rope_append at pos == s_max writes nothing
    import ctypes  # noqa: F401
    from paper_2412_17246_b200._native import cuda_lib
    a = arch
    qkv = torch.randn(2, a.d_model + 2 * a.kv_dim, device="cuda").to(torch.bfloat16)
    cuda_lib().bz_rope_append(qkv.data_ptr(), qkv.stride(0), 2, a.n_heads, a.n_kv_heads, a.head_dim,
                              a.rope_theta, kv.k[0].data_ptr(), kv.v[0].data_ptr(), kv.max_seq,
                              kv.pos_dev.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(kv.k[0], before[0][0]) and torch.equal(kv.v[0], before[0][1])
    slab.close()


def test_per_row_positions_continuous_batch():
    """Continuous batching: rows of one cache at different lengths decode in one step
    (bz_rope_append_rows / bz_decode_attention_rows), each row against its own fp32
    recompute; a graph over the first rows (rows_view) replays the same step."""
    arch = TINY_GQA
    lay, slab, w = _slab(arch)
    ref_w = weights_to_cpu_fp32(w)
    ex = LlamaExecutor(w, max_tokens=64, device="cuda")
    lens = [20, 12, 7]
    prompts = [_prompt(1, n, 30 + n, arch.vocab) for n in lens]
    kv = KVCache(arch, 4, 40, "cuda", per_row=True)          # 4 slots, slot 3 idle
    first = []
    for slot, p in enumerate(prompts):
        one = KVCache(arch, 1, 40, "cuda")
        lg = ex.forward(p, kv=one)
        first.append(lg.argmax(-1))
        for l in kv.k:
            kv.k[l][slot, :, :p.shape[1]].copy_(one.k[l][0, :, :p.shape[1]])
            kv.v[l][slot, :, :p.shape[1]].copy_(one.v[l][0, :, :p.shape[1]])
    kv.pos_dev.copy_(torch.tensor(lens + [0], dtype=torch.int32))
    toks = torch.cat(first + [torch.zeros(1, dtype=torch.int64, device="cuda")])
    logits = ex.decode(toks, kv)
    torch.cuda.synchronize()
    assert kv.pos_dev.tolist() == [n + 1 for n in lens] + [1]
    for slot, p in enumerate(prompts):
        seq = torch.cat([p.cpu(), first[slot].cpu()[:, None]], 1)
        _check(logits[slot:slot + 1], forward_fp32(arch, ref_w, seq))
    # the same step captured over the first 3 rows, replayed from the same positions
    kv.pos_dev.copy_(torch.tensor(lens + [0], dtype=torch.int32))
    view = kv.rows_view(3)
    g = ex.decode_graph(view)
    out = g(toks[:3])
    torch.cuda.synchronize()
    assert torch.equal(out, logits[:3]) or _rel(out.cpu(), logits[:3].cpu()) < 1e-3
    assert kv.pos_dev.tolist()[:3] == [n + 1 for n in lens]
    slab.close()
