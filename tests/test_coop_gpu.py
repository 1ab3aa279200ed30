"""Cooperative (ZigZag) execution on the GPU vs the fp32 CPU oracle.

Tolerance (north star): max relative error of logits <= 1e-2 (max-normalised)
and identical greedy tokens, for a Llama-style model whose weights live in
layer slabs; the split comes from configure_pipeline and the target order
from zigzag_schedule, exactly as the reference computes them.
"""

import pytest
import torch

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.coop import CooperativePair
from paper_2412_17246_b200.dataplane import DeviceSlab, Fabric, HostCache, ScaleExecutor, execute_plan_loopback
from paper_2412_17246_b200.llama import LlamaExecutor, SlabWeights
from oracle.forward_ref import forward_fp32, weights_to_cpu_fp32

pytestmark = pytest.mark.gpu

ARCH = S.TINY_4L


def _rel(a, b):
    return ((a - b).abs().max() / (b.abs().max() + 1e-6)).item()


def _check_logits(got, want):
    assert _rel(got.cpu(), want) <= 1e-2
    top2 = want.topk(2, dim=-1).values
    margin_ok = (top2[:, 0] - top2[:, 1]) > 2e-2 * want.abs().max()
    # greedy tokens identical wherever the oracle's top-2 margin exceeds the tolerance
    assert torch.equal(got.cpu().argmax(-1)[margin_ok], want.argmax(-1)[margin_ok])


@pytest.fixture(scope="module")
def model():
    lay = S.SlabLayout.for_arch(ARCH, tile_bytes=128 * 1024)
    src = DeviceSlab(lay, 0)
    w = SlabWeights(ARCH, lay, src.data)
    w.init_random(seed=0)
    torch.cuda.synchronize()
    yield lay, src, w, weights_to_cpu_fp32(w)
    src.close()


def _tokens(n, b, s, seed):
    g = torch.Generator().manual_seed(seed)
    return [torch.randint(0, ARCH.vocab, (b, s), generator=g).cuda() for _ in range(n)]


def test_unsplit_forward_matches_oracle(model):
    lay, src, w, ref_w = model
    ex = LlamaExecutor(w, max_tokens=4 * 64, device="cuda")
    toks = _tokens(1, 4, 64, 1)[0]
    logits = ex.forward(toks)
    torch.cuda.synchronize()
    _check_logits(logits, forward_fp32(ARCH, ref_w, toks.cpu()))


@pytest.mark.parametrize("n,time_l", [(4, 1.0), (6, 0.5), (3, 2.0)])
def test_zigzag_split_matches_oracle(model, n, time_l):
    lay, src, w, ref_w = model
    tgt = DeviceSlab(lay, 0)
    plan = ss.generate_plan(
        ss.build_scale_request(S.model_spec_for(ARCH), ["gpu0"], ["gpu1"],
                               ss.load_topology("b200-hgx"), ss.FlowSet(ss.load_topology("b200-hgx"))),
        ss.load_topology("b200-hgx"), ss.FlowSet(ss.load_topology("b200-hgx")))
    execute_plan_loopback(plan, {"gpu0": src, "gpu1": tgt}, epoch=1)
    torch.cuda.synchronize()
    cfg = ss.configure_pipeline(n, ARCH.n_layers, time_l)
    tl = ss.zigzag_schedule(cfg)
    source = LlamaExecutor(w, max_tokens=2 * 32, device="cuda")
    target = LlamaExecutor(SlabWeights(ARCH, lay, tgt.data), max_tokens=2 * 32, device="cuda")
    pair = CooperativePair(source, target, tgt.loaded)
    batches = _tokens(n, 2, 32, 7)
    res = pair.run(batches, cfg, tl)
    assert res.executed_order == [(b, k) for b, k, _, _ in tl.target_intervals]
    assert res.handoff_bytes == sum(2 * 32 * ARCH.d_model * 2 for t, _ in cfg.splits if t > 0)
    for b, logits in zip(batches, res.logits):
        _check_logits(logits, forward_fp32(ARCH, ref_w, b.cpu()))
    tgt.close()


@pytest.mark.multigpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_cross_gpu_zigzag_handoff_over_nvlink(model):
    """Source on cuda:0, target on cuda:1 loading from the host cache; the hidden
    states cross NVLink through bz_handoff (peer access), logits vs the oracle."""
    from paper_2412_17246_b200._native import cuda_lib
    lay, src, w, ref_w = model
    lib = cuda_lib()
    lib.bz_enable_peer_mesh(0)
    lib.bz_enable_peer_mesh(1)
    hc = HostCache(lay)
    hc.tensor.copy_(src.data.cpu())
    with torch.cuda.device(1):
        tgt = DeviceSlab(lay, 1)
        plan = ss.ScalePlan(edges=[ss.planner.PlanEdge("mem0", "gpu1", 512.0, "pcie")],
                            chains=[["mem0", "gpu1"]])
        ex = ScaleExecutor(Fabric(1), plan, tgt, {"gpu1": 0}, host_cache=hc)
        target = LlamaExecutor(SlabWeights(ARCH, lay, tgt.data), max_tokens=64, device="cuda:1")
    source = LlamaExecutor(w, max_tokens=64, device="cuda:0")
    cfg = ss.configure_pipeline(4, ARCH.n_layers, 1.0)
    tl = ss.zigzag_schedule(cfg)
    pair = CooperativePair(source, target, tgt.loaded)
    batches = _tokens(4, 2, 32, 13)
    with torch.cuda.device(1):
        ex.launch()
    res = pair.run(batches, cfg, tl)
    ex.synchronize()
    for b, logits in zip(batches, res.logits):
        assert logits.device.index == 0
        _check_logits(logits, forward_fp32(ARCH, ref_w, b.cpu()))
    ex.close()
    hc.close()
    tgt.close()


def test_serving_overlaps_host_staging(model):
    """Target slab streams in from the pinned host cache (copy engines, per-layer
    publish) while the cooperative pair is already executing layer-gated work."""
    lay, src, w, ref_w = model
    fabric = Fabric(0)
    hc = HostCache(lay)
    hc.tensor.copy_(src.data.cpu())
    tgt = DeviceSlab(lay, 0)
    plan = ss.ScalePlan(edges=[ss.planner.PlanEdge("mem0", "gpu0", 512.0, "pcie")],
                        chains=[["mem0", "gpu0"]])
    ex = ScaleExecutor(fabric, plan, tgt, {"gpu0": 0}, host_cache=hc)
    cfg = ss.configure_pipeline(4, ARCH.n_layers, 1.0)
    tl = ss.zigzag_schedule(cfg)
    source = LlamaExecutor(w, max_tokens=64, device="cuda")
    target = LlamaExecutor(SlabWeights(ARCH, lay, tgt.data), max_tokens=64, device="cuda")
    pair = CooperativePair(source, target, tgt.loaded)
    batches = _tokens(4, 2, 32, 11)
    ex.launch()                      # staging runs on its own stream
    res = pair.run(batches, cfg, tl)  # target work waits on each layer's publish
    ex.synchronize()
    assert torch.equal(tgt.data, src.data)
    for b, logits in zip(batches, res.logits):
        _check_logits(logits, forward_fp32(ARCH, ref_w, b.cpu()))
    ex.close()
    hc.close()
    tgt.close()


def test_target_embedding_waits_for_unit_one(model):
    """The target's first work item reads the embedding table, which lives in unit 1:
    with a target slab full of garbage and its readiness counter at 0, nothing may read
    it before the gate opens (logits still match once the weights land late)."""
    lay, src, w, ref_w = model
    tgt = DeviceSlab(lay, 0)
    tgt.data.fill_(0xFF)                       # NaN bf16 everywhere until the load lands
    tgt.loaded.zero_()
    cfg = ss.configure_pipeline(2, ARCH.n_layers, 1.0)
    tl = ss.zigzag_schedule(cfg)
    pair = CooperativePair(LlamaExecutor(w, max_tokens=64, device="cuda"),
                           LlamaExecutor(SlabWeights(ARCH, lay, tgt.data), max_tokens=64, device="cuda"),
                           tgt.loaded)
    batches = _tokens(2, 2, 32, 17)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)          # the weights land ~tens of ms after the pair starts
        tgt.data.copy_(src.data)
        tgt.loaded.fill_(ARCH.n_layers)
    res = pair.run(batches, cfg, tl)
    torch.cuda.synchronize()
    for b, logits in zip(batches, res.logits):
        _check_logits(logits, forward_fp32(ARCH, ref_w, b.cpu()))
    tgt.close()
