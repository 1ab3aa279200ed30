"""Measured pair-throughput ramp: the executed counterpart of the reference's
``steady_state_throughput`` (livescale.py:349-363) and of the simulator's
``_prefill_rate_factor`` (simcore.py:408-417).

With ``k`` of ``L`` layers resident on the new instance, a cooperating pair runs
every batch's first ``k`` layers on the target and the rest on the source, in
the ZigZag order; in steady state a batch completes every max(k, L - k)
layer-times.  Here the pair is real (two GPUs, tcgen05 GEMMs, fused NVLink
hand-off): the same (k, L - k) split for every batch, the target's gates open,
and the throughput is taken over the second half of the batches exactly as the
reference rehearsal does.  Measured for 0 <= k <= L/2 (source-bound side).
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import livescale
from ._native import cuda_lib
from .coop import CooperativePair
from .dataplane import DeviceSlab
from .llama import LlamaExecutor, SlabWeights
from .slab import LlamaArch, SlabLayout


def measure_ramp(arch: LlamaArch, src_dev: int = 0, tgt_dev: int = 1, ks: Sequence[int] | None = None,
                 batches: int = 16, seqs: int = 1, seq_len: int = 2000, tile_bytes: int = 1 << 20) -> dict:
    """Measured and reference pair throughput for each loaded-layer count ``k``.

    Returns ``{"points": [{"k", "measured_batches_per_s", "measured_rel",
    "reference_rel"}...], ...}`` where ``*_rel`` is the throughput relative to the
    source alone (k = 0); the reference column is ``steady_state_throughput``.
    """
    L = arch.n_layers
    # k <= L/2: the source-bound side the reference's formula describes (1/(L - k));
    # configure_pipeline's C2 (cumulative prefixes <= suffixes, livescale.py:93-110)
    # keeps uniform splits at k <= L/3, so the planner never schedules k > L/2
    ks = list(ks) if ks is not None else sorted(set(list(range(0, L // 2 + 1, max(1, L // 16))) + [L // 2]))
    if any(not 0 <= k <= L // 2 for k in ks):
        raise ValueError("the ramp is measured for 0 <= k <= L/2")
    lay = SlabLayout.for_arch(arch, tile_bytes=tile_bytes)
    for d in (src_dev, tgt_dev):
        cuda_lib(d).bz_enable_peer_mesh(d)   # the target's GEMM stores the hand-off into the source
    slabs = []
    try:
        for d in (src_dev, tgt_dev):
            with torch.cuda.device(d):
                s = DeviceSlab(lay, d)
                SlabWeights(arch, lay, s.data).init_random(seed=0)
                slabs.append(s)
        src, tgt = slabs
        with torch.cuda.device(tgt_dev):
            tgt.loaded.fill_(L)  # every layer resident: the ramp isolates the split
        torch.cuda.synchronize(tgt_dev)
        tokens = seqs * seq_len
        ex0 = LlamaExecutor(SlabWeights(arch, lay, src.data), tokens, torch.device("cuda", src_dev))
        ex1 = LlamaExecutor(SlabWeights(arch, lay, tgt.data), tokens, torch.device("cuda", tgt_dev))
        pair = CooperativePair(ex0, ex1, tgt.loaded)
        g = torch.Generator().manual_seed(5)
        toks = [torch.randint(0, arch.vocab, (seqs, seq_len), generator=g).to(f"cuda:{src_dev}")
                for _ in range(batches)]
        half = batches // 2
        points = []
        ref0 = livescale.steady_state_throughput(L, 0)
        meas0 = None
        # one untimed source-alone pass first: the first split measured must not
        # pay the clock ramp and lazy module loads (they depress k = 0 and make the
        # later splits look super-linear)
        with torch.cuda.device(src_dev):
            cfg0 = livescale.PipelineConfig([(0, L)] * batches, L, 0.0, [1.0] * batches)
            pair.run(toks, cfg0, livescale.zigzag_schedule(cfg0, [0.0] * L))
        for k in ks:
            cfg = livescale.PipelineConfig([(k, L - k)] * batches, L, 0.0, [1.0] * batches)
            tl = livescale.zigzag_schedule(cfg, [0.0] * L)
            with torch.cuda.device(src_dev):
                pair.run(toks[:2], livescale.PipelineConfig([(k, L - k)] * 2, L, 0.0, [1.0] * 2),
                         livescale.zigzag_schedule(livescale.PipelineConfig([(k, L - k)] * 2, L, 0.0, [1.0] * 2),
                                                   [0.0] * L))          # warm this split
                best = None
                for _ in range(3):
                    res = pair.run(toks, cfg, tl)
                    f = res.finish_ms
                    rate = (batches - half) / ((f[-1] - f[half - 1]) / 1e3)
                    best = rate if best is None else max(best, rate)
            if k == 0:
                meas0 = best
            points.append({"k": k, "measured_batches_per_s": best,
                           "reference_rel": livescale.steady_state_throughput(L, k) / ref0})
        for p in points:
            p["measured_rel"] = p["measured_batches_per_s"] / meas0 if meas0 else None
        return {"model": arch.name, "layers": L, "batches": batches, "tokens_per_batch": tokens,
                "window": f"batches {half + 1}..{batches} (as steady_state_throughput)", "points": points}
    finally:
        torch.cuda.synchronize(src_dev)
        torch.cuda.synchronize(tgt_dev)
        for s in slabs:
            s.close()
