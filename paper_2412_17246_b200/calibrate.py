"""Measure the B200 costs the serving replay needs (prefill line, layer arrivals).

``measure_prefill`` times real Llama prefill passes of the tcgen05 executor
(one block at each token count, scaled by the layer count, plus the head),
``measure_decode`` times KV-cache decode steps the same way, and
``c3_report`` replays the C3 burst trace through ``simcore`` twice -- with the
reference's analytic costs and with the measured ones -- for each strategy.
"""

from __future__ import annotations

import time
from typing import Optional, Sequence

import torch

from .costs import MeasuredCosts, fit_line
from .slab import LlamaArch, SlabLayout


def measure_prefill(arch: LlamaArch, token_counts: Sequence[int] = (256, 512, 1024, 2048),
                    seq_len: int = 512, iters: int = 5, device: int = 0) -> dict:
    """ms of a full-model prefill at each token count (B sequences of <= seq_len)."""
    from .dataplane import DeviceSlab
    from .llama import LlamaExecutor, SlabWeights

    probe = LlamaArch(arch.name + "-probe", arch.d_model, 1, arch.n_heads, arch.n_kv_heads,
                      arch.ffn, arch.vocab, arch.norm_eps, arch.rope_theta)
    lay = SlabLayout.for_arch(probe, tile_bytes=1 << 20)
    slab = DeviceSlab(lay, device)
    w = SlabWeights(probe, lay, slab.data)
    w.init_random(seed=0)
    ex = LlamaExecutor(w, max_tokens=max(token_counts), device=torch.device("cuda", device))
    out = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for n in token_counts:
        s = min(seq_len, n)
        b = max(1, n // s)
        toks = torch.randint(0, arch.vocab, (b, s), device=f"cuda:{device}")
        pos = torch.arange(s, dtype=torch.int32, device=toks.device).repeat(b)
        x = ex.embed(toks)
        for _ in range(2):
            ex.block(0, x, pos, (b, s))
            ex.head(x, (b, s))
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(iters):
            ex.block(0, x, pos, (b, s))
        ev[1].record()
        for _ in range(iters):
            ex.head(x, (b, s))
        ev[2].record()
        ev[2].synchronize()
        block_ms = ev[0].elapsed_time(ev[1]) / iters
        head_ms = ev[1].elapsed_time(ev[2]) / iters
        out[b * s] = block_ms * arch.n_layers + head_ms
    slab.close()
    return out


def measure_decode(arch: LlamaArch, batches: Sequence[int] = (1, 8, 32, 64), context: int = 1024,
                   iters: int = 20, device: int = 0, probe_layers: int = 8, warmup: int = 5,
                   trials: int = 3) -> dict:
    """ms of one full-model decode step for ``b`` sequences at ``context`` cached
    tokens each: ``probe_layers`` distinct blocks captured as one CUDA graph (as
    served), replayed from position ``context`` on and scaled to the layer count,
    plus the head timed separately."""
    from .dataplane import DeviceSlab
    from .llama import KVCache, LlamaExecutor, SlabWeights

    nl = min(probe_layers, arch.n_layers)
    probe = LlamaArch(arch.name + "-probe", arch.d_model, nl, arch.n_heads, arch.n_kv_heads,
                      arch.ffn, arch.vocab, arch.norm_eps, arch.rope_theta)
    lay = SlabLayout.for_arch(probe, tile_bytes=1 << 20)
    slab = DeviceSlab(lay, device)
    w = SlabWeights(probe, lay, slab.data)
    w.init_random(seed=0)
    dev = torch.device("cuda", device)
    ex = LlamaExecutor(w, max_tokens=max(batches), device=dev)
    out = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for b in batches:
        kv = KVCache(probe, b, context + warmup + iters + 2, dev)
        for t in list(kv.k.values()) + list(kv.v.values()):
            t.normal_(0, 1)
        kv.length = context
        step = ex.decode_graph(kv, 0, nl, hidden_in=True, head=False)
        step.hidden.normal_(0, 1)
        x = step.hidden
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        # best of `trials` timed runs (the first graph replays of a fresh process
        # can run slow while clocks and caches settle)
        per_block = float("inf")
        for _ in range(trials):
            kv.length = context
            ev[0].record()
            for _ in range(iters):
                step()
            ev[1].record()
            ev[1].synchronize()
            per_block = min(per_block, ev[0].elapsed_time(ev[1]) / iters / nl)
        ev[1].record()
        for _ in range(iters):
            ex.head(x, (b, 1))
        ev[2].record()
        ev[2].synchronize()
        out[b] = per_block * arch.n_layers + ev[1].elapsed_time(ev[2]) / iters
        del step, kv
    slab.close()
    return out


def measure_ssd_load(nbytes: int = 2 << 30, chunk: int = 64 << 20, directory: str = "/tmp",
                     device: int = 0) -> dict:
    """The ServerlessLLM miss path on this box, run by the real mechanism
    (``diskload.DiskSlabLoader``): a shard image of ``nbytes`` (32 layer units) written
    to local storage, then streamed with O_DIRECT through two pinned buffers into a
    GPU slab with per-layer publish, checked bit-exact.  Returns the disk-only and the
    disk -> HBM rates (GB/s)."""
    import os
    import tempfile

    from .dataplane import DeviceSlab
    from .diskload import DiskSlabLoader, write_slab_image

    lay = SlabLayout.uniform(32, nbytes // 32)
    src, dst = DeviceSlab(lay, device), DeviceSlab(lay, device)
    d = tempfile.mkdtemp(dir=directory, prefix="blitz_ssd_")
    path = os.path.join(d, "shard.img")
    try:
        src.fill_random(seed=5)
        write_slab_image(src.data, path, chunk=chunk)
        res = DiskSlabLoader(lay, path, device, chunk=chunk).load(dst, epoch=1)
        exact = bool(torch.equal(dst.fingerprints().cpu(), src.fingerprints().cpu()))
    finally:
        if os.path.exists(path):
            os.unlink(path)
        os.rmdir(d)
        src.close()
        dst.close()
    return {"bytes": int(res["bytes"]), "disk_read_GBps": res["disk_read_GBps"],
            "ssd_to_gpu_GBps": res["ssd_to_gpu_GBps"], "bit_exact": exact,
            "first_layer_ms": res["layer_ms"][0],
            "method": "diskload.DiskSlabLoader: O_DIRECT reads of a %d MiB slab image into 2 pinned %d MiB "
                      "buffers, H2D overlapped, per-layer publish" % (nbytes >> 20, chunk >> 20)}


def build_costs(prefill: Optional[dict] = None, nvlink_layer_ms=None, host_layer_ms=None,
                source: Optional[dict] = None, decode: Optional[dict] = None,
                ssd_gbs: Optional[float] = None) -> MeasuredCosts:
    a = b = da = db = None
    if prefill:
        xs = sorted(prefill)
        a, b = fit_line(xs, [prefill[x] for x in xs])
    if decode:
        xs = sorted(decode)
        da, db = fit_line(xs, [decode[x] for x in xs])
    return MeasuredCosts(prefill_alpha_ms=a, prefill_beta_ms=b, nvlink_layer_ms=nvlink_layer_ms,
                         host_layer_ms=host_layer_ms, decode_alpha_ms=da, decode_beta_ms=db,
                         ssd_to_gpu_gbs=ssd_gbs, source=source or {})


def c3_report(costs: MeasuredCosts, topo_name: str = "b200-hgx-2x8",
              strategies: Sequence[str] = ("blitz-live", "blitz-stop", "allcache", "sllm"),
              executed: Optional[MeasuredCosts] = None) -> dict:
    """C3: Llama-2 7B under the 5x-burst trace; p99 TTFT/TBT with modeled and measured costs."""
    from . import simcore
    from .slab import LLAMA2_7B, model_spec_for
    from .topology import load_topology
    from .traces import generate_trace

    trace = generate_trace("burst", {"rate_per_s": 20, "duration_s": 30, "prompt_tokens": [512, 2048],
                                     "output_tokens": [16, 128],
                                     "bursts": [{"start_s": 10, "duration_s": 2, "multiplier": 5}]},
                           seed=1)
    spec = model_spec_for(LLAMA2_7B)
    topo = load_topology(topo_name)
    out = {"trace": f"burst 20 req/s x 30 s, 5x for 2 s at t=10 s, seed 1 ({len(trace)} requests)",
           "topology": topo_name, "model": spec.name, "costs": costs.describe(), "strategies": {}}
    for strat in strategies:
        row = {}
        # executed: every scale-up the replay plans is run by the data plane in this
        # process and its layer / transfer events are the device stamps (inprocess.py)
        providers = [("modeled", simcore.ReferenceCosts()), ("measured", costs)]
        if executed is not None:
            providers.append(("executed", executed))
        for label, c in providers:
            t0 = time.perf_counter()
            res = simcore.run_simulation(topo, [spec], trace, simcore.SimPolicy(strategy=strat), costs=c)
            s = res.summary()
            row[label] = {"p99_ttft_ms": s["ttft_ms"]["p99"], "p50_ttft_ms": s["ttft_ms"]["p50"],
                          "p99_tbt_ms": s["tbt_ms"]["p99"], "slo_attainment": s["slo_attainment"],
                          "scale_ups": s["counters"]["scale_ups"],
                          "replay_cpu_s": time.perf_counter() - t0}
        out["strategies"][strat] = row
    if executed is not None:
        out["executed_costs"] = executed.describe()
    return out
