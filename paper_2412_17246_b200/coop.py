"""ZigZag cooperative execution on real GPUs (cooperative-executor data path).

Reference: the layer split ``(T_i, S_i)`` of livescale.py:4-14 solved by
``configure_pipeline`` (livescale.py:113-181) and the target-side order
rehearsed by ``zigzag_schedule`` (livescale.py:269-346); PAPER.md:585-589,
786-895.  The reference only rehearses in abstract time units; this module
executes the rehearsal:

* the **target** (new instance, still receiving its slab) runs batch ``i``'s
  layers ``1..T_i`` in the rehearsed (batch, layer) order, each gated on the
  device readiness counter of its landing slab (``bz_wait_layer`` -- a
  stream-side wait, no spinning kernel), then hands the hidden state to the
  source (``bz_handoff``: a peer copy + release flag; K5 of SURVEY.md §2.2);
* the **source** (overloaded instance, full weights) waits for batch ``i``'s
  hand-off and runs layers ``T_i+1..L`` plus the LM head, FCFS (livescale.py:327-337).

Both instances may share one GPU (two streams, stream-ordered events) or sit
on two GPUs (handoff over NVLink into the source's buffer, cross-GPU flag).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from ._native import cuda_lib
from .livescale import PipelineConfig, ZigzagTimeline
from .dataplane import gate
from .llama import KVCache, LlamaExecutor


@dataclass
class CoopResult:
    logits: list[torch.Tensor]                 # per batch, fp32 [B, vocab]
    executed_order: list[tuple[int, int]]      # (batch, layer) as enqueued on the target
    handoff_bytes: int = 0
    source_ms: Optional[float] = None
    total_ms: Optional[float] = None
    finish_ms: Optional[list[float]] = None     # per batch, from the common start


class CooperativePair:
    """A (source, target) pair on this process's GPU(s).

    ``target_loaded`` is the target slab's device ``loaded_layers`` counter
    (``DeviceSlab.loaded``): the target's block ``k`` (1-based) is enqueued
    behind ``bz_wait_layer(target_loaded, k)``.
    """

    def __init__(self, source: LlamaExecutor, target: LlamaExecutor, target_loaded: torch.Tensor,
                 handoff_ctas: int = 16, fused_handoff: bool = True):
        self.src = source
        self.tgt = target
        self.loaded = target_loaded
        self.lib = cuda_lib()
        self.handoff_ctas = handoff_ctas
        # fused: the target's last down-projection GEMM stores straight into the
        # source's buffer (peer mapping) and signals; otherwise a bz_handoff copy
        self.fused = fused_handoff
        sdev = source.h.device
        tdev = target.h.device
        self.src_stream = torch.cuda.Stream(device=sdev)
        self.tgt_stream = torch.cuda.Stream(device=tdev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=sdev)
        self._handoffs = 0

    @torch.no_grad()
    def run(self, batches: Sequence[torch.Tensor], config: PipelineConfig,
            timeline: ZigzagTimeline, caches: Optional[list[tuple[KVCache, KVCache]]] = None) -> CoopResult:
        """Prefill every batch with its split; with ``caches`` (see ``make_caches``)
        each side keeps the keys/values of the blocks it ran, for ``decode``."""
        L = self.src.arch.n_layers
        n = len(batches)
        if config.batches != n:
            raise ValueError("one split per batch")
        shapes = [tuple(b.shape) for b in batches]
        pos = [torch.arange(s, dtype=torch.int32, device=b.device).repeat(bsz)
               for b, (bsz, s) in zip(batches, shapes)]
        x: list[Optional[torch.Tensor]] = [None] * n
        handed_at = [0] * n          # cumulative signal value that releases batch i
        recv: list[Optional[torch.Tensor]] = [None] * n
        for i, (t_i, _) in enumerate(config.splits):
            if t_i > 0:  # receive buffers live with the source
                recv[i] = torch.empty(batches[i].numel(), self.src.arch.d_model,
                                      dtype=torch.bfloat16, device=self.src.h.device)
        order: list[tuple[int, int]] = []
        nbytes = 0
        kv_t = [c[0] for c in caches] if caches else [None] * n
        kv_s = [c[1] for c in caches] if caches else [None] * n
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        start.record(cur)
        self.tgt_stream.wait_stream(cur)
        self.src_stream.wait_stream(cur)
        src_start = torch.cuda.Event(enable_timing=True)   # per-batch finish times, source-side clock
        src_start.record(self.src_stream)
        # ---- target: the rehearsed zigzag order, gated per layer -------------------------
        with torch.cuda.stream(self.tgt_stream):
            for b, layer, _s, _e in timeline.target_intervals:
                gate(self.loaded.data_ptr(), layer, self.tgt_stream.cuda_stream)
                if x[b] is None:  # the embedding table lives in unit 1: after its gate
                    x[b] = self.tgt.embed(batches[b])
                last = layer == config.splits[b][0]
                if last and self.fused:
                    # K5 fused into the GEMM epilogue: tiles land in the source's buffer
                    self.tgt.block(layer - 1, x[b], pos[b], shapes[b], out=recv[b], signal=self.flag,
                                   kv=kv_t[b])
                    self._handoffs += self.tgt.last_signal_ctas
                else:
                    x[b] = self.tgt.block(layer - 1, x[b], pos[b], shapes[b], kv=kv_t[b])
                    if last:
                        self.lib.bz_handoff(x[b].data_ptr(), recv[b].data_ptr(), x[b].numel() * 2,
                                            self.flag.data_ptr(), 0, self.handoff_ctas,
                                            self.tgt_stream.cuda_stream)
                        self._handoffs += self.handoff_ctas
                order.append((b, layer))
                if last:
                    nbytes += recv[b].numel() * 2
                    handed_at[b] = self._handoffs
                    if kv_t[b] is not None:
                        kv_t[b].length = shapes[b][1]

        # ---- source: suffixes FCFS, each gated on its hand-off counter -----------------------
        logits: list[Optional[torch.Tensor]] = [None] * n
        fin = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        with torch.cuda.stream(self.src_stream):
            for i in range(n):
                t_i, s_i = config.splits[i]
                if t_i == 0:
                    h = None
                else:
                    gate(self.flag.data_ptr(), handed_at[i], self.src_stream.cuda_stream)
                    h = recv[i]
                logits[i] = self.src.forward(batches[i], first=t_i, last=L, x=h, kv=kv_s[i])
                fin[i].record(self.src_stream)
        cur.wait_stream(self.src_stream)
        cur.wait_stream(self.tgt_stream)
        end.record(cur)
        end.synchronize()
        self._check_gates()
        return CoopResult(logits=logits, executed_order=order, handoff_bytes=nbytes,
                          total_ms=start.elapsed_time(end), finish_ms=[src_start.elapsed_time(e) for e in fin])

    def _check_gates(self):
        """A gate that timed out let its kernels run on data that never arrived: raise."""
        from .scaleup import check_wait_timeouts
        # only this pair's streams: a device-wide sync would also wait for the weight
        # transfer still streaming into the target on its own stream
        for st, dev in ((self.tgt_stream, self.tgt.h.device), (self.src_stream, self.src.h.device)):
            with torch.cuda.device(dev):
                st.synchronize()
        for dev in {self.tgt.h.device.index, self.src.h.device.index}:
            check_wait_timeouts(dev)

    def make_caches(self, batches: Sequence[torch.Tensor], config: PipelineConfig,
                    max_new_tokens: int) -> list[tuple[KVCache, KVCache]]:
        """Per batch: the target's cache for blocks [0, T_i) and the source's for
        [T_i, L), each sized for the prompt plus ``max_new_tokens``."""
        L = self.src.arch.n_layers
        out = []
        for b, (t_i, _) in zip(batches, config.splits):
            B, S = b.shape
            out.append((KVCache(self.tgt.arch, B, S + max_new_tokens, self.tgt.h.device, 0, t_i),
                        KVCache(self.src.arch, B, S + max_new_tokens, self.src.h.device, t_i, L)))
        return out

    @torch.no_grad()
    def decode(self, tokens: Sequence[torch.Tensor], config: PipelineConfig,
               caches: list[tuple[KVCache, KVCache]]) -> CoopResult:
        """One cooperative decode step per batch (tokens[i] int64 [B]): the target
        runs blocks [0, T_i) against its cache and hands the [B, d] hidden state to
        the source (fused into the last down-projection), which finishes blocks
        [T_i, L) and the head.  Only ``B*d*2`` bytes per batch cross."""
        L = self.src.arch.n_layers
        n = len(tokens)
        for kt, ks in caches[:n]:   # before anything is enqueued on either GPU
            kt.require_room()
            ks.require_room()
        recv: list[Optional[torch.Tensor]] = [None] * n
        handed_at = [0] * n
        nbytes = 0
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        start.record(cur)
        self.tgt_stream.wait_stream(cur)
        self.src_stream.wait_stream(cur)
        with torch.cuda.stream(self.tgt_stream):
            for i, (t_i, _) in enumerate(config.splits):
                if t_i == 0:
                    continue
                kv = caches[i][0]
                recv[i] = torch.empty(tokens[i].numel(), self.src.arch.d_model, dtype=torch.bfloat16,
                                      device=self.src.h.device)
                gate(self.loaded.data_ptr(), 1, self.tgt_stream.cuda_stream)   # embedding: unit 1
                x = self.tgt.embed(tokens[i])
                for k in range(t_i):
                    gate(self.loaded.data_ptr(), k + 1, self.tgt_stream.cuda_stream)
                    if k == t_i - 1 and self.fused:
                        self.tgt.decode_block(k, x, kv, out=recv[i], signal=self.flag)
                        self._handoffs += self.tgt.last_signal_ctas
                    else:
                        x = self.tgt.decode_block(k, x, kv)
                if not self.fused:
                    self.lib.bz_handoff(x.data_ptr(), recv[i].data_ptr(), x.numel() * 2, self.flag.data_ptr(), 0,
                                        self.handoff_ctas, self.tgt_stream.cuda_stream)
                    self._handoffs += self.handoff_ctas
                kv.advance()
                handed_at[i] = self._handoffs
                nbytes += recv[i].numel() * 2
        logits: list[Optional[torch.Tensor]] = [None] * n
        with torch.cuda.stream(self.src_stream):
            for i, (t_i, _) in enumerate(config.splits):
                h = None
                if t_i > 0:
                    gate(self.flag.data_ptr(), handed_at[i], self.src_stream.cuda_stream)
                    h = recv[i]
                logits[i] = self.src.decode(tokens[i], caches[i][1], first=t_i, last=L, x=h)
        cur.wait_stream(self.src_stream)
        cur.wait_stream(self.tgt_stream)
        end.record(cur)
        end.synchronize()
        self._check_gates()
        return CoopResult(logits=logits, executed_order=[], handoff_bytes=nbytes,
                          total_ms=start.elapsed_time(end))

    @torch.no_grad()
    def consolidate(self, caches: list[tuple[KVCache, KVCache]], nctas: int = 128
                    ) -> tuple[list[KVCache], int, float]:
        """Hand the sequences to the new instance once its weights are resident: the
        source's KV blocks [T_i, L) (their cached prefix only) are copied to the
        target's device (``bz_copy_panels``; NVLink when the pair spans two GPUs) and
        merged with the target's own [0, T_i) blocks, so the target decodes alone and
        the source is free (the KV hand-over the reference accounts as a flow,
        simcore.py:462-514).  Returns (full caches on the target, bytes moved, ms)."""
        tdev, sdev = self.tgt.h.device, self.src.h.device
        a = self.src.arch
        nbytes = 0
        out = []
        with torch.cuda.device(sdev):
            s = torch.cuda.current_stream(sdev)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(s)
            for kt, ks in caches:
                full = KVCache(self.tgt.arch, kt.batch, kt.max_seq, tdev, 0, 0)
                full.k.update(kt.k)
                full.v.update(kt.v)
                stride = kt.max_seq * a.head_dim * 2
                prefix = ks.length * a.head_dim * 2
                panels = kt.batch * a.n_kv_heads
                for layer in sorted(ks.k):
                    for side, dst_map in ((ks.k, full.k), (ks.v, full.v)):
                        dst = torch.empty_like(side[layer], device=tdev)
                        self.lib.bz_copy_panels(side[layer].data_ptr(), dst.data_ptr(), panels, stride, stride,
                                                prefix, nctas, s.cuda_stream)
                        dst_map[layer] = dst
                        nbytes += panels * prefix
                out.append(full)
            t1.record(s)
            t1.synchronize()
        for full, (kt, ks) in zip(out, caches):
            full.length = ks.length
        torch.cuda.synchronize(tdev)
        return out, nbytes, t0.elapsed_time(t1)

    def decode_graph(self, tokens: Sequence[torch.Tensor], config: PipelineConfig,
                     caches: list[tuple[KVCache, KVCache]]) -> "CoopDecodeGraph":
        """The cooperative decode step of ``decode`` captured once as a two-stream
        CUDA graph (target blocks -> graph edge -> source blocks + head, per batch):
        once a batch's prefix layers are resident no gate or hand-off counter is
        needed, and a replay costs no host work per kernel.  Source and target must
        share a device (one process, one GPU); ``decode`` covers the cross-GPU pair."""
        if self.src.h.device != self.tgt.h.device:
            raise NotImplementedError("graph capture of a cross-GPU pair: use decode()")
        return CoopDecodeGraph(self, tokens, config, caches)


class CoopDecodeGraph:
    def __init__(self, pair: CooperativePair, tokens: Sequence[torch.Tensor], config: PipelineConfig,
                 caches: list[tuple[KVCache, KVCache]]):
        self.pair, self.config, self.caches = pair, config, caches
        src, tgt = pair.src, pair.tgt
        dev = src.h.device
        self.tokens = [t.detach().clone() for t in tokens]
        self.recv = [torch.empty(t.numel(), src.arch.d_model, dtype=torch.bfloat16, device=dev)
                     for t in tokens]
        main, side = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        main.wait_stream(torch.cuda.current_stream(dev))
        saved = [(kt.length, ks.length) for kt, ks in caches]
        with torch.cuda.stream(main):
            self._step(main, side)          # warm-up outside capture (lazy library init)
            for (kt, ks), (lt, ls) in zip(caches, saved):
                kt.length, ks.length = lt, ls
            main.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=main):
                self.logits = self._step(main, side)
        torch.cuda.current_stream(dev).wait_stream(main)
        for (kt, ks), (lt, ls) in zip(caches, saved):
            kt._length, ks._length = lt, ls

    def _step(self, main, side):
        pair, L = self.pair, self.pair.src.arch.n_layers
        out = []
        side.wait_stream(main)
        for i, (t_i, _) in enumerate(self.config.splits):
            kt, ks = self.caches[i]
            h = None
            if t_i > 0:
                with torch.cuda.stream(side):       # target: blocks [0, T_i) into recv[i]
                    x = pair.tgt.embed(self.tokens[i])
                    for k in range(t_i):
                        x = pair.tgt.decode_block(k, x, kt, out=self.recv[i] if k == t_i - 1 else None)
                    kt.pos_dev.add_(1)
                main.wait_stream(side)
                h = self.recv[i]
            with torch.cuda.stream(main):           # source: blocks [T_i, L) + head
                x = h if h is not None else pair.src.embed(self.tokens[i])
                x = pair.src.decode_blocks(t_i, L, x, ks)   # as decode(): fused for <= 4 rows
                ks.pos_dev.add_(1)
                out.append(pair.src.head(x, (x.shape[0], 1)))
        main.wait_stream(side)
        return out

    def __call__(self, tokens: Sequence[torch.Tensor]) -> list[torch.Tensor]:
        if any(ks.length >= ks.max_seq for _, ks in self.caches):
            raise ValueError("KV cache full")
        for buf, t in zip(self.tokens, tokens):
            buf.copy_(t)
        self.graph.replay()
        for (t_i, _), (kt, ks) in zip(self.config.splits, self.caches):
            if t_i > 0:
                kt._length += 1
            ks._length += 1
        return self.logits
