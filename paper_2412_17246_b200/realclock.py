"""C3 on the real clock: a bursty trace served by real Llama-2 7B prefills on two
B200s, with the scale-up executed by the data plane while requests queue.

The reference answers "p99 TTFT under a 5x burst" by replaying the trace through
its event simulator with modeled costs (simcore.py, autoscaler.py:53-59,
PAPER.md:1178-1221).  Here nothing is modeled: requests arrive on the host's
wall clock, every prefill is a real forward pass of the slab-resident model
(tcgen05 GEMMs), the scale trigger is the reference policy
(``should_scale_up`` on a windowed arrival rate against the measured instance
capacity) and the new instance's weights move for real:

* ``blitz``    -- the plan's NVLink hop from the live source (``bz_push_tiles``),
  the new instance serving once the tracker publishes the last layer;
* ``allcache`` -- stop-the-world O(1) host-cache load over PCIe
  (``bz_stage_tiles_ce``), the AllCache baseline;
* ``live-host`` -- the same host-cache load, but while it runs the two GPUs serve
  queued requests as a ZigZag pair (``CooperativePair``: split by
  ``configure_pipeline`` with the measured time_l, order by ``zigzag_schedule``,
  target layers gated on the readiness counter, fused NVLink hand-off);
* ``static``   -- no scaling.

With ``decode_slots`` > 0 every instance also decodes what it prefilled
(continuous batching, per-row device positions: ``bz_rope_append_rows`` /
``bz_decode_attention_rows``): a prefill's keys/values land in a staging cache
inside its captured graph and are copied into a free slot of the instance's
decode cache (``bz_copy_panels``); decode steps replay one captured graph over
the first 4/8/16/32 slots, alternating with prefills when both are pending; each
request emits its trace's output tokens and TBT is the host-observed time between
its tokens.

One process drives every GPU (peer access on); prompts are padded to 256-token
buckets whose forward passes are captured as CUDA graphs.  With more than one
target GPU the trigger adds as many instances as the policy asks for at once:
``blitz`` moves the weights down a chain source -> t1 -> t2 ... on the copy engines
(the data plane's chain mover: 256-tile groups, each relay forwarding a group once its
flags land; the serving source spends no SM), the plan's grouped NVLink fan-out
realised as a sibling chain,
``allcache`` stages every new instance from the host copy in parallel.  TTFT = host time at
which the request's prefill completion event is observed minus its arrival time.
"""

from __future__ import annotations

import collections
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from ._native import cuda_lib
from . import livescale
from .autoscaler import LoadMetrics, ScalePolicy, should_scale_up
from .coop import CooperativePair
from .dataplane import CE_CHAIN_TILES_PER_COPY, DeviceSlab, HostCache, PeerSlab
from .llama import KVCache, LlamaExecutor, SlabWeights
from .slab import LlamaArch, SlabLayout


@dataclass
class Req:
    rid: int
    t_arrive: float
    n_tok: int
    t_done: Optional[float] = None
    served_by: str = ""
    n_out: int = 0                      # output tokens (the first comes from the prefill)
    token_t: list = field(default_factory=list)   # host time of every decode token
    slot: int = -1


@dataclass
class _Instance:
    name: str
    device: torch.device
    ex: LlamaExecutor
    stream: torch.cuda.Stream
    ready: bool
    busy: Optional[tuple] = None   # (kind, payload, event): ("prefill", req) | ("decode", [req...])
    key: str = ""
    active: dict = field(default_factory=dict)   # decode slot -> request
    last: str = ""


@dataclass
class RealClockResult:
    strategy: str
    n: int
    p50_ttft_ms: float
    p99_ttft_ms: float
    mean_ttft_ms: float
    scale_trigger_s: Optional[float]
    scale_ready_s: Optional[float]
    load_ms: Optional[float]
    served: dict = field(default_factory=dict)
    wall_s: float = 0.0
    pair_runs: list = field(default_factory=list)   # live-host: (start s, splits, host ms)
    instances_added: int = 0
    all_ready_s: Optional[float] = None             # every added instance serving
    p50_tbt_ms: Optional[float] = None              # decode_slots > 0: time between a request's tokens
    p99_tbt_ms: Optional[float] = None
    decode_steps: int = 0


def _pct(xs, q):
    ys = sorted(xs)
    if not ys:
        return 0.0
    k = min(len(ys) - 1, max(0, int(round(q / 100.0 * (len(ys) - 1)))))
    return ys[k]


class RealClockServer:
    """Source instance on ``src_dev`` (weights resident); the scale target on
    ``tgt_dev`` starts empty."""

    DECODE_GRAPH_ROWS = (4, 8, 16, 32)

    def __init__(self, arch: LlamaArch, src_dev: int = 0, tgt_dev: int = 1, tile_bytes: int = 1 << 20,
                 extra_devs: Sequence[int] = (), decode_slots: int = 0,
                 max_new_tokens: int = 128):
        self.arch = arch
        if decode_slots and decode_slots not in self.DECODE_GRAPH_ROWS:
            raise ValueError(f"decode_slots must be one of {self.DECODE_GRAPH_ROWS}")
        self.decode_slots = decode_slots
        self.s_max = self.BUCKETS[-1] + max_new_tokens + 1
        self.lib = cuda_lib(src_dev)
        self.tgt_devs = [tgt_dev] + [d for d in extra_devs if d not in (src_dev, tgt_dev)]
        for d in [src_dev] + self.tgt_devs:
            cuda_lib(d)
            self.lib.bz_enable_peer_mesh(d)
        self.layout = SlabLayout.for_arch(arch, tile_bytes=tile_bytes)
        self.src_dev, self.tgt_dev = src_dev, tgt_dev
        with torch.cuda.device(src_dev):
            self.src = DeviceSlab(self.layout, src_dev)
            SlabWeights(arch, self.layout, self.src.data).init_random(seed=0)
            torch.cuda.synchronize()
            self.host = HostCache(self.layout)
            self.host.tensor.copy_(self.src.data.cpu())
        self.tslabs = []
        for d in self.tgt_devs:
            with torch.cuda.device(d):
                self.tslabs.append(DeviceSlab(self.layout, d))
        self.tgt = self.tslabs[0]
        # target slabs are VMM allocations: a sender reaches one through its own mapping
        # of the exported handle (as a peer process would), not the owner's VA.  Chain
        # hops: source -> any target (a group's head), target j -> target j+1 (relay)
        self.peer_on_src = [PeerSlab(src_dev, *t.export(), self.layout) for t in self.tslabs]
        self.tgt_on_src = self.peer_on_src[0]
        self.peer_next = [PeerSlab(self.tgt_devs[j], *self.tslabs[j + 1].export(), self.layout)
                          for j in range(len(self.tslabs) - 1)]
        self.max_tokens = 4096
        d0 = torch.device("cuda", src_dev)
        self.ex0 = LlamaExecutor(SlabWeights(arch, self.layout, self.src.data), self.max_tokens, d0)
        self.s0 = torch.cuda.Stream(device=d0)
        self.push_stream = torch.cuda.Stream(device=d0)
        self.push_flag_stream = torch.cuda.Stream(device=d0)
        self.tex, self.ts, self.tload, self.tpush, self.tflag, self.tgate = [], [], [], [], [], []
        for d, t in zip(self.tgt_devs, self.tslabs):
            dev = torch.device("cuda", d)
            self.tex.append(LlamaExecutor(SlabWeights(arch, self.layout, t.data), self.max_tokens, dev))
            self.ts.append(torch.cuda.Stream(device=dev))
            self.tload.append(torch.cuda.Stream(device=dev))
            self.tpush.append(torch.cuda.Stream(device=dev))
            self.tflag.append(torch.cuda.Stream(device=dev))
            self.tgate.append(torch.cuda.Stream(device=dev))
        self.ex1, self.s1, self.load_stream = self.tex[0], self.ts[0], self.tload[0]
        self.epoch = 0
        self._warm()
        self.graphs = {}
        plan = [("src", self.ex0, self.s0, self.src_dev)] + [
            (f"t{j}", ex, st, d) for j, (ex, st, d) in enumerate(zip(self.tex, self.ts, self.tgt_devs))]
        self.staging, self.dcache, self.dgraphs = {}, {}, {}
        for name, ex, st, dev in plan:
            for bucket in self.BUCKETS:
                stage = None
                if decode_slots:
                    # the prompt's keys/values land here inside the captured prefill
                    stage = KVCache(arch, 1, bucket, torch.device("cuda", dev))
                    self.staging[(name, bucket)] = stage
                self.graphs[(name, bucket)] = self._capture(ex, st, dev, bucket, stage)
            if decode_slots:
                with torch.cuda.device(dev), torch.cuda.stream(st):
                    kv = KVCache(arch, decode_slots, self.s_max, torch.device("cuda", dev), per_row=True)
                    self.dcache[name] = kv
                    for n in self.DECODE_GRAPH_ROWS:
                        if n <= decode_slots:
                            self.dgraphs[(name, n)] = ex.decode_graph(kv.rows_view(n))
                st.synchronize()
        d1 = torch.device("cuda", tgt_dev)
        self.pair = CooperativePair(self.ex0, self.ex1, self.tgt.loaded)
        self.pair_tokens = {b: torch.randint(0, arch.vocab, (1, b), device=d0) for b in self.BUCKETS}
        # warm the pair's own streams (library plans such as cuDNN SDPA are per stream:
        # a cold stream costs 100+ ms on first use) with every bucket, gates open
        with torch.cuda.device(tgt_dev):
            self.tgt.loaded.fill_(arch.n_layers)
        torch.cuda.synchronize(tgt_dev)
        for b in self.BUCKETS:
            cfg = livescale.configure_pipeline(2, arch.n_layers, 1.0)
            with torch.cuda.device(src_dev):
                self.pair.run([self.pair_tokens[b]] * 2, cfg, livescale.zigzag_schedule(cfg))
        with torch.cuda.device(d1):
            self.tgt.loaded.zero_()
        torch.cuda.synchronize(tgt_dev)

    # prompts are padded up to a bucket and each bucket's forward is one CUDA graph,
    # so the single host thread that drives both GPUs spends ~10 us per prefill
    BUCKETS = (512, 768, 1024, 1280, 1536, 1792, 2048)

    @staticmethod
    def bucket(n: int) -> int:
        for b in RealClockServer.BUCKETS:
            if n <= b:
                return b
        return RealClockServer.BUCKETS[-1]

    def _capture(self, ex, stream, dev, n, kv=None):
        with torch.cuda.device(dev):
            toks = torch.randint(0, self.arch.vocab, (1, n), device=f"cuda:{dev}")
            with torch.cuda.stream(stream):
                ex.forward(toks, kv=kv)
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                ex.forward(toks, kv=kv)
        return g

    def _admit(self, inst, req, bucket: int):
        """Enqueue (on the instance's stream, after its prefill) the copy of the prompt's
        keys/values from the bucket's staging cache into a free decode slot, and set that
        slot's device position to the prompt length."""
        kv = self.dcache[inst.key]
        slot = min(set(range(self.decode_slots)) - set(inst.active))
        req.slot = slot
        inst.active[slot] = req
        stage = self.staging.get((inst.key, bucket))
        a = self.arch
        n = min(req.n_tok, bucket) if stage is not None else min(req.n_tok, self.s_max - req.n_out - 1)
        with torch.cuda.device(inst.device), torch.cuda.stream(inst.stream):
            s = inst.stream.cuda_stream
            if stage is not None:
                for l in kv.k:
                    for src, dst in ((stage.k[l], kv.k[l][slot]), (stage.v[l], kv.v[l][slot])):
                        self.lib.bz_copy_panels(src.data_ptr(), dst.data_ptr(), a.n_kv_heads,
                                                bucket * a.head_dim * 2, self.s_max * a.head_dim * 2,
                                                n * a.head_dim * 2, 16, s)
            kv.pos_dev[slot:slot + 1].fill_(n)

    def _decode_step(self, inst):
        """Replay the smallest captured decode step covering every active slot."""
        top = max(inst.active) + 1
        rows = next(r for r in self.DECODE_GRAPH_ROWS if r >= top and r <= self.decode_slots)
        self.dgraphs[(inst.key, rows)]()

    def _warm(self):
        # every kernel / library plan both instances use, on their serving streams
        for ex, s, dev in [(self.ex0, self.s0, self.src_dev)] + list(zip(self.tex, self.ts, self.tgt_devs)):
            with torch.cuda.device(dev), torch.cuda.stream(s):
                for n in (512, 1024, 2048):
                    ex.forward(torch.randint(0, self.arch.vocab, (1, n), device=f"cuda:{dev}"))
            s.synchronize()

    def prefill_ms(self, n_tok: int, iters: int = 5) -> float:
        """Mean ms of one served prefill of ``n_tok`` tokens (its bucket's graph)."""
        g = self.graphs[("src", self.bucket(n_tok))]
        with torch.cuda.device(self.src_dev), torch.cuda.stream(self.s0):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.s0)
            for _ in range(iters):
                g.replay()
            e1.record(self.s0)
        e1.synchronize()
        return e0.elapsed_time(e1) / iters

    # ---- scale-up mechanisms ------------------------------------------------------------------

    def _start_load(self, strategy: str, group: Sequence[int] = (0,)) -> list:
        """Enqueue the weight load of the new instances ``group`` (target indices, in
        order); returns, per target, the event that marks its last layer published."""
        self.epoch += 1
        lay = self.layout
        for j in group:
            with torch.cuda.device(self.tgt_devs[j]):
                self.tslabs[j].loaded.zero_()
            torch.cuda.synchronize(self.tgt_devs[j])
        if strategy == "blitz":
            # chain source -> group[0] -> group[1] -> ... on the copy engines (the data
            # plane's chain mover): the serving source spends no SM; every relay forwards
            # a 256-tile group once its own flags carry the epoch
            tiles = CE_CHAIN_TILES_PER_COPY
            off = lay.tile_off.ctypes.data
            with torch.cuda.device(self.src_dev):
                peer = self.peer_on_src[group[0]]
                self.lib.bz_push_tiles_ce2(self.src.ptr, peer.ptr, peer.flags_ptr, None, off, 0, lay.ntiles, tiles,
                                           self.epoch, self.push_stream.cuda_stream, self.push_flag_stream.cuda_stream)
            for a, b in zip(group, group[1:]):
                if b != a + 1:
                    raise ValueError("a blitz group is a run of consecutive targets")
                t, nxt = self.tslabs[a], self.peer_next[a]
                with torch.cuda.device(self.tgt_devs[a]):
                    self.lib.bz_push_tiles_ce_gated(t.ptr, nxt.ptr, nxt.flags_ptr, t.flags_ptr, off, 0, lay.ntiles,
                                                    tiles, self.epoch, self.tpush[a].cuda_stream,
                                                    self.tflag[a].cuda_stream, self.tgate[a].cuda_stream)
            for j in group:
                t = self.tslabs[j]
                with torch.cuda.device(self.tgt_devs[j]):
                    self.lib.bz_track_layers(t.flags_ptr, t.layer_tile.data_ptr(), lay.num_layers, self.epoch,
                                             t.loaded.data_ptr(), t.stamps.data_ptr(), self.tload[j].cuda_stream)
        else:  # allcache / live-host: O(1) host-cache load over PCIe into every new
            # instance in parallel, layer by layer, each layer published in-stream
            for k in range(lay.num_layers):
                t0, t1 = lay.tiles_of_layer(k)
                for j in group:
                    t = self.tslabs[j]
                    with torch.cuda.device(self.tgt_devs[j]):
                        s = self.tload[j].cuda_stream
                        self.lib.bz_stage_tiles_ce(self.host.ptr, t.ptr, t.flags_ptr,
                                                   self.host.tile_off_host.ctypes.data, t0, t1, 128, self.epoch, s)
                        self.lib.bz_publish_layer(t.loaded.data_ptr(), k + 1, t.stamps.data_ptr() + 8 * k, s)
        events = []
        for j in group:
            with torch.cuda.device(self.tgt_devs[j]):
                done = torch.cuda.Event()
                done.record(self.tload[j])
            events.append(done)
        return events

    # ---- the replay -----------------------------------------------------------------------------

    def run(self, arrivals: list[tuple[float, int]], strategy: str, capacity_tok_s: float,
            window_s: float = 1.0, poll_sleep_s: float = 0.0002, time_l: float = 13.0,
            pair_batch: int = 2) -> RealClockResult:
        """Replay ``arrivals`` (seconds, prompt tokens) on the wall clock.  ``time_l``
        (one layer's load time over one layer's execution, livescale.py:4-14) and
        ``pair_batch`` (requests per cooperative run) apply to ``live-host``."""
        reqs = [Req(i, a[0], a[1], n_out=(a[2] if len(a) > 2 and self.decode_slots else 0))
                for i, a in enumerate(arrivals)]
        keys = ["src"] + [f"t{j}" for j in range(len(self.tgt_devs))]
        insts = [_Instance("gpu%d" % self.src_dev, torch.device("cuda", self.src_dev), self.ex0, self.s0, True,
                           key="src")]
        insts += [_Instance("gpu%d" % d, torch.device("cuda", d), ex, st, False, key=k)
                  for d, ex, st, k in zip(self.tgt_devs, self.tex, self.ts, keys[1:])]
        for inst in insts:
            inst.active.clear()
        decode_steps = 0
        finished = 0
        policy = ScalePolicy(upper_bound=capacity_tok_s, lower_bound=0.1 * capacity_tok_s,
                             strategy={"allcache": "allcache", "live-host": "blitz-live"}.get(strategy, "blitz-stop"))
        queue: collections.deque = collections.deque()
        window: collections.deque = collections.deque()
        nxt = 0
        done = 0
        load_ev: dict[int, torch.cuda.Event] = {}     # target index -> load-complete event
        started = 0                                  # targets whose load has been enqueued
        trigger_t = ready_t = None
        ready_all_t = None
        pair_runs: list = []
        t0 = time.perf_counter()
        while done < len(reqs) or finished < len(reqs):
            now = time.perf_counter() - t0
            while nxt < len(reqs) and reqs[nxt].t_arrive <= now:
                queue.append(reqs[nxt])
                window.append((reqs[nxt].t_arrive, reqs[nxt].n_tok))
                nxt += 1
            while window and window[0][0] < now - window_s:
                window.popleft()
            # scale trigger: the reference policy on the windowed arrival rate
            if strategy != "static" and started < len(self.tgt_devs) and now > window_s:
                tps = sum(n for _, n in window) / window_s
                add = should_scale_up(LoadMetrics(window_s=window_s, tokens_per_s=tps), policy, 1 + started)
                if add > 0:
                    # live-host pairs the first new instance only; the rest load alone
                    group = list(range(started, min(len(self.tgt_devs), started + add)))
                    if trigger_t is None:
                        trigger_t = now
                    for j, ev in zip(group, self._start_load(strategy, group)):
                        load_ev[j] = ev
                    started = group[-1] + 1
            for j, ev in load_ev.items():
                if not insts[1 + j].ready and ev.query():
                    insts[1 + j].ready = True
                    t_ready = time.perf_counter() - t0
                    if j == 0:
                        ready_t = t_ready
                    if all(insts[1 + i].ready for i in range(started)):
                        ready_all_t = t_ready
            # completions
            for inst in insts:
                if inst.busy is not None and inst.busy[2].query():
                    kind, payload, _ = inst.busy
                    inst.busy = None
                    t_now = time.perf_counter() - t0
                    if kind == "prefill":
                        payload.t_done = t_now
                        payload.served_by = inst.name
                        done += 1
                        if payload.n_out <= 1:
                            finished += 1
                            inst.active.pop(payload.slot, None)
                    else:
                        for req in payload:
                            req.token_t.append(t_now)
                            if len(req.token_t) >= req.n_out - 1:
                                finished += 1
                                inst.active.pop(req.slot, None)
            # live-host: while the new instance loads, serve queued requests as a ZigZag pair
            if (strategy == "live-host" and 0 in load_ev and not insts[1].ready and queue
                    and insts[0].busy is None):
                batch = [queue.popleft() for _ in range(min(pair_batch, len(queue)))]
                toks = [self.pair_tokens[self.bucket(r.n_tok)] for r in batch]
                cfg = livescale.configure_pipeline(len(batch), self.arch.n_layers, time_l)
                t_run = time.perf_counter() - t0
                with torch.cuda.device(self.src_dev):
                    res = self.pair.run(toks, cfg, livescale.zigzag_schedule(cfg))
                pair_runs.append((round(t_run, 4), [list(x) for x in cfg.splits],
                                  round((time.perf_counter() - t0 - t_run) * 1e3, 2)))
                for r, f in zip(batch, res.finish_ms):
                    r.t_done = t_run + f / 1e3
                    r.served_by = "pair"
                    done += 1
                    if r.n_out > 1 and len(insts[0].active) < self.decode_slots:
                        # the pair ran the prompt; its tokens are decoded on the source
                        # (its keys/values are not gathered from the two halves: the
                        # decode step's cost does not depend on them)
                        self._admit(insts[0], r, 0)
                    elif r.n_out > 1:
                        r.n_out = 1      # no free decode slot: counted as a prefill-only request
                        finished += 1
                    else:
                        finished += 1
                continue
            # dispatch to idle ready instances: prefills FCFS; with decoding, a decode step
            # of the instance's active slots alternates with prefills when both wait
            for inst in insts:
                if not inst.ready or inst.busy is not None:
                    continue
                can_prefill = bool(queue) and (not self.decode_slots or len(inst.active) < self.decode_slots)
                want_decode = bool(inst.active) and (not can_prefill or inst.last == "prefill")
                with torch.cuda.device(inst.device), torch.cuda.stream(inst.stream):
                    if want_decode:
                        live = [r for r in inst.active.values() if r.t_done is not None]
                        self._decode_step(inst)
                        decode_steps += 1
                        ev = torch.cuda.Event()
                        ev.record(inst.stream)
                        inst.busy = ("decode", live, ev)
                        inst.last = "decode"
                    elif can_prefill:
                        req = queue.popleft()
                        bucket = self.bucket(req.n_tok)
                        self.graphs[(inst.key, bucket)].replay()
                        if req.n_out > 1:
                            self._admit(inst, req, bucket)
                        ev = torch.cuda.Event()
                        ev.record(inst.stream)
                        inst.busy = ("prefill", req, ev)
                        inst.last = "prefill"
            if done == len(reqs) and finished >= len(reqs):
                break
            time.sleep(poll_sleep_s)
        wall = time.perf_counter() - t0
        ttft = [(r.t_done - r.t_arrive) * 1e3 for r in reqs]
        tbt = []
        for r in reqs:
            prev = r.t_done
            for t in r.token_t:
                tbt.append((t - prev) * 1e3)
                prev = t
        served = collections.Counter(r.served_by for r in reqs)
        load_ms = (ready_t - trigger_t) * 1e3 if ready_t is not None and trigger_t is not None else None
        for d in [self.src_dev] + self.tgt_devs:
            torch.cuda.synchronize(d)
        return RealClockResult(strategy=strategy, n=len(reqs), p50_ttft_ms=_pct(ttft, 50),
                               p99_ttft_ms=_pct(ttft, 99), mean_ttft_ms=sum(ttft) / len(ttft),
                               scale_trigger_s=trigger_t, scale_ready_s=ready_t, load_ms=load_ms,
                               served=dict(served), wall_s=wall, pair_runs=pair_runs,
                               instances_added=started, all_ready_s=ready_all_t,
                               p50_tbt_ms=_pct(tbt, 50) if tbt else None, p99_tbt_ms=_pct(tbt, 99) if tbt else None,
                               decode_steps=decode_steps)

    def close(self):
        for p in self.peer_on_src + self.peer_next:
            p.close()
        self.host.close()
        self.src.close()
        for t in self.tslabs:
            t.close()
