"""The simulator's scale-ups executed for real, in process.

The reference's hot-path caller ``Simulation._scale_via_network``
(simcore.py:676-750) plans a scale-up and then *models* it: it pushes one
``layer`` event per layer at ``(d - 1 + k) * layer_shard / B`` and a ``transfer``
event at the modeled completion (simcore.py:727-738; handlers 752-795).
``ExecutedCosts`` is a cost provider whose ``on_plan`` hook runs each plan the
simulator makes on this process's GPUs -- real bytes through the data-plane
kernels -- and whose ``layer_arrival_s`` / ``completion_s`` then return the
device stamps of that execution (``%globaltimer`` written by the per-layer
tracker), so the replay's ``layer`` and ``transfer`` events are measured, not
looked up.  Stop-the-world host-cache loads (AllCache, ServerlessLLM hits) are
executed the same way.

What runs where:
* every plan edge inside one host (``nvlink`` chain hops and ``pcie`` host-cache
  staging; fan-out groups as a pipelined sibling chain, the measured ``auto``
  realisation) runs on local devices, one plan GPU per device, all hops
  concurrently -- relays forward each tile as its flag lands, exactly as the
  multi-process executor does;
* with fewer devices than plan GPUs and ``loopback=True`` (tests on one GPU) the
  hops run stream-ordered on device 0 (``execute_plan_loopback``): the events are
  still device stamps, but of serialized HBM-local copies;
* nodes reached over an ``rdma`` edge (another host) stay on the reference
  model -- there is no second host in this process.
Every execution is verified: each receiving slab's tile fingerprints equal the
source's.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from ._native import cuda_lib, ptr_array
from .costs import MeasuredCosts
from .dataplane import (CE_CHAIN_TILES_PER_COPY, DeviceSlab, HostCache, PeerSlab, execute_plan_loopback,
                        plan_roles)
from .planner import ScalePlan
from .slab import LlamaArch, SlabLayout


@dataclass
class Execution:
    plan_edges: list
    mode: str                                   # "devices" | "loopback" | "host-load"
    arrivals_s: dict = field(default_factory=dict)   # node -> [layer k arrival, s after launch]
    bit_exact: bool = True
    wall_ms: float = 0.0


class LocalPlanExecutor:
    """Runs the intra-host part of a plan on this process's devices."""

    def __init__(self, arch: LlamaArch, devices: Sequence[int], tile_bytes: int = 1 << 20, nctas: int = 48,
                 seed: int = 241217, loopback: bool = False):
        self.arch = arch
        self.devices = list(devices)
        self.layout = SlabLayout.for_arch(arch, tile_bytes=tile_bytes)
        self.nctas = nctas
        self.seed = seed
        self.loopback = loopback
        self.lib = cuda_lib(self.devices[0])
        for d in self.devices:
            cuda_lib(d)
        self._slabs: dict = {}      # key -> DeviceSlab
        self._peers: dict = {}      # (sender device, receiver key) -> PeerSlab
        self._streams: dict = {}
        self._host: Optional[HostCache] = None
        self._want: Optional[torch.Tensor] = None
        self.epoch = 0

    # ---- resources ------------------------------------------------------------------------
    def _slab(self, key, device: int) -> DeviceSlab:
        if key not in self._slabs:
            with torch.cuda.device(device):
                self._slabs[key] = DeviceSlab(self.layout, device)
        return self._slabs[key]

    def _source(self, key, device: int) -> DeviceSlab:
        s = self._slab(("src", key), device)
        if not getattr(s, "_filled", False):
            s.fill_random(self.seed)
            torch.cuda.synchronize(device)
            s._filled = True
            if self._want is None:
                self._want = s.fingerprints().cpu()
        return s

    def _host_cache(self) -> HostCache:
        if self._host is None:
            d = self.devices[0]
            tmp = self._source("ref", d)
            self._host = HostCache(self.layout)
            self._host.tensor.copy_(tmp.data.cpu())
        return self._host

    def _peer(self, sender_dev: int, recv_key, recv: DeviceSlab) -> int:
        if sender_dev == recv.device:
            return recv.ptr
        k = (sender_dev, recv_key)
        if k not in self._peers:
            pid, fd, nb = recv.export()
            self._peers[k] = PeerSlab(sender_dev, pid, fd, nb, self.layout)
        return self._peers[k].ptr

    def _stream(self, device: int, kind: str) -> torch.cuda.Stream:
        k = (device, kind)
        if k not in self._streams:
            self._streams[k] = torch.cuda.Stream(device=device)
        return self._streams[k]

    # ---- execution ------------------------------------------------------------------------
    @staticmethod
    def local_subplan(plan: ScalePlan) -> tuple[ScalePlan, list[str]]:
        """(the executable part of ``plan``, targets left on the model): the nvlink /
        pcie edges whose sender holds the weights -- a live source, a host cache, or a
        node itself fed by such an edge; nodes behind an rdma edge are not."""
        fed_anywhere = {e.dst for e in plan.edges}
        ok = {e.src for e in plan.edges if e.src not in fed_anywhere}
        keep: list = []
        changed = True
        while changed:
            changed = False
            for e in plan.edges:
                if e.kind in ("nvlink", "pcie") and e not in keep and e.src in ok:
                    keep.append(e)
                    ok.add(e.dst)
                    changed = True
        fan = {rep: list(sibs) for rep, sibs in plan.nvlink_fanout.items() if rep in ok}
        local = ScalePlan(edges=keep, chains=[], nvlink_fanout=fan)
        covered = {e.dst for e in keep} | {s for sibs in fan.values() for s in sibs}
        return local, [n for n in plan.targets() if n not in covered]

    def execute(self, plan: ScalePlan) -> Optional[Execution]:
        local, _ = self.local_subplan(plan)
        if not local.edges:
            return None
        gpus = sorted({n for e in local.edges for n in (e.src, e.dst) if n.startswith("gpu")} |
                      {s for sibs in local.nvlink_fanout.values() for s in sibs}, key=lambda n: int(n[3:]))
        if len(gpus) <= len(self.devices):
            return self._execute_devices(local, {n: self.devices[i] for i, n in enumerate(gpus)})
        if self.loopback:
            return self._execute_loopback(local, gpus)
        return None

    def _execute_loopback(self, plan: ScalePlan, gpus: list[str]) -> Execution:
        d = self.devices[0]
        roles = plan_roles(plan)
        slabs = {n: (self._source(n, d) if not roles[n].receives else self._slab(("dst", n), d)) for n in gpus}
        self.epoch += 1
        hc = self._host_cache() if any(e.src.startswith("mem") for e in plan.edges) else None
        with torch.cuda.device(d):
            s = self._stream(d, "loop")
            for n in gpus:
                if roles[n].receives:
                    self.lib.bz_publish_layer(slabs[n].loaded.data_ptr(), 0,
                                              slabs[n].stamps.data_ptr() + 8 * self.layout.num_layers, s.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            execute_plan_loopback(plan, slabs, self.epoch, host_cache=hc, nctas=self.nctas, stream=s)
            e1.record(s)
            e1.synchronize()
        out = Execution(plan_edges=[(e.src, e.dst, e.kind) for e in plan.edges], mode="loopback",
                        wall_ms=e0.elapsed_time(e1))
        self._collect(out, {n: slabs[n] for n in gpus if roles[n].receives})
        return out

    def _execute_devices(self, plan: ScalePlan, dev_of: dict) -> Execution:
        roles = plan_roles(plan)
        lay, lib = self.layout, self.lib
        self.epoch += 1
        e = self.epoch
        # one receiving and one source slab per device, whatever node name the plan gives it
        slabs = {n: (self._slab(("dst", dev_of[n]), dev_of[n]) if roles[n].receives
                     else self._source(("dev", dev_of[n]), dev_of[n])) for n in dev_of}
        hc = self._host_cache() if any(x.src.startswith("mem") for x in plan.edges) else None
        for d in set(dev_of.values()):
            torch.cuda.synchronize(d)
        # receivers first (reset + launch stamp, tracker), then staging, then pushes
        for n, slab in slabs.items():
            if not roles[n].receives:
                continue
            d = dev_of[n]
            st = self._stream(d, "track").cuda_stream
            with torch.cuda.device(d):
                lib.bz_publish_layer(slab.loaded.data_ptr(), 0, slab.stamps.data_ptr() + 8 * lay.num_layers, st)
                lib.bz_track_layers(slab.flags_ptr, slab.layer_tile.data_ptr(), lay.num_layers, e,
                                    slab.loaded.data_ptr(), slab.stamps.data_ptr(), st)
        for n, slab in slabs.items():
            if (roles[n].parent or "").startswith("mem"):
                d = dev_of[n]
                with torch.cuda.device(d):
                    lib.bz_stage_tiles_ce(hc.ptr, slab.ptr, slab.flags_ptr, hc.tile_off_host.ctypes.data, 0,
                                          lay.ntiles, 128, e, self._stream(d, "stage").cuda_stream)
        for n, slab in slabs.items():
            r = roles[n]
            outs = list(r.children)
            if r.fanout:                       # fan-out as a pipelined sibling chain
                outs.append(r.fanout[0])
            if r.rep is not None:
                sibs = plan.nvlink_fanout[r.rep]
                i = sibs.index(n)
                if i + 1 < len(sibs):
                    outs.append(sibs[i + 1])
            outs = [o for o in outs if o in slabs]
            if not outs:
                continue
            d = dev_of[n]
            with torch.cuda.device(d):
                if len(outs) == 1:
                    # the data plane's chain mover: copy engines in 256-tile groups, a relay's
                    # gates enqueued ahead on their own stream (no SM on any GPU)
                    dst = self._peer(d, ("dst", dev_of[outs[0]]), slabs[outs[0]])
                    off = lay.tile_off.ctypes.data
                    if r.receives:
                        lib.bz_push_tiles_ce_gated(slab.ptr, dst, dst + lay.flag_offset, slab.flags_ptr, off, 0,
                                                   lay.ntiles, CE_CHAIN_TILES_PER_COPY, e,
                                                   self._stream(d, "copy").cuda_stream,
                                                   self._stream(d, "ceflag").cuda_stream,
                                                   self._stream(d, "cegate").cuda_stream)
                    else:
                        lib.bz_push_tiles_ce2(slab.ptr, dst, dst + lay.flag_offset, None, off, 0, lay.ntiles,
                                              CE_CHAIN_TILES_PER_COPY, e, self._stream(d, "copy").cuda_stream,
                                              self._stream(d, "ceflag").cuda_stream)
                    continue
                ptrs = ptr_array([self._peer(d, ("dst", dev_of[o]), slabs[o]) for o in outs])
                flags = ptr_array([self._peer(d, ("dst", dev_of[o]), slabs[o]) + lay.flag_offset for o in outs])
                lib.bz_push_tiles(slab.ptr, ptrs, flags, len(outs), slab.flags_ptr if r.receives else None,
                                  slab.tile_off.data_ptr(), 0, lay.ntiles, e, self.nctas, 0,
                                  self._stream(d, "copy").cuda_stream)
        for (d, _), st in self._streams.items():
            st.synchronize()
        from .scaleup import check_wait_timeouts
        for d in set(dev_of.values()):
            check_wait_timeouts(d)
        out = Execution(plan_edges=[(x.src, x.dst, x.kind) for x in plan.edges], mode="devices")
        self._collect(out, {n: s for n, s in slabs.items() if roles[n].receives})
        return out

    def _collect(self, out: Execution, receivers: dict):
        L = self.layout.num_layers
        for n, slab in receivers.items():
            st = slab.stamps.cpu().tolist()
            out.arrivals_s[n] = [(x - st[L]) / 1e9 for x in st[:L]]
            ok = torch.equal(slab.fingerprints().cpu(), self._want) and int(slab.loaded.item()) == L
            out.bit_exact &= bool(ok)
        out.wall_ms = out.wall_ms or 1e3 * max(a[-1] for a in out.arrivals_s.values())

    def host_load(self) -> Execution:
        """One O(1) host-cache load into a fresh slab on the first device (copy engines,
        per-layer publish) -- the stop-the-world load of AllCache / a ServerlessLLM hit."""
        d = self.devices[0]
        slab = self._slab(("dst", "host-load"), d)
        hc = self._host_cache()
        self.epoch += 1
        lay = self.layout
        with torch.cuda.device(d):
            s = self._stream(d, "stage").cuda_stream
            self.lib.bz_publish_layer(slab.loaded.data_ptr(), 0, slab.stamps.data_ptr() + 8 * lay.num_layers, s)
            for k in range(lay.num_layers):
                t0, t1 = lay.tiles_of_layer(k)
                self.lib.bz_stage_tiles_ce(hc.ptr, slab.ptr, slab.flags_ptr, hc.tile_off_host.ctypes.data, t0, t1,
                                           128, self.epoch, s)
                self.lib.bz_publish_layer(slab.loaded.data_ptr(), k + 1, slab.stamps.data_ptr() + 8 * k, s)
            self._stream(d, "stage").synchronize()
        out = Execution(plan_edges=[("mem0", "gpu", "pcie")], mode="host-load")
        self._collect(out, {"host-load": slab})
        return out

    def close(self):
        for st in self._streams.values():
            st.synchronize()
        for p in self._peers.values():
            p.close()
        for s in self._slabs.values():
            s.close()
        if self._host is not None:
            self._host.close()


class ExecutedCosts(MeasuredCosts):
    """Reference-compatible cost provider whose scale-up events are executed.

    ``simscale._scale_via_network`` calls ``on_plan(plan, model)`` right after
    planning; ``layer_arrival_s`` / ``completion_s`` for that plan's nodes then
    return the device stamps of the execution.  Anything not executed (rdma
    paths, plans larger than the local GPUs) falls through to ``MeasuredCosts``
    (its measured tables if given, else the reference model)."""

    name = "b200-executed"

    def __init__(self, executor: LocalPlanExecutor, **measured):
        super().__init__(**measured)
        self.executor = executor
        self.executions: list[Execution] = []
        self._plan_id: Optional[int] = None
        self._arrivals: dict = {}
        self._host_cache_s: dict = {}

    def on_plan(self, plan, model) -> None:
        ex = self.executor.execute(plan)
        self._plan_id = id(plan)
        self._arrivals = dict(ex.arrivals_s) if ex is not None else {}
        if ex is not None:
            self.executions.append(ex)

    def layer_arrival_s(self, plan, node, model, eta) -> list[float]:
        if id(plan) == self._plan_id and node in self._arrivals and \
                len(self._arrivals[node]) == model.num_layers:
            return list(self._arrivals[node])
        return super().layer_arrival_s(plan, node, model, eta)

    def completion_s(self, plan, est, node, model, eta) -> float:
        if id(plan) == self._plan_id and node in self._arrivals:
            return self._arrivals[node][-1]
        return super().completion_s(plan, est, node, model, eta)

    def stop_the_world_s(self, strategy, model, topo, pool, host_id, now_s, eta) -> float:
        hit = strategy == "allcache" or (strategy == "sllm" and pool is not None and host_id is not None
                                         and pool.cache_hit(model.name, host_id, now_s))
        if hit and model.num_layers == self.executor.layout.num_layers:
            key = (strategy, now_s, host_id)
            if key not in self._host_cache_s:
                ex = self.executor.host_load()
                self.executions.append(ex)
                self._host_cache_s[key] = ex.arrivals_s["host-load"][-1]
            return self._host_cache_s[key]
        return super().stop_the_world_s(strategy, model, topo, pool, host_id, now_s, eta)

    def describe(self) -> dict:
        d = super().describe()
        modes: dict = {}
        for ex in self.executions:
            modes[ex.mode] = modes.get(ex.mode, 0) + 1
        d.update({"executed": modes, "executed_bit_exact": all(ex.bit_exact for ex in self.executions),
                  "layer_events": "device stamps of the executed plan (rdma paths: fallback)"})
        return d
