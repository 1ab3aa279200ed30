"""Scale-up sessions: the user-facing call that turns "add instances of model M
on these GPUs" into a plan (reference API) and a measured transfer (B200 data plane).

Mirrors the reference caller ``simcore.Simulation._scale_via_network``
(simcore.py:676-750): sources from the parameter pool, ``build_scale_request``
-> ``generate_plan`` -> ``estimate_completion``, then -- instead of pushing
modeled ``transfer``/``layer`` events -- the plan is executed by
``ScaleExecutor`` and the per-layer arrival stamps come back from the GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

import os
from typing import Callable

from .dataplane import ENGINE_VECTOR, DeviceSlab, Fabric, HostCache, ScaleExecutor, host_fed_groups, plan_roles
from .planner import build_scale_request, estimate_completion, generate_plan
from .slab import LlamaArch, SlabLayout, model_spec_for
from .topology import FlowSet, load_topology


@dataclass
class ScaleUpResult:
    epoch: int
    elapsed_ms: float                       # this rank: launch -> its share done
    kernel_ms: Optional[float] = None       # this rank's bulk mover (stream-event timed)
    layer_ms: list[float] = field(default_factory=list)
    verified: Optional[bool] = None


def plan_for(arch: LlamaArch, sources: Sequence[str], targets: Sequence[str],
             topo="b200-hgx", group: bool = True, tp: int = 1):
    """Reference planning path for a real architecture (bytes = real shard size).

    Sources/targets are instance *anchors* (``InstanceState.node = gpus[0]``,
    simcore.py:142-144); the returned plan is the anchor plan.  Use
    ``rank_plan`` to expand it over the TP ranks of every instance.
    """
    t = load_topology(topo)
    flows = FlowSet(t)
    model = model_spec_for(arch, tp=tp)
    req = build_scale_request(model, list(sources), list(targets), t, flows)
    plan = generate_plan(req, t, flows, group=group)
    return plan, model, estimate_completion(plan, model, t, eta=1.0)


def rank_plan(anchor_plan, tp: int):
    """Per-GPU plan: rank r of every instance talks to rank r of the others."""
    from .dataplane import expand_tp, merge_plans

    return anchor_plan if tp == 1 else merge_plans(expand_tp(anchor_plan, tp))


def plan_host_cache(fabric: Fabric, layout: SlabLayout, plan, node_rank: dict[str, int],
                    fill: Callable[[torch.Tensor], None], host_stripe: bool = True,
                    tag: str = "hc") -> Optional[HostCache]:
    """This rank's view of the O(1) pinned host copy, or None if it stages nothing.

    Collective (every rank calls it).  One /dev/shm region per host-fed group:
    the rank of the rep (the ``mem<h> -> rep`` edge's target) creates it and
    ``fill``s it; with ``host_stripe`` its NVLink siblings map the same pages
    (each registers them pinned) and stage their own pieces of every layer.
    """
    node = {r: n for n, r in node_rank.items()}.get(fabric.rank)
    roles = plan_roles(plan)
    groups = host_fed_groups(plan) if host_stripe else {}
    owner = node is not None and node in roles and (roles[node].parent or "").startswith("mem")
    group_of = {m: rep for rep, members in groups.items() for m in members}
    # only a group whose siblings map the same pages needs a named /dev/shm region;
    # a lone rep stages from anonymous pinned memory (no tmpfs size limit, no leftovers)
    shared = owner and len(groups.get(node, [])) > 1
    name = f"bz_{tag}_{node}_{os.getpid()}" if shared else None
    names = fabric.allgather((node, name))
    by_node = {n: nm for n, nm in names if nm}
    hc = None
    err = None
    try:
        if owner:
            if shared:
                _require_shm_space(layout.data_bytes)
            hc = HostCache(layout, shm_name=name, create=True)
            fill(hc.tensor)
    except BaseException as e:  # noqa: BLE001 -- re-raised after the collective below
        err = e
    failed = fabric.allgather(err is not None)
    try:
        if err is not None:
            raise err
        if any(failed):
            raise RuntimeError("host cache: another rank failed to create or fill its host copy")
        if not owner and node in group_of:
            hc = HostCache(layout, shm_name=by_node[group_of[node]], create=False)
        fabric.barrier()
    finally:
        if owner and name and os.path.exists(f"/dev/shm/{name}"):
            # every member has mapped it (or setup failed): drop the name; the
            # mappings keep the pages
            os.unlink(f"/dev/shm/{name}")
            if hc is not None:
                hc.path = None
    return hc


def _require_shm_space(nbytes: int) -> None:
    """A /dev/shm file larger than the tmpfs would SIGBUS on first touch: refuse early."""
    st = os.statvfs("/dev/shm")
    free = st.f_bavail * st.f_frsize
    if free < nbytes:
        raise RuntimeError(f"/dev/shm has {free / 1e9:.2f} GB free, the shared host copy needs "
                           f"{nbytes / 1e9:.2f} GB (enlarge /dev/shm or pass host_stripe=False)")


class TransferTimeout(RuntimeError):
    """A device-side wait gave up (its upstream never published)."""


_seen_timeouts: dict[int, int] = {}


def new_wait_timeouts(device: Optional[int] = None) -> int:
    """Device-side waits on ``device`` (default: current) that gave up since the
    last call (they skipped their copy and withheld their downstream flags)."""
    import ctypes

    from ._native import cuda_lib
    dev = torch.cuda.current_device() if device is None else int(device)
    n = ctypes.c_uint64()
    with torch.cuda.device(dev):
        cuda_lib().bz_wait_timeouts(ctypes.byref(n), 0)
    new = n.value - _seen_timeouts.get(dev, 0)
    _seen_timeouts[dev] = n.value
    return max(0, int(new))


def check_wait_timeouts(device: Optional[int] = None) -> None:
    """Raise if a bounded device-side wait on ``device`` (default: current) gave up
    since the last check -- the kernels behind it ran on data that never arrived."""
    dev = torch.cuda.current_device() if device is None else int(device)
    n = new_wait_timeouts(dev)
    if n:
        raise TransferTimeout(f"cuda:{dev}: {n} device-side waits timed out (upstream never published)")


def expected_fingerprints(layout: SlabLayout, device: int, seed: int) -> torch.Tensor:
    """Fingerprints of the synthetic shard made from ``seed`` (regenerated locally)."""
    tmp = DeviceSlab(layout, device)
    tmp.fill_random(seed)
    prints = tmp.fingerprints().cpu()
    tmp.close()
    return prints


class ScaleUpSession:
    """One rank's persistent scale-up machinery for a (plan, model) pair.

    Construction is collective (all ranks): slabs are allocated, exported,
    peer-mapped and multicast-bound once -- the connection pool.  ``run()``
    executes one scale-up and blocks until this rank's share is done.  The
    source shard is synthetic: random bits from ``seed`` (bf16 NaN/Inf
    patterns included), on the source GPU or in the pinned host cache.
    """

    def __init__(self, fabric: Fabric, layout: SlabLayout, plan, node_rank: dict[str, int],
                 host_cache: Optional[HostCache] = None, engine: int = ENGINE_VECTOR,
                 nctas: int = 32, fanout_mode: str = "auto", seed: int = 241217,
                 stage_engine: str = "ce", tiles_per_copy: int = 128, host_stripe: bool = True,
                 ce_tiles_per_copy: int = 0):
        self.fabric = fabric
        self.layout = layout
        self.plan = plan
        self.seed = seed
        self.node_rank = node_rank
        self.slab = DeviceSlab(layout, fabric.device)
        node = {r: n for n, r in node_rank.items()}.get(fabric.rank)
        self.node = node
        self.is_source = node is not None and node not in plan.targets()
        if self.is_source:
            self.slab.fill_random(seed)
        torch.cuda.synchronize()
        self.executor = ScaleExecutor(fabric, plan, self.slab, node_rank, host_cache=host_cache,
                                      engine=engine, nctas=nctas, fanout_mode=fanout_mode,
                                      stage_engine=stage_engine, tiles_per_copy=tiles_per_copy,
                                      host_stripe=host_stripe, ce_tiles_per_copy=ce_tiles_per_copy)
        self.receives = self.executor.role.receives
        self.fabric_nodes = {r: n for n, r in node_rank.items()}
        self._expected: Optional[torch.Tensor] = None

    def run(self, verify: bool = False, time_kernel: bool = False) -> ScaleUpResult:
        """Barrier, launch, wait; CUDA-event timed on this rank."""
        self.fabric.barrier()
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kev = None
        if time_kernel:
            kev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        start.record(cur)
        for s in self.executor.streams.values():
            s.wait_stream(cur)
        epoch = self.executor.launch(kernel_events=kev)
        for s in self.executor.streams.values():
            cur.wait_stream(s)
        end.record(cur)
        end.synchronize()
        # every rank learns of a timeout anywhere in the plan (a dead relay starves
        # all GPUs below it; none of them may report the transfer as done)
        mine = new_wait_timeouts()
        counts = self.fabric.allgather(mine)
        if any(counts):
            bad = {self.fabric_nodes.get(r, r): c for r, c in enumerate(counts) if c}
            raise TransferTimeout(f"scale-up epoch {epoch}: device-side waits timed out on {bad}")
        res = ScaleUpResult(epoch, start.elapsed_time(end))
        if kev is not None and self.executor.dominant_stream() is not None:
            res.kernel_ms = kev[0].elapsed_time(kev[1])
        if self.receives:
            res.layer_ms = self.executor.layer_arrivals_ms()
        if verify:
            res.verified = self.verify(epoch)
        return res

    def verify(self, epoch: int) -> bool:
        """Bit-exactness of this rank's slab: tile fingerprints vs the regenerated
        source, every tile flag at ``epoch``, every layer tracked."""
        if not self.receives:
            return True
        if self._expected is None:
            self._expected = expected_fingerprints(self.layout, self.fabric.device, self.seed)
        ok = torch.equal(self.slab.fingerprints().cpu(), self._expected)
        ok = ok and int(self.slab.flags.min()) == epoch and int(self.slab.flags.max()) == epoch
        return ok and int(self.slab.loaded.item()) == self.layout.num_layers

    def close(self):
        self.executor.close()
        self.slab.close()
