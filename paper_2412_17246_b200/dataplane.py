"""B200 parameter data plane: executes a ``ScalePlan`` with real bytes.

Reference mapping (``/root/reference/pkg/src/scalesim``):

* ``ScalePlan.edges`` (planner.py:72-109) -> a chain hop: the edge's sender
  pushes every tile of its slab into the receiver's slab through a peer
  mapping (``bz_push_tiles``); a sender that is itself a receiver forwards
  tile ``t`` as soon as its own flag ``t`` is raised (store-and-forward of
  planner.py:240-244 at tile granularity, so a hop costs one tile of fill,
  not one layer).
* ``ScalePlan.nvlink_fanout`` (planner.py:86-87, 245-253) -> the
  representative relays each tile into an NVLS multicast object bound to the
  slabs of the whole fan-out group (``bz_multicast_tiles``): one stream out of
  the representative, replicated by the NVSwitch.  Without NVLS the group is
  served as a pipelined sibling chain.
* ``mem<h>`` sources (topology.py:174-176) -> the O(1) pinned host cache is
  staged by the copy engines on a side stream (``bz_stage_tiles_ce``).
* ``simcore`` per-layer ``layer`` events (simcore.py:727-733) -> every receiver
  runs a one-warp tracker (``bz_track_layers``) that raises a monotone
  ``loaded_layers`` counter in device memory and stamps each layer's arrival
  with ``%globaltimer``; compute streams gate on it (``bz_wait_layer``).

Process model: one process per GPU (``torchrun``); a slab is exported once
as a POSIX fd, peers import it with ``pidfd_getfd`` -- the pre-established
connection pool of PAPER.md:997-1006, no communicator creation on the scale
path.  ``torch.distributed`` is only used to exchange (pid, fd) pairs and for
barriers.  A single process can also drive several slabs on one GPU
("loopback"), which is how the single-GPU tests exercise the same kernels.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from ._native import BzMc, BzSlab, cuda_lib, ptr_array
from .planner import ScalePlan
from .slab import SlabLayout

ENGINE_VECTOR = 0
ENGINE_TMA = 1
ENGINE_VEC256 = 2   # 32-byte LDG/STG.E.ENL2.256 (sm_100)
ENGINE_CE = 3       # copy engines (cudaMemcpyAsync into the peer VA), SMs left for compute
# auto: a source -> leaf hop (the sender holds the shard, the receiver forwards nothing)
# is PULLED: the receiver's SMs read the sender's slab through the peer mapping
# (bz_pull_tiles), 781 GB/s vs 748 for the copy engines and 717 for an SM push
# (profiles/r2_pull_probe_n2.txt: NVLink reads carry less protocol than writes), and the
# sender -- the live instance -- spends no SM.  Along a relay chain every hop runs on the
# copy engines in 256-tile groups (bz_push_tiles_ce2 out of the source, a relay's gates
# enqueued ahead on their own stream: bz_push_tiles_ce_gated): 715-726 GB/s per
# destination on 1->4 vs 673-692 with SM-push relays and 582-627 with pulled relays (a
# GPU that pulls and is pulled from carries the read requests of both directions;
# profiles/r2_pull_chain_n4.txt, r2_ce2_chain_n4.txt).  Striped host-load pieces, NVLS
# fan-out and multi-destination sends keep their own movers.
ENGINE_AUTO = 4
# every single-destination hop on the copy engines (flags on a second stream; a relay's
# gates ahead on a third): auto's relay-chain mover applied to leaf hops as well -- the
# live pair's engine, whose target computes while it receives and so should not pull
ENGINE_CE2 = 5
PULL_CTAS = 64      # minimum receiver CTAs of a pulled hop (781 GB/s at 64, 768 at 48); a
                    # new instance is idle while it loads, so the pull takes all its SMs (783)
CE_TILES_PER_COPY = 16
CE2_TILES_PER_COPY = 128
CE_CHAIN_TILES_PER_COPY = 256   # copy-engine groups along a relay chain (128: 715, 256: 726 GB/s)
MAX_DST = 8  # BZ_MAX_DST (include/blitz.h): destinations per push launch


class _CudaView:
    """Expose raw device memory to torch without copying."""

    def __init__(self, ptr: int, nbytes: int, typestr: str, itemsize: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes // itemsize,), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": None,
        }


def device_view(ptr: int, nbytes: int, dtype: torch.dtype, device) -> torch.Tensor:
    typestr = {torch.uint8: "|u1", torch.int32: "<i4", torch.int64: "<i8",
               torch.int16: "<i2"}[dtype]
    item = torch.empty((), dtype=dtype).element_size()
    return torch.as_tensor(_CudaView(ptr, nbytes, typestr, item), device=device)


# ---- control plane (pid/fd exchange) ---------------------------------------------------


class Fabric:
    """This process's GPU plus the control channel to the other ranks."""

    def __init__(self, device: int, rank: int = 0, world: int = 1, group=None):
        self.device = device
        self.rank = rank
        self.world = world
        self.group = group
        self.lib = cuda_lib(device)
        import ctypes
        vals = [ctypes.c_int() for _ in range(4)]
        self.lib.bz_device_caps(device, *[ctypes.byref(v) for v in vals])
        self.multicast_supported = bool(vals[0].value)
        self.posix_fd_supported = bool(vals[1].value)
        self.sm_count = vals[3].value

    @classmethod
    def from_env(cls) -> "Fabric":
        """torchrun-style environment; initialises a gloo control group if needed."""
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        local = int(os.environ.get("LOCAL_RANK", str(rank)))
        # BZ_OVERSUBSCRIBE=<gpus>: more ranks than GPUs (rank r on GPU r % gpus) to check the
        # control flow of a large world on a small box -- gloo only (NCCL refuses two ranks
        # on one GPU); a functional mode, its bandwidths mean nothing
        over = int(os.environ.get("BZ_OVERSUBSCRIBE", "0"))
        device = local % over if over > 0 else local
        torch.cuda.set_device(device)
        group = None
        if world > 1:
            import torch.distributed as dist
            if not dist.is_initialized():
                if over > 0:
                    dist.init_process_group("gloo")
                else:
                    dist.init_process_group("nccl", device_id=torch.device("cuda", device))
            group = dist.new_group(backend="gloo")
        return cls(device, rank, world, group)

    def allgather(self, obj):
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)


# ---- slabs -----------------------------------------------------------------------------


class DeviceSlab:
    """One VMM allocation holding a shard (layer units, tiles) + its tile flags."""

    def __init__(self, layout: SlabLayout, device: int):
        self.layout = layout
        self.device = device
        self.lib = cuda_lib(device)
        self.raw = BzSlab()
        self.lib.bz_slab_create(device, layout.total_bytes, self.raw)
        dev = torch.device("cuda", device)
        self.data = device_view(self.raw.ptr, layout.data_bytes, torch.uint8, dev)
        self.flags = device_view(self.raw.ptr + layout.flag_offset, layout.ntiles * 4,
                                 torch.int32, dev)
        self.flags.zero_()
        self.tile_off = torch.from_numpy(layout.tile_off).to(dev)
        self.layer_tile = torch.from_numpy(layout.layer_tile).to(dev)
        self.loaded = torch.zeros(1, dtype=torch.int32, device=dev)
        self.stamps = torch.zeros(layout.num_layers + 1, dtype=torch.int64, device=dev)
        self._exported = False

    @property
    def ptr(self) -> int:
        return int(self.raw.ptr)

    @property
    def flags_ptr(self) -> int:
        return int(self.raw.ptr + self.layout.flag_offset)

    def export(self) -> tuple[int, int, int]:
        """(pid, fd, bytes) a peer needs to map this slab."""
        if not self._exported:
            self.lib.bz_slab_export(self.raw)
            self._exported = True
        return (os.getpid(), int(self.raw.fd), int(self.raw.bytes))

    def fill_random(self, seed: int, stream=None):
        # launched on this slab's device (one process may drive slabs on several GPUs)
        with torch.cuda.device(self.device):
            s = _stream_handle(stream, self.device)
            self.lib.bz_fill_random(self.ptr, self.layout.data_bytes, seed, s)

    def fingerprints(self, stream=None) -> torch.Tensor:
        with torch.cuda.device(self.device):
            out = torch.empty(self.layout.ntiles, dtype=torch.int64, device=self.data.device)
            self.lib.bz_tile_fingerprints(self.ptr, self.tile_off.data_ptr(), 0, self.layout.ntiles,
                                          out.data_ptr(), _stream_handle(stream, self.device))
        return out

    def close(self):
        if self.raw.ptr:
            torch.cuda.synchronize(self.device)
            self.lib.bz_slab_free(self.raw)


class PeerSlab:
    """A peer process's slab mapped into this process (NVLink peer VA)."""

    def __init__(self, local_device: int, pid: int, fd: int, nbytes: int, layout: SlabLayout):
        self.lib = cuda_lib(local_device)
        self.raw = BzSlab()
        self.lib.bz_slab_import(local_device, pid, fd, nbytes, self.raw)
        self.layout = layout

    @property
    def ptr(self) -> int:
        return int(self.raw.ptr)

    @property
    def flags_ptr(self) -> int:
        return int(self.raw.ptr + self.layout.flag_offset)

    def close(self):
        if self.raw.ptr:
            self.lib.bz_slab_free(self.raw)


class MulticastGroup:
    """NVLS multicast object bound to the slabs of a fan-out group."""

    def __init__(self, fabric: Fabric, slab: DeviceSlab, members: Sequence[int]):
        self.fabric = fabric
        self.members = sorted(members)
        self.lib = cuda_lib()
        self.raw = BzMc()
        self.bound = 0
        me = fabric.rank
        root = self.members[0]
        nbytes = int(slab.raw.bytes)
        info = None
        if me == root:
            self.lib.bz_mc_create(len(self.members), nbytes, self.raw)
            info = (os.getpid(), int(self.raw.fd), nbytes)
        infos = fabric.allgather(info)
        root_info = infos[root]
        if me in self.members and me != root:
            self.lib.bz_mc_import(root_info[0], root_info[1], root_info[2], self.raw)
        fabric.barrier()  # root's fd stays open until every member imported
        if me in self.members:
            self.lib.bz_mc_add_device(self.raw, fabric.device)
        fabric.barrier()
        if me in self.members:
            self.lib.bz_mc_bind(self.raw, fabric.device, slab.raw, 0, 0, nbytes)
            self.bound = nbytes
        fabric.barrier()
        if me in self.members:
            self.lib.bz_mc_map(self.raw, fabric.device)
        self.layout = slab.layout

    @property
    def ptr(self) -> int:
        return int(self.raw.mc_ptr)

    @property
    def flags_ptr(self) -> int:
        return int(self.raw.mc_ptr + self.layout.flag_offset)

    def close(self):
        if self.raw.handle:
            self.lib.bz_mc_free(self.raw, self.fabric.device, self.bound)


class LocalMulticastGroup:
    """An NVLS multicast object bound by ONE process to slabs on several of its GPUs
    (the single-process form of ``MulticastGroup``: tests, ncu captures, and a
    process that drives more than one GPU).  ``cuMulticastCreate`` rejects a
    one-device object on B200 (CUDA_ERROR_INVALID_VALUE, scripts/nvlink_probe.py),
    so at least two devices are required."""

    def __init__(self, slabs: Sequence[DeviceSlab], map_device: int):
        if len({s.device for s in slabs}) != len(slabs) or len(slabs) < 2:
            raise ValueError("one slab per distinct device, at least two devices")
        self.lib = cuda_lib()
        self.raw = BzMc()
        self.slabs = list(slabs)
        self.nbytes = int(slabs[0].raw.bytes)
        self.layout = slabs[0].layout
        self.map_device = map_device
        self.lib.bz_mc_create(len(slabs), self.nbytes, self.raw)
        for s in slabs:                      # every device joins before any binds
            self.lib.bz_mc_add_device(self.raw, s.device)
        for s in slabs:
            self.lib.bz_mc_bind(self.raw, s.device, s.raw, 0, 0, self.nbytes)
        self.lib.bz_mc_map(self.raw, map_device)

    @property
    def ptr(self) -> int:
        return int(self.raw.mc_ptr)

    @property
    def flags_ptr(self) -> int:
        return int(self.raw.mc_ptr + self.layout.flag_offset)

    def close(self):
        if not self.raw.handle:
            return
        for s in self.slabs:
            torch.cuda.synchronize(s.device)
        for s in self.slabs:
            if s.device != self.map_device:   # unbind the other members; bz_mc_free does the mapper
                self.lib.bz_mc_unbind(self.raw, s.device, self.nbytes)
        self.lib.bz_mc_free(self.raw, self.map_device, self.nbytes)


GATE_MODE = os.environ.get("BZ_GATE", "kernel")


def gate(flag_ptr: int, value: int, stream_handle: int, mode: Optional[str] = None) -> None:
    """Block ``stream`` until the u32 at ``flag_ptr`` >= ``value``.

    ``kernel`` (default): a one-thread gate kernel spinning with ld.acquire.sys
    (bounded, ~µs wake-up).  ``memop``: cuStreamWaitValue32 in the stream front
    end (no SM, but its re-polling interval backs off: measured ~100 ms late
    wake-ups when the flag is raised by a peer GPU's NVLink atomics).
    """
    lib = cuda_lib()
    if (mode or GATE_MODE) == "memop":
        lib.bz_wait_layer(flag_ptr, value, stream_handle)
    else:
        lib.bz_wait_flag_kernel(flag_ptr, value, stream_handle)


def _stream_handle(stream, device: Optional[int] = None) -> int:
    if stream is None:
        return int(torch.cuda.current_stream(device).cuda_stream)
    return int(stream.cuda_stream)


# ---- host cache -------------------------------------------------------------------------


class HostCache:
    """The O(1) host copy of a shard: page-locked memory the copy engines read.

    ``shm_name`` backs it with /dev/shm so every GPU process of the host maps
    the same single copy (one copy per host, parampool.py one-copy policy).
    """

    def __init__(self, layout: SlabLayout, shm_name: Optional[str] = None, create: bool = True):
        self.layout = layout
        nbytes = layout.data_bytes
        if shm_name:
            path = f"/dev/shm/{shm_name}"
            if create:
                with open(path, "wb") as f:
                    f.truncate(nbytes)
            self.array = np.memmap(path, dtype=np.uint8, mode="r+", shape=(nbytes,))
            self.tensor = torch.from_numpy(self.array)
        else:
            self.tensor = torch.empty(nbytes, dtype=torch.uint8)
        self.path = f"/dev/shm/{shm_name}" if shm_name else None
        cudart = torch.cuda.cudart()
        rc = cudart.cudaHostRegister(self.tensor.data_ptr(), nbytes, 1 | 2)  # portable | mapped
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister failed ({rc})")
        self.registered = True
        self.tile_off_host = np.ascontiguousarray(layout.tile_off)

    @property
    def ptr(self) -> int:
        return int(self.tensor.data_ptr())

    def close(self, unlink: bool = False):
        if self.registered:
            torch.cuda.cudart().cudaHostUnregister(self.tensor.data_ptr())
            self.registered = False
        if unlink and self.path and os.path.exists(self.path):
            os.unlink(self.path)


# ---- plan roles ---------------------------------------------------------------------------


@dataclass
class Role:
    """What one node does in a plan (derived identically on every rank)."""

    node: str
    parent: Optional[str] = None          # edge sender (gpu or mem) that feeds this node
    children: list[str] = field(default_factory=list)   # chain edges out of this node
    fanout: list[str] = field(default_factory=list)     # NVLink siblings this rep serves
    rep: Optional[str] = None             # if this node is a fan-out sibling: its rep

    @property
    def receives(self) -> bool:
        return self.parent is not None or self.rep is not None


def plan_roles(plan: ScalePlan) -> dict[str, Role]:
    roles: dict[str, Role] = {}

    def role(n: str) -> Role:
        return roles.setdefault(n, Role(n))

    for e in plan.edges:
        role(e.src).children.append(e.dst)
        role(e.dst).parent = e.src
    for rep, sibs in plan.nvlink_fanout.items():
        role(rep).fanout = list(sibs)
        for s in sibs:
            role(s).rep = rep
    return roles


def expand_tp(plan: ScalePlan, tp: int) -> list[ScalePlan]:
    """Per-TP-rank plans: rank r of every anchor gpu<g> is gpu<g+r> (simcore.py:321-323)."""
    if tp == 1:
        return [plan]
    from .planner import PlanEdge

    def shift(n: str, r: int) -> str:
        return f"gpu{int(n[3:]) + r}" if n.startswith("gpu") else n

    out = []
    for r in range(tp):
        edges = [PlanEdge(shift(e.src, r), shift(e.dst, r), e.gbps, e.kind) for e in plan.edges]
        fan = {shift(k, r): [shift(s, r) for s in v] for k, v in plan.nvlink_fanout.items()}
        chains = [[shift(n, r) for n in c] for c in plan.chains]
        out.append(ScalePlan(edges=edges, chains=chains, nvlink_fanout=fan))
    return out


def merge_plans(plans: Sequence[ScalePlan]) -> ScalePlan:
    """Union of node-disjoint per-TP-rank plans; every rank derives its role from it,
    so collective setup (multicast groups) iterates the same list on every rank."""
    edges, chains, fan = [], [], {}
    for p in plans:
        edges.extend(p.edges)
        chains.extend(p.chains)
        fan.update(p.nvlink_fanout)
    return ScalePlan(edges=edges, chains=chains, nvlink_fanout=fan)


def host_fed_groups(plan: ScalePlan) -> dict[str, list[str]]:
    """rep -> [rep, *siblings] for every NVLink fan-out group whose rep is fed from a
    host cache (``mem<h> -> rep`` pcie edge plus ``nvlink_fanout[rep]``)."""
    roles = plan_roles(plan)
    return {rep: [rep] + list(sibs) for rep, sibs in plan.nvlink_fanout.items()
            if sibs and (roles[rep].parent or "").startswith("mem")}


def stripe_pieces(layout: SlabLayout, members: int, index: int) -> list[tuple[int, int]]:
    """Tile range [lo, hi) of every layer that member ``index`` of a striped host
    load stages: each layer's tiles split into ``members`` contiguous pieces, so
    every layer lands at the group's aggregate host rate."""
    if not 0 <= index < members:
        raise ValueError(f"member index {index} outside a group of {members}")
    out = []
    for k in range(layout.num_layers):
        t0, t1 = layout.tiles_of_layer(k)
        n = t1 - t0
        out.append((t0 + n * index // members, t0 + n * (index + 1) // members))
    return out


# ---- fan-out realisation ----------------------------------------------------------------------

# Per-destination GB/s of the two realisations of an NVLink fan-out group, 7B shard,
# measured on B200 by GPUs in the group (writer included):
#   2: single-process probe, 16-64 CTAs (profiles/r2_nvlink_probe_n2.jsonl): sibling-chain
#      hop (k_push_tiles) 717, NVLS multimem.st 565 -- flat from 48 to 148 CTAs and for
#      4/8/16 stores in flight per thread, i.e. a multimem store-rate ceiling, not occupancy
#   4: multi-process bench (profiles/r1_nvls_vs_chain_n4.txt): chain 691, NVLS 530
MEASURED_FANOUT_GBPS = {2: {"chain": 717.0, "nvls": 565.0}, 4: {"chain": 691.0, "nvls": 530.0}}


def choose_fanout(group_size: int, table: Optional[dict] = None) -> str:
    """``auto`` realisation of a fan-out group of ``group_size`` GPUs: the faster one
    per destination in the measurement for the largest measured size <= the group
    (both realisations are receiver-count independent once pipelined, so the nearest
    smaller measurement stands for larger groups)."""
    table = MEASURED_FANOUT_GBPS if table is None else table
    if group_size <= 1 or not table:
        return "chain"
    keys = sorted(k for k in table if k <= group_size) or [min(table)]
    row = table[keys[-1]]
    return max(("chain", "nvls"), key=lambda m: (row.get(m, 0.0), m == "chain"))


# ---- executor -------------------------------------------------------------------------------


class ScaleExecutor:
    """Runs one node's share of a plan on its GPU, every epoch a fresh transfer.

    ``node_rank`` maps plan nodes (``gpu<i>``) to process ranks.  Every rank
    constructs the executor with the same plan; collective setup (fd exchange,
    multicast binding) happens in ``__init__``.
    """

    def __init__(self, fabric: Fabric, plan: ScalePlan, slab: DeviceSlab,
                 node_rank: dict[str, int], host_cache: Optional[HostCache] = None,
                 engine: int = ENGINE_VECTOR, nctas: int = 32, fanout_mode: str = "auto",
                 stage_engine: str = "ce", tiles_per_copy: int = 128, host_stripe: bool = True,
                 ce_tiles_per_copy: int = 0):
        self.fabric = fabric
        self.plan = plan
        # tiles per copy-engine memcpy of an ENGINE_CE chain hop (0: CE_TILES_PER_COPY) and
        # of a bz_push_tiles_ce2 hop (0: CE2_TILES_PER_COPY)
        self.ce_tiles = ce_tiles_per_copy or CE_TILES_PER_COPY
        self.ce2_tiles = ce_tiles_per_copy
        self.slab = slab
        self.layout = slab.layout
        self.node_rank = dict(node_rank)
        self.rank_node = {r: n for n, r in node_rank.items()}
        self.node = self.rank_node.get(fabric.rank)
        self.roles = plan_roles(plan)
        self.role = self.roles.get(self.node, Role(self.node)) if self.node else Role("")
        self.host_cache = host_cache
        self.engine = engine
        self.nctas = nctas
        self.stage_engine = stage_engine
        self.tiles_per_copy = tiles_per_copy
        self.lib = cuda_lib()
        if fanout_mode == "auto":
            sizes = [len(v) + 1 for v in plan.nvlink_fanout.values()]
            fanout_mode = choose_fanout(max(sizes) if sizes else 1)
        self.fanout_mode = fanout_mode
        # every rank exports its slab (and says whether it holds a host-cache view);
        # peers it sends to are imported below
        exports = fabric.allgather((self.node, slab.export(), host_cache is not None))
        # (bystander ranks of a smaller plan join with None)
        with_cache = {e[0] for e in exports if e is not None and e[0] is not None and e[2]}
        # striped host load: a host-fed rep and its NVLink siblings each stage one
        # piece of every layer over their own PCIe link and forward it to the others
        # (only for groups whose every member maps the host copy)
        groups = host_fed_groups(plan) if host_stripe and stage_engine == "ce" else {}
        self.stripe_groups = {rep: m for rep, m in groups.items() if all(n in with_cache for n in m)}
        self.stripe_members: Optional[list[str]] = None
        for members in self.stripe_groups.values():
            if self.node in members:
                self.stripe_members = members
        dev = torch.device("cuda", fabric.device)
        self.streams = {k: torch.cuda.Stream(device=dev)
                        for k in ("copy", "fan", "track", "stage", "ceflag", "cegate")}
        self.epoch = 0
        self._tile_off_host = np.ascontiguousarray(self.layout.tile_off)
        self.writers = self._fanout_writers() if fanout_mode == "nvls" else {}
        self._stripe_ids = None
        if self.stripe_members is not None:
            pieces = stripe_pieces(self.layout, len(self.stripe_members),
                                   self.stripe_members.index(self.node))
            self._pieces = pieces
            ids = np.concatenate([np.arange(lo, hi, dtype=np.int32) for lo, hi in pieces])
            self._stripe_ids = torch.from_numpy(ids).to(dev)

        self.peers: dict[str, PeerSlab] = {}
        for n in self._feeds()[0] + self._stripe_peers():
            r = self.node_rank[n]
            pid, fd, nbytes = exports[r][1]
            self.peers[n] = PeerSlab(fabric.device, pid, fd, nbytes, self.layout)
        # a pulled hop: map the sender's slab here
        self.pull_from = self._pull_source()
        self.pull_peer: Optional[PeerSlab] = None
        if self.pull_from is not None:
            pid, fd, nbytes = exports[self.node_rank[self.pull_from]][1]
            self.pull_peer = PeerSlab(fabric.device, pid, fd, nbytes, self.layout)
        fabric.barrier()
        self.mc_out: list[MulticastGroup] = []     # groups this rank writes
        self._mc_all: list[MulticastGroup] = []
        if self.fanout_mode == "nvls":
            # one multicast object per fan-out group, built collectively in plan order
            for rep, (writer, members) in self.writers.items():
                ranks = [self.node_rank[n] for n in members]
                grp = MulticastGroup(fabric, slab, ranks)
                self._mc_all.append(grp)
                if self.node == writer:
                    self.mc_out.append(grp)

    def _fanout_writers(self) -> dict[str, tuple[str, list[str]]]:
        """rep -> (writer, multicast members) for every NVLink fan-out group.

        NVLS replicates a multimem.st to every bound member, the writer included.
        If the representative is fed over NVLink by a root source (1 -> N on one
        box: ``gpu0 -> gpu1`` + ``gpu1 => {gpu2..}``), the source writes the group
        {source, rep, siblings} itself: one stream out of the source, and the echo
        lands on the source's idle ingress instead of doubling the rep's ingress.
        Otherwise (rep staged from the host cache over PCIe, or a relayed rep) the
        rep writes {rep, siblings} as it receives.
        """
        out = {}
        for rep, sibs in self.plan.nvlink_fanout.items():
            if rep in self.stripe_groups:
                continue
            parent = self.roles[rep].parent
            writer = rep
            if parent is not None and parent.startswith("gpu"):
                edge = next(e for e in self.plan.edges if e.dst == rep)
                prole = self.roles[parent]
                if edge.kind == "nvlink" and prole.parent is None and prole.rep is None:
                    writer = parent
            members = ([writer] if writer != rep else []) + [rep] + list(sibs)
            out[rep] = (writer, members)
        return out

    # chain children, plus siblings when the fan-out is served by unicast
    def _targets_for(self, node: Optional[str]) -> list[str]:
        role = self.roles.get(node) if node else None
        if role is None:
            return []
        if any(node in m for m in self.stripe_groups.values()):
            # chain children get the whole slab (relayed); the group peers get this
            # member's pieces (_stripe_peers)
            return list(role.children)
        covered = {rep for rep, (w, _) in self.writers.items() if w == node and w != rep}
        out = [c for c in role.children if c not in covered]
        if self.fanout_mode == "chain" and role.fanout:
            out.append(role.fanout[0])
        if self.fanout_mode == "chain" and role.rep is not None:
            sibs = self.plan.nvlink_fanout[role.rep]
            i = sibs.index(node)
            if i + 1 < len(sibs):
                out.append(sibs[i + 1])
        if self.fanout_mode == "star" and role.fanout:
            out.extend(role.fanout)
        return out

    def _unicast_targets(self) -> list[str]:
        return self._targets_for(self.node)

    def _pulled(self, sender: str, dst: str) -> bool:
        """The hop sender -> dst is pulled by dst: auto engine, GPU to GPU, the sender a
        source (receives nothing, not a striped host-load member), dst a leaf."""
        srole = self.roles.get(sender)
        return (self.engine == ENGINE_AUTO and sender.startswith("gpu") and dst.startswith("gpu")
                and srole is not None and not srole.receives and not self._forwards(dst)
                and not any(sender in m for m in self.stripe_groups.values()))

    def _pull_source_of(self, node: Optional[str]) -> Optional[str]:
        """The node ``node`` pulls its shard from, if any."""
        role = self.roles.get(node) if node else None
        if role is None or not role.receives:
            return None
        for n in self.roles:
            if node in self._targets_for(n) and self._pulled(n, node):
                return n
        return None

    def _pull_source(self) -> Optional[str]:
        return self._pull_source_of(self.node)

    def _stripe_peers(self) -> list[str]:
        if self.stripe_members is None:
            return []
        return [n for n in self.stripe_members if n != self.node]

    def _staged(self) -> bool:
        """This GPU copies (part of) the shard from a host cache."""
        return self.stripe_members is not None or (
            self.role.parent is not None and self.role.parent.startswith("mem"))

    def _feeds(self) -> tuple[list[str], bool]:
        """(unicast destinations this node pushes to, relay?) -- pulled hops excluded."""
        return [n for n in self._unicast_targets() if not self._pulled(self.node, n)], self.role.receives

    def dominant_stream(self) -> Optional[str]:
        """Stream of this rank's bulk mover (for per-kernel timing), if any."""
        if self._staged():
            return "stage"
        if self.mc_out:
            return "fan"
        if self._feeds()[0] or self.pull_peer is not None:
            return "copy"
        return None

    def launch(self, epoch: Optional[int] = None, track: bool = True, kernel_events=None,
               async_stage: bool = False):
        """Enqueue this rank's work for a new transfer; returns the epoch.

        ``kernel_events=(start, end)`` brackets the bulk mover on its own stream.
        ``async_stage``: host-cache staging is enqueued by a helper thread (call
        ``join_stage``/``synchronize`` before relying on the stage stream).
        """
        if async_stage and kernel_events is not None:
            raise ValueError("kernel_events need a synchronous enqueue")
        self.epoch = epoch if epoch is not None else self.epoch + 1
        e = self.epoch
        lay, slab = self.layout, self.slab
        st = self.streams
        dom = self.dominant_stream()
        if kernel_events is not None and dom is not None:
            kernel_events[0].record(st[dom])
        staged = self._staged()
        # a locally staged slab is published in-stream after each layer; a striped
        # member also receives pieces from its peers, so the tracker publishes
        self_published = staged and self.stage_engine == "ce" and self.stripe_members is None
        if self.role.receives and (track or staged):
            # reset loaded_layers and stamp this rank's launch time
            stream = st["stage"] if self_published else st["track"]
            self.lib.bz_publish_layer(slab.loaded.data_ptr(), 0, slab.stamps.data_ptr()
                                      + 8 * lay.num_layers, stream.cuda_stream)
        if staged:
            if async_stage:
                # a few thousand copy-engine calls take host time; let a helper
                # thread enqueue them so the caller can enqueue compute meanwhile
                import threading

                def worker():
                    try:
                        torch.cuda.set_device(self.fabric.device)  # new threads start on device 0
                        self._stage(e)
                    except BaseException as exc:  # surfaced by join_stage()
                        self._stage_error = exc

                self._stage_error = None
                self._stage_thread = threading.Thread(target=worker, daemon=True)
                self._stage_thread.start()
            else:
                self._stage(e)
        if self.role.receives and track and not self_published:
            # a peer (or a staging kernel) produces the tiles: one-warp in-order tracker
            self.lib.bz_track_layers(slab.flags_ptr, slab.layer_tile.data_ptr(), lay.num_layers, e,
                                     slab.loaded.data_ptr(), slab.stamps.data_ptr(),
                                     st["track"].cuda_stream)
        dsts, relay = self._feeds()
        if dsts and self._ce2_hop(dsts, relay):
            n = dsts[0]
            per_copy = self._ce_tiles()
            if relay:   # gates ahead on their own stream: the copy engine runs back to back
                self.lib.bz_push_tiles_ce_gated(slab.ptr, self.peers[n].ptr, self.peers[n].flags_ptr,
                                                slab.flags_ptr, self._tile_off_host.ctypes.data, 0, lay.ntiles,
                                                per_copy, e, st["copy"].cuda_stream, st["ceflag"].cuda_stream,
                                                st["cegate"].cuda_stream)
            else:
                self.lib.bz_push_tiles_ce2(slab.ptr, self.peers[n].ptr, self.peers[n].flags_ptr, None,
                                           self._tile_off_host.ctypes.data, 0, lay.ntiles, per_copy, e,
                                           st["copy"].cuda_stream, st["ceflag"].cuda_stream)
        elif dsts and self.engine == ENGINE_CE:
            for n in dsts:
                self.lib.bz_push_tiles_ce(slab.ptr, self.peers[n].ptr, self.peers[n].flags_ptr,
                                          slab.flags_ptr if relay else None,
                                          self._tile_off_host.ctypes.data, 0, lay.ntiles,
                                          self.ce_tiles, e, st["copy"].cuda_stream)
        elif dsts:
            ptrs = ptr_array([self.peers[n].ptr for n in dsts])
            flags = ptr_array([self.peers[n].flags_ptr for n in dsts])
            sm_engine = ENGINE_VECTOR if self.engine == ENGINE_AUTO else self.engine
            self.lib.bz_push_tiles(slab.ptr, ptrs, flags, len(dsts),
                                   slab.flags_ptr if relay else None, slab.tile_off.data_ptr(),
                                   0, lay.ntiles, e, self.nctas, sm_engine, st["copy"].cuda_stream)
        if self.pull_peer is not None:
            # pull: this GPU's SMs read the source's slab and publish the local tile flags
            self.lib.bz_pull_tiles(self.pull_peer.ptr, slab.ptr, slab.flags_ptr, None, None,
                                   slab.tile_off.data_ptr(), 0, lay.ntiles, e,
                                   max(self.nctas, PULL_CTAS, self.fabric.sm_count), st["copy"].cuda_stream)
        peers = self._stripe_peers()
        for i in range(0, len(peers), MAX_DST):
            # forward this member's pieces (gated on its own staged flags) to the group,
            # at most MAX_DST peers per launch
            part = peers[i:i + MAX_DST]
            self.lib.bz_push_tile_list(slab.ptr, ptr_array([self.peers[n].ptr for n in part]),
                                       ptr_array([self.peers[n].flags_ptr for n in part]), len(part),
                                       slab.flags_ptr, slab.tile_off.data_ptr(), self._stripe_ids.data_ptr(),
                                       int(self._stripe_ids.numel()), e, self.nctas, st["copy"].cuda_stream)
        for grp in self.mc_out:
            self.lib.bz_multicast_tiles(slab.ptr, grp.ptr, grp.flags_ptr,
                                        slab.flags_ptr if relay else None, slab.tile_off.data_ptr(),
                                        0, lay.ntiles, e, self.nctas, st["fan"].cuda_stream)
        if kernel_events is not None and dom is not None:
            kernel_events[1].record(st[dom])
        return e

    def _forwards(self, node: str) -> bool:
        """``node`` relays what it receives (chain child, fan-out, or a next sibling)."""
        r = self.roles.get(node)
        if r is None:
            return False
        if r.children or r.fanout:
            return True
        if r.rep is not None:
            sibs = self.plan.nvlink_fanout[r.rep]
            return sibs.index(node) + 1 < len(sibs)
        return False

    def _ce2_hop(self, dsts, relay) -> bool:
        """This node's (non-pulled) single-destination hop runs on the copy engines: always
        under ENGINE_CE2; under auto when the hop is part of a relay chain (this node
        relays, or its destination does) -- the whole chain then moves in copy-engine
        groups (a copy-engine hop into an SM-push relay made its forwarding bursty)."""
        if len(dsts) != 1 or self.stripe_members is not None:
            return False
        if self.engine == ENGINE_CE2:
            return True
        return self.engine == ENGINE_AUTO and (relay or self._forwards(dsts[0]))

    def _ce_tiles(self) -> int:
        if self.ce2_tiles:
            return self.ce2_tiles
        return CE_CHAIN_TILES_PER_COPY if self.engine == ENGINE_AUTO else CE2_TILES_PER_COPY

    def kernels_per_launch(self) -> int:
        """Our kernels one ``launch`` enqueues on this rank (CE memcpys excluded)."""
        n = 0
        staged = self._staged()
        striped = self.stripe_members is not None
        if self.role.receives:
            n += 1  # reset/publish
            if not (staged and self.stage_engine == "ce") or striped:
                n += 1  # tracker
        if striped:
            n += sum((hi - lo + self.tiles_per_copy - 1) // self.tiles_per_copy for lo, hi in self._pieces)
            n += (len(self._stripe_peers()) + MAX_DST - 1) // MAX_DST  # tile-list pushes
        elif staged:
            if self.stage_engine == "ce":
                lay = self.layout
                for k in range(lay.num_layers):
                    t0, t1 = lay.tiles_of_layer(k)
                    n += (t1 - t0 + self.tiles_per_copy - 1) // self.tiles_per_copy + 1
            else:
                n += 1
        if self.pull_peer is not None:
            n += 1  # the pull kernel
        dsts = self._feeds()[0]
        if dsts and self._ce2_hop(dsts, self.role.receives):
            per_copy = self._ce_tiles()
            groups = (self.layout.ntiles + per_copy - 1) // per_copy
            n += groups * (2 if self.role.receives else 1)   # flag kernels [+ relay gates]
        elif dsts and self.engine == ENGINE_CE:
            groups = (self.layout.ntiles + self.ce_tiles - 1) // self.ce_tiles
            per_group = 2 if self.role.receives else 1  # [gate] + flag kernel (memcpy not counted)
            n += len(dsts) * groups * per_group
        elif dsts:
            n += 1
        return n + len(self.mc_out)

    def _stage(self, e: int):
        hc, slab, lay = self.host_cache, self.slab, self.layout
        if hc is None:
            raise RuntimeError(f"{self.node} stages from a host cache but none was given")
        s = self.streams["stage"].cuda_stream
        if self.stripe_members is not None:
            # this member's piece of every layer, in layer order; the tracker publishes
            for lo, hi in self._pieces:
                self.lib.bz_stage_tiles_ce(hc.ptr, slab.ptr, slab.flags_ptr, hc.tile_off_host.ctypes.data,
                                           lo, hi, self.tiles_per_copy, e, s)
        elif self.stage_engine == "ce":
            # copy engines, layer by layer; each layer is published in-stream right
            # after its last tile (no spinning tracker on a locally produced slab)
            for k in range(lay.num_layers):
                t0, t1 = lay.tiles_of_layer(k)
                self.lib.bz_stage_tiles_ce(hc.ptr, slab.ptr, slab.flags_ptr,
                                           hc.tile_off_host.ctypes.data, t0, t1,
                                           self.tiles_per_copy, e, s)
                self.lib.bz_publish_layer(slab.loaded.data_ptr(), k + 1,
                                          slab.stamps.data_ptr() + 8 * k, s)
        else:
            self.lib.bz_stage_tiles_sm(hc.ptr, slab.ptr, slab.flags_ptr, slab.tile_off.data_ptr(),
                                       0, lay.ntiles, e, self.nctas, s)

    def join_stage(self):
        t = getattr(self, "_stage_thread", None)
        if t is not None:
            t.join()
            self._stage_thread = None
            if self._stage_error is not None:
                err, self._stage_error = self._stage_error, None
                raise RuntimeError("host-cache staging enqueue failed") from err

    def synchronize(self):
        self.join_stage()
        for s in self.streams.values():
            s.synchronize()

    def layer_arrivals_ms(self) -> list[float]:
        """Per-layer arrival on this GPU, ms after this rank's launch (receivers only)."""
        st = self.slab.stamps.cpu().tolist()
        t0 = st[self.layout.num_layers]
        return [(x - t0) / 1e6 for x in st[: self.layout.num_layers]]

    def close(self):
        self.synchronize()
        for p in self.peers.values():
            p.close()
        if self.pull_peer is not None:
            self.pull_peer.close()
            self.pull_peer = None
        for grp in self._mc_all:
            grp.close()


# ---- loopback (several slabs driven by one process on one GPU) -------------------------------


def execute_plan_loopback(plan: ScalePlan, slabs: dict[str, DeviceSlab], epoch: int,
                          host_cache: Optional[HostCache] = None, engine: int = ENGINE_VECTOR,
                          nctas: int = 32, stage_engine: str = "ce", stream=None) -> None:
    """Execute ``plan`` with every node's slab on this GPU, hop by hop on one stream.

    The same kernels as the multi-GPU path; hops are stream-ordered, so a relay
    finds its upstream flags already raised (no cross-kernel spinning on one GPU).
    Fan-out groups are served as a sibling chain.
    """
    lib = cuda_lib()
    s = _stream_handle(stream)
    roles = plan_roles(plan)
    order = _topological(plan)
    for node in order:
        role = roles[node]
        if node.startswith("mem"):
            continue
        slab = slabs[node]
        lay = slab.layout
        published = False
        if role.parent is not None and role.parent.startswith("mem"):
            if host_cache is None:
                raise RuntimeError("host cache required")
            if stage_engine == "ce":
                # layer by layer, each published in-stream after its last copy (as ScaleExecutor)
                for k in range(lay.num_layers):
                    t0, t1 = lay.tiles_of_layer(k)
                    lib.bz_stage_tiles_ce(host_cache.ptr, slab.ptr, slab.flags_ptr,
                                          host_cache.tile_off_host.ctypes.data, t0, t1, 8, epoch, s)
                    lib.bz_publish_layer(slab.loaded.data_ptr(), k + 1, slab.stamps.data_ptr() + 8 * k, s)
                published = True
            else:
                lib.bz_stage_tiles_sm(host_cache.ptr, slab.ptr, slab.flags_ptr,
                                      slab.tile_off.data_ptr(), 0, lay.ntiles, epoch, nctas, s)
        outs = list(role.children)
        if role.fanout:
            outs.append(role.fanout[0])
        if role.rep is not None:
            sibs = plan.nvlink_fanout[role.rep]
            i = sibs.index(node)
            if i + 1 < len(sibs):
                outs.append(sibs[i + 1])
        if outs:
            ptrs = ptr_array([slabs[n].ptr for n in outs])
            flags = ptr_array([slabs[n].flags_ptr for n in outs])
            lib.bz_push_tiles(slab.ptr, ptrs, flags, len(outs),
                              slab.flags_ptr if role.receives else None, slab.tile_off.data_ptr(),
                              0, lay.ntiles, epoch, nctas, engine, s)
        if role.receives and not published:
            lib.bz_track_layers(slab.flags_ptr, slab.layer_tile.data_ptr(), lay.num_layers, epoch,
                                slab.loaded.data_ptr(), slab.stamps.data_ptr(), s)


def _topological(plan: ScalePlan) -> list[str]:
    """Senders before receivers: plan edge order, then fan-out groups after their rep."""
    order: list[str] = []
    seen = set()

    def add(n):
        if n not in seen:
            seen.add(n)
            order.append(n)

    for e in plan.edges:
        add(e.src)
        add(e.dst)
        for rep in [e.dst]:
            for s in plan.nvlink_fanout.get(rep, []):
                add(s)
    for rep, sibs in plan.nvlink_fanout.items():
        add(rep)
        for s in sibs:
            add(s)
    return order
