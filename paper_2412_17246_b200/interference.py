"""Serving traffic vs scale traffic on NVLink, with the serving flow MEASURED
(planner.py:147-159, 265-285; simcore.py:462-514).

Collective over a ``Fabric`` of >= 4 ranks (one per GPU):
  gpu0 = prefill instance pushing KV cache to gpu1 (decode) continuously;
  gpu1 = decode instance; both hold the Llama-2 7B weights; gpu2, gpu3 = new instances.

1. The KV stream runs alone; its measured rate (bytes / CUDA-event time, max over
   ranks) is registered in the FlowSet as the ``kvcache`` flow gpu0 -> gpu1
   (``MeasuredFlow``).
2. ``generate_plan(prune=True)`` on that FlowSet drops the serving sender gpu0 and
   scales from gpu1 (its NVLink egress is idle); the "naive" plan is forced to
   send from gpu0, whose egress the KV stream occupies.
3. Both plans execute with the KV stream running; reported: scale-up time, the KV
   stream's rate during the scale-up, bit-exactness, and what the planner's own
   interference check said about each plan under the measured flow.
"""

from __future__ import annotations

import torch

from . import planner
from .dataplane import Fabric
from .kvflows import MeasuredFlow
from .planner import PlanEdge, ScalePlan, build_scale_request, generate_plan, plan_is_interference_free
from .scaleup import ScaleUpSession
from .slab import LLAMA2_7B, LlamaArch, SlabLayout, model_spec_for
from .topology import FlowSet, load_topology


def _max_over_ranks(x: float, fabric: Fabric) -> float:
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_interference(fabric: Fabric, arch: LlamaArch = LLAMA2_7B, kv_bytes: int = 2 << 30, reps: int = 6) -> dict:
    if fabric.world < 4:
        raise ValueError("needs 4 GPUs (prefill, decode, two new instances)")
    import torch.distributed as dist
    rank = fabric.rank
    node_rank = {f"gpu{i}": i for i in range(fabric.world)}
    layout = SlabLayout.for_arch(arch, tile_bytes=1 << 20)
    model = model_spec_for(arch)
    topo = load_topology("b200-hgx")
    flows = FlowSet(topo)
    kv_layout = SlabLayout.uniform(8, kv_bytes // 8, tile_bytes=1 << 20)
    kv_plan = ScalePlan(edges=[PlanEdge("gpu0", "gpu1", 7200.0, "nvlink")], chains=[["gpu0", "gpu1"]])
    kv = ScaleUpSession(fabric, kv_layout, kv_plan, node_rank, nctas=32, seed=5)

    def kv_window(n: int) -> float:
        fabric.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(kv.executor.streams["copy"])
        for _ in range(n):
            kv.executor.launch(track=False)
        e1.record(kv.executor.streams["copy"])
        kv.executor.synchronize()
        return _max_over_ranks(e0.elapsed_time(e1) if rank == 0 else 0.0, fabric)

    kv_window(1)                                  # warm
    alone_ms = kv_window(4)
    flow = MeasuredFlow(flows, "gpu0", "gpu1", "kvcache")
    flow.update(4 * kv_bytes, alone_ms)          # the FlowSet now carries the measured KV rate
    req = build_scale_request(model, ["gpu0", "gpu1"], ["gpu2", "gpu3"], topo, flows)
    pruned = generate_plan(req, topo, flows, group=False, prune=True)
    naive = ScalePlan(edges=[PlanEdge("gpu0", "gpu2", 7200.0, "nvlink"), PlanEdge("gpu2", "gpu3", 7200.0, "nvlink")],
                      chains=[["gpu0", "gpu2", "gpu3"]])
    out = {"kv_alone_GBps": 4 * kv_bytes / (alone_ms / 1e3) / 1e9,
           "kv_flow_registered_gbps": flow.gbps, "kv_flow_clamped_to_free_capacity": flow.clamped,
           "request_out_gbps": {s.node: s.outcast_gbps for s in req.sources}, "plans": {}}
    for name, plan in (("pruned", pruned), ("naive", naive)):
        sess = ScaleUpSession(fabric, layout, plan, node_rank, nctas=48)
        sess.run(verify=True)                     # warm + bit-exact
        fabric.barrier()
        torch.cuda.synchronize()
        kv_e0, kv_e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kv_e0.record(kv.executor.streams["copy"])
        for _ in range(reps):
            kv.executor.launch(track=False)
        kv_e1.record(kv.executor.streams["copy"])
        res = sess.run(verify=True)
        kv.executor.synchronize()
        kv_ms = _max_over_ranks(kv_e0.elapsed_time(kv_e1) if rank == 0 else 0.0, fabric)
        scale_ms = _max_over_ranks(res.elapsed_ms, fabric)
        ok = torch.tensor([1.0 if res.verified else 0.0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        out["plans"][name] = {
            "edges": [(e.src, e.dst) for e in plan.edges],
            "interference_free_under_measured_flow": plan_is_interference_free(plan, flows, topo),
            "scale_up_ms": scale_ms, "kv_during_scale_GBps": reps * kv_bytes / (kv_ms / 1e3) / 1e9,
            "bit_exact": bool(ok.item() == 1.0)}
        sess.close()
    flow.release()
    kv.close()
    return out
