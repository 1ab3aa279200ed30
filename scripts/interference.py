"""Interference between serving (KV-cache) traffic and scale traffic on NVLink, and
what the planner's source pruning buys (planner.py:147-159,
265-285).  Run under torchrun with 4 GPUs:

  gpu0 = prefill instance, continuously pushing KV cache to gpu1 (decode);
  gpu1 = decode instance; both hold the Llama-2 7B weights;
  gpu2, gpu3 = new instances to scale up.

Case "pruned": the FlowSet carries the kvcache flow gpu0->gpu1, so
generate_plan(prune=True) drops gpu0 and scales from gpu1 (its NVLink egress
is idle -- only its ingress carries KV).  Case "naive": the plan is forced to
use gpu0, whose egress is shared with the KV stream.  Reported: scale-up time,
and the KV stream's throughput while the scale-up runs vs alone.
"""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2412_17246_b200 as ss  # noqa: E402
from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200.dataplane import Fabric  # noqa: E402
from paper_2412_17246_b200.scaleup import ScaleUpSession  # noqa: E402

KV_BYTES = 2 << 30   # one KV burst: 2 GiB (~ 13k tokens of 7B KV at 160 KB/token)


def max_over_ranks(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    fabric = Fabric.from_env()
    assert fabric.world >= 4, "needs 4 GPUs"
    rank = fabric.rank
    node_rank = {f"gpu{i}": i for i in range(fabric.world)}
    arch = S.LLAMA2_7B
    layout = S.SlabLayout.for_arch(arch, tile_bytes=1 << 20)
    model = S.model_spec_for(arch)
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    flows.register("gpu0", "gpu1", 2000.0, "kvcache")   # the serving flow the planner sees

    req = ss.build_scale_request(model, ["gpu0", "gpu1"], ["gpu2", "gpu3"], topo, flows)
    pruned = ss.generate_plan(req, topo, flows, group=False, prune=True)
    naive = ss.ScalePlan(edges=[ss.planner.PlanEdge("gpu0", "gpu2", 7200.0, "nvlink"),
                                ss.planner.PlanEdge("gpu2", "gpu3", 7200.0, "nvlink")],
                         chains=[["gpu0", "gpu2", "gpu3"]])
    kv_layout = S.SlabLayout.uniform(8, KV_BYTES // 8, tile_bytes=1 << 20)
    kv_plan = ss.ScalePlan(edges=[ss.planner.PlanEdge("gpu0", "gpu1", 7200.0, "nvlink")],
                           chains=[["gpu0", "gpu1"]])
    kv = ScaleUpSession(fabric, kv_layout, kv_plan, node_rank, nctas=32, seed=5)

    def kv_alone(reps=4):
        fabric.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            kv.executor.launch(track=False)
        kv.executor.synchronize()
        e1.record()
        e1.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) if rank == 0 else 0.0)
        return reps * KV_BYTES / (ms / 1e3) / 1e9

    out = {"kv_alone_GBps": kv_alone(), "plans": {}}
    for name, plan in (("pruned", pruned), ("naive", naive)):
        sess = ScaleUpSession(fabric, layout, plan, node_rank, nctas=48)
        sess.run(verify=True)  # warm + bit-exact check
        # scale-up with the KV stream running on gpu0 the whole time
        fabric.barrier()
        torch.cuda.synchronize()
        kv_e0, kv_e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 6
        kv_e0.record(kv.executor.streams["copy"])
        for _ in range(reps):
            kv.executor.launch(track=False)
        kv_e1.record(kv.executor.streams["copy"])
        res = sess.run(verify=True)
        kv.executor.synchronize()
        kv_ms = kv_e0.elapsed_time(kv_e1) if rank == 0 else 0.0
        scale_ms = max_over_ranks(res.elapsed_ms)
        kv_ms = max_over_ranks(kv_ms)
        ok = torch.tensor([1.0 if res.verified else 0.0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        out["plans"][name] = {
            "edges": [(e.src, e.dst) for e in plan.edges],
            "interference_free": ss.plan_is_interference_free(plan, flows, topo),
            "scale_up_ms": scale_ms, "kv_during_scale_GBps": reps * KV_BYTES / (kv_ms / 1e3) / 1e9,
            "bit_exact": bool(ok.item() == 1.0)}
        sess.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    kv.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BZ_WATCHDOG_S", "300")), exit=True)
    main()
