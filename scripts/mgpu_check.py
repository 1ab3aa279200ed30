"""Multi-GPU parity check of the data plane (run under torchrun, one process per GPU).

For every plan shape the reference planner produces on an HGX B200 box
(1->N grouped = rep + NVLS fan-out; 1->N chain; host cache -> rep -> fan-out),
every receiving GPU must hold the bit-exact source shard (tile fingerprints
vs the regenerated source), all tile flags must carry the epoch and the
tracker must have published every layer.  Prints one JSON line per case on
rank 0 and exits non-zero on any mismatch.
"""

import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200.dataplane import ENGINE_AUTO, ENGINE_TMA, ENGINE_VECTOR, DeviceSlab, Fabric  # noqa: E402
from paper_2412_17246_b200.scaleup import ScaleUpSession, plan_for, plan_host_cache  # noqa: E402


def main():
    arch = S.ARCHS[os.environ.get("BZ_ARCH", "tiny-4l")]
    tile = int(os.environ.get("BZ_TILE_KIB", "256")) * 1024
    fabric = Fabric.from_env()
    N, rank = fabric.world, fabric.rank
    gpus = [f"gpu{i}" for i in range(N)]
    node_rank = {g: i for i, g in enumerate(gpus)}
    layout = S.SlabLayout.for_arch(arch, tile_bytes=tile)
    failures = 0
    # (name, sources, targets, group, fanout realisation requested, engine); the
    # realisation actually used and the multicast groups built are printed per case
    cases = [
        ("grouped-nvls", ["gpu0"], gpus[1:], True, "nvls", ENGINE_VECTOR),
        ("grouped-chain", ["gpu0"], gpus[1:], True, "chain", ENGINE_VECTOR),
        ("chain-vector", ["gpu0"], gpus[1:], False, "auto", ENGINE_VECTOR),
        ("chain-tma", ["gpu0"], gpus[1:], False, "auto", ENGINE_TMA),
        ("chain-auto", ["gpu0"], gpus[1:], False, "auto", ENGINE_AUTO),
        ("hostcache-rep-nvls", ["mem0"], gpus, True, "nvls", ENGINE_VECTOR),
        ("hostcache-rep-chain", ["mem0"], gpus, True, "chain", ENGINE_VECTOR),
        ("hostcache-stripe", ["mem0"], gpus, True, "auto", ENGINE_VECTOR),
    ]

    def fill(host):
        tmp = DeviceSlab(layout, fabric.device)
        tmp.fill_random(241217)
        host.copy_(tmp.data.cpu())
        tmp.close()

    for name, srcs, tgts, group, fan, engine in cases:
        plan, _, _ = plan_for(arch, srcs, tgts, group=group)
        stripe = name == "hostcache-stripe"
        hc = plan_host_cache(fabric, layout, plan, node_rank, fill, host_stripe=stripe, tag=name.replace("-", "_"))
        t0 = time.perf_counter()
        # hostcache-rep: striping requested, but only the rep maps the host copy -> the
        # executor keeps the rep-only realisation
        sess = ScaleUpSession(fabric, layout, plan, node_rank, host_cache=hc, engine=engine,
                              nctas=16, fanout_mode=fan, seed=241217, host_stripe=True)
        if name.startswith("hostcache"):
            assert bool(sess.executor.stripe_groups) == stripe, (name, sess.executor.stripe_groups)
        oks, ms = [], []
        for _ in range(3):
            r = sess.run(verify=True)
            oks.append(bool(r.verified))
            ms.append(r.elapsed_ms)
        ok_t = torch.tensor([0.0 if all(oks) else 1.0], device="cuda")
        ms_t = torch.tensor([max(ms)], device="cuda")
        import torch.distributed as dist
        if N > 1:
            dist.all_reduce(ok_t)
            dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        failures += int(ok_t.item() > 0)
        if rank == 0:
            print(json.dumps({"case": name, "n_gpus": N, "arch": arch.name, "ok": ok_t.item() == 0,
                              "max_ms": ms_t.item(), "fanout_requested": fan,
                              "fanout_mode": sess.executor.fanout_mode,
                              "multicast_groups": len(sess.executor._mc_all),
                              "edges": [(e.src, e.dst) for e in plan.edges],
                              "fanout": plan.nvlink_fanout,
                              "striped": bool(sess.executor.stripe_groups),
                              "setup_s": time.perf_counter() - t0}), flush=True)
        sess.close()
        if hc is not None:
            hc.close()
        fabric.barrier()
    if N > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BZ_WATCHDOG_S", "240")), exit=True)
    main()
