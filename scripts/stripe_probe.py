"""Probe the striped host-cache load step by step (torchrun, 2+ GPUs), with a
watchdog that dumps every thread's stack if a step hangs."""
import faulthandler
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
faulthandler.dump_traceback_later(int(os.environ.get("BZ_WATCHDOG_S", "150")), exit=True)

import torch  # noqa: E402

from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200.dataplane import DeviceSlab, Fabric  # noqa: E402
from paper_2412_17246_b200.scaleup import ScaleUpSession, plan_for, plan_host_cache  # noqa: E402

T0 = time.perf_counter()


def log(*a):
    print(f"[r{os.environ.get('RANK')} {time.perf_counter() - T0:7.2f}s]", *a, flush=True)


fabric = Fabric.from_env()
N = fabric.world
arch = S.ARCHS[os.environ.get("BZ_ARCH", "llama2-7b")]
layout = S.SlabLayout.for_arch(arch, tile_bytes=1 << 20)
gpus = [f"gpu{i}" for i in range(N)]
node_rank = {g: i for i, g in enumerate(gpus)}
plan, _, _ = plan_for(arch, ["mem0"], gpus)
log("plan", [(e.src, e.dst) for e in plan.edges], plan.nvlink_fanout)


def fill(host):
    log("fill: device slab")
    tmp = DeviceSlab(layout, fabric.device)
    tmp.fill_random(241217)
    log("fill: d2h")
    cpu = tmp.data.cpu()
    log("fill: copy into host cache")
    host.copy_(cpu)
    tmp.close()
    log("fill: done")


private = os.environ.get("BZ_PRIVATE_HC") == "1"
stripe = os.environ.get("BZ_STRIPE", "1") == "1"
if private:
    from paper_2412_17246_b200.dataplane import HostCache
    hc = HostCache(layout)
    fill(hc.tensor)
else:
    hc = plan_host_cache(fabric, layout, plan, node_rank, fill, tag="probe", host_stripe=stripe)
log("host cache", None if hc is None else hc.ptr, "private" if private else "shm")
sess = ScaleUpSession(fabric, layout, plan, node_rank, host_cache=hc, nctas=48, host_stripe=stripe)
log("session ready; striped:", sess.executor.stripe_members)
ex = sess.executor
side = torch.cuda.Stream()
pin = torch.empty(sess.slab.flags.numel(), dtype=torch.int32).pin_memory()
pld = torch.empty(1, dtype=torch.int32).pin_memory()


def poll(tag, e, stream, secs=8.0):
    t = time.perf_counter()
    while time.perf_counter() - t < secs:
        if stream.query():
            break
        time.sleep(0.2)
    with torch.cuda.stream(side):
        pin.copy_(sess.slab.flags.view(torch.int32), non_blocking=True)
        pld.copy_(sess.slab.loaded, non_blocking=True)
    side.synchronize()
    mine = ex._stripe_ids.cpu().long() if ex._stripe_ids is not None else None
    own = int((pin[mine] == e).sum()) if mine is not None else -1
    log(f"{tag}: stream done={stream.query()} after {time.perf_counter() - t:.2f}s; flags at epoch "
        f"{int((pin == e).sum())}/{pin.numel()} (own pieces {own}/{0 if mine is None else mine.numel()}) "
        f"loaded={int(pld)}")


fabric.barrier()
torch.cuda.synchronize()
if ex.stripe_members is not None and os.environ.get("BZ_MANUAL") == "1":
    e = 1
    ex.epoch = e
    st = ex.streams
    ex._stage(e)
    poll("stage only", e, st["stage"])
    fabric.barrier()
    peers = ex._stripe_peers()
    from paper_2412_17246_b200.dataplane import ptr_array
    rc = ex.lib.bz_push_tile_list(sess.slab.ptr, ptr_array([ex.peers[n].ptr for n in peers]),
                                  ptr_array([ex.peers[n].flags_ptr for n in peers]), len(peers),
                                  sess.slab.flags_ptr, sess.slab.tile_off.data_ptr(), ex._stripe_ids.data_ptr(),
                                  int(ex._stripe_ids.numel()), e, ex.nctas, st["copy"].cuda_stream)
    log("push rc", rc)
    poll("push", e, st["copy"])
    fabric.barrier()
    ex.lib.bz_track_layers(sess.slab.flags_ptr, sess.slab.layer_tile.data_ptr(), layout.num_layers, e,
                           sess.slab.loaded.data_ptr(), sess.slab.stamps.data_ptr(), st["track"].cuda_stream)
    poll("track", e, st["track"])
    fabric.barrier()
    ex.synchronize()
    log("manual epoch verify", sess.verify(e))
for i in range(3):
    r = sess.run(verify=(i == 0))
    log(f"run {i}: {r.elapsed_ms:.1f} ms verified={r.verified} first/last layer "
        f"{r.layer_ms[0] if r.layer_ms else None} {r.layer_ms[-1] if r.layer_ms else None}")
sess.close()
if hc is not None:
    hc.close()
log("done")
