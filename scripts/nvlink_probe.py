"""Single-process NVLink / NVLS probe of the tile movers (one process drives every GPU).

Why one process: ncu can only profile a single process, and a multicast object can
be bound by one process to slabs on several GPUs.  Cases (JSON line each):

  mc1      one-device multicast object (numDevices=1) bound to a second slab on
           cuda:0: k_multicast_tiles writes through the multicast VA, bytes and
           flags checked (what a 1-GPU box can run)
  ceiling  torch peer copy gpu0 -> gpu1 (copy engines) of the same bytes
  push     k_push_tiles gpu0 -> gpu1 peer mapping, engines x CTA counts
  mc       k_multicast_tiles from gpu0 into a multicast object bound to the slabs
           of gpu0..gpu{G-1} (the writer's own slab is a member: its echo lands on
           its idle ingress), unroll x CTA counts; bytes delivered per destination

``--once <case>`` runs one launch of one configuration (for ncu).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200._native import BzMc, cuda_lib, ptr_array  # noqa: E402
from paper_2412_17246_b200.dataplane import DeviceSlab, PeerSlab  # noqa: E402


def emit(d):
    print(json.dumps(d), flush=True)


class LocalMc:
    """Multicast object bound (by this one process) to slabs on several GPUs."""

    def __init__(self, slabs: list[DeviceSlab], map_dev: int):
        self.lib = cuda_lib()
        self.raw = BzMc()
        self.slabs = slabs
        nbytes = int(slabs[0].raw.bytes)
        self.lib.bz_mc_create(len(slabs), nbytes, self.raw)
        for s in slabs:
            self.lib.bz_mc_add_device(self.raw, s.device)
        for s in slabs:
            self.lib.bz_mc_bind(self.raw, s.device, s.raw, 0, 0, nbytes)
        self.lib.bz_mc_map(self.raw, map_dev)
        self.map_dev = map_dev
        self.nbytes = nbytes
        self.layout = slabs[0].layout

    @property
    def ptr(self):
        return int(self.raw.mc_ptr)

    @property
    def flags_ptr(self):
        return int(self.raw.mc_ptr + self.layout.flag_offset)

    def close(self):
        for s in self.slabs:
            torch.cuda.synchronize(s.device)
        # unmap + unbind the mapping device + release (the other members' bindings
        # go with the process; their slabs are not freed before exit)
        self.lib.bz_mc_free(self.raw, self.map_dev, self.nbytes)


def timed(fn, stream, reps=3):
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def check(dst: DeviceSlab, want: torch.Tensor, epoch: int) -> bool:
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)
    got = dst.fingerprints().cpu()
    fl = dst.flags.cpu()
    ok = bool(torch.equal(got, want)) and int(fl.min()) == epoch and int(fl.max()) == epoch
    if not ok:
        emit({"check": "mismatch", "device": dst.device, "tiles_equal": int((got == want).sum()),
              "tiles": int(want.numel()), "flag_min": int(fl.min()), "flag_max": int(fl.max()), "epoch": epoch})
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="llama2-7b")
    ap.add_argument("--tile-kib", type=int, default=1024)
    ap.add_argument("--ctas", default="16,32,48,64,96,148")
    ap.add_argument("--unrolls", default="4,8,16")
    ap.add_argument("--once", default=None, help="push|pull|mc|mc1|panels: one launch (for ncu)")
    ap.add_argument("--nctas", type=int, default=48)
    ap.add_argument("--gb", type=float, default=0.0, help="uniform payload of this many GB instead of --arch")
    args = ap.parse_args()
    G = torch.cuda.device_count()
    if args.gb > 0:
        lay = S.SlabLayout.uniform(32, int(args.gb * 1e9 / 32), tile_bytes=args.tile_kib * 1024)
    else:
        lay = S.SlabLayout.for_arch(S.ARCHS[args.arch], tile_bytes=args.tile_kib * 1024)
    lib = cuda_lib(0)
    for d in range(G):
        cuda_lib(d)
    torch.cuda.set_device(0)
    src = DeviceSlab(lay, 0)
    src.fill_random(99)
    want = src.fingerprints().cpu()
    stream = torch.cuda.Stream(device=0)
    epoch = [0]
    payload = lay.data_bytes

    def nxt():
        epoch[0] += 1
        return epoch[0]

    # ---- mc1: one-device multicast object on cuda:0 ----------------------------------
    if args.once in (None, "mc1"):
        dst = DeviceSlab(lay, 0)
        try:
            mc = LocalMc([dst], 0)
        except Exception as e:  # noqa: BLE001
            gmin, grec = ctypes.c_uint64(), ctypes.c_uint64()
            try:
                lib.bz_mc_granularity(0, 1, ctypes.byref(gmin), ctypes.byref(grec))
            except Exception:  # noqa: BLE001
                pass
            probe = {}
            for ndev in (1, 2):
                for size in (gmin.value, grec.value):
                    raw = BzMc()
                    try:
                        lib.bz_mc_create(ndev, size, raw)
                        probe[f"{ndev}dev_{size}"] = "ok"
                        lib.bz_mc_free(raw, 0, 0)
                    except Exception as e2:  # noqa: BLE001
                        probe[f"{ndev}dev_{size}"] = str(e2)[-60:]
            emit({"case": "mc1", "supported": False, "error": str(e)[:300], "slab_bytes": int(dst.raw.bytes),
                  "mc_gran_min": gmin.value, "mc_gran_rec": grec.value, "create_probe": probe})
            mc = None
        if mc is not None:
            e = nxt()
            fn = lambda: lib.bz_multicast_tiles(src.ptr, mc.ptr, mc.flags_ptr, None, src.tile_off.data_ptr(),  # noqa: E731
                                                0, lay.ntiles, e, args.nctas, stream.cuda_stream)
            ms = timed(fn, stream, reps=1 if args.once else 3)
            emit({"case": "mc1", "supported": True, "ok": check(dst, want, e), "ms": ms,
                  "GBps": payload / ms / 1e6, "nctas": args.nctas})
            mc.close()
        dst.close()
        if args.once:
            return
    if G < 2:
        emit({"case": "multi", "skipped": f"{G} GPU(s) visible"})
        return

    dsts = [DeviceSlab(lay, d) for d in range(1, G)]
    peer = dsts[0]
    pid, fd, nb = peer.export()
    mapped = PeerSlab(0, pid, fd, nb, lay)

    # ---- ceiling: torch peer copy --------------------------------------------------------
    if args.once is None:
        from paper_2412_17246_b200.dataplane import device_view
        n = min(payload, 4 << 30)
        a = src.data[:n]
        b = device_view(mapped.ptr, n, torch.uint8, torch.device("cuda", 0))  # gpu1's slab seen from gpu0
        with torch.cuda.stream(stream):
            ms = timed(lambda: b.copy_(a, non_blocking=True), stream)
        emit({"case": "ceiling", "what": "torch peer copy gpu0->gpu1 (copy engines)", "bytes": n,
              "GBps": n / ms / 1e6})

    # ---- push --------------------------------------------------------------------------------
    def push(nctas, engine):
        e = nxt()
        fn = lambda: lib.bz_push_tiles(src.ptr, ptr_array([mapped.ptr]), ptr_array([mapped.flags_ptr]), 1,  # noqa: E731
                                       None, src.tile_off.data_ptr(), 0, lay.ntiles, e, nctas, engine,
                                       stream.cuda_stream)
        return fn, e

    # ---- KV hand-over mover: strided panel prefixes into the peer (k_copy_panels) --------------
    def panels(nctas):
        # 7B KV shape of one sequence batch: 32 heads x 4 seqs panels of [s_max=2048, 128] bf16,
        # first 2000 tokens of each copied
        n_panels, s_max, hd, length = 128, 2048, 128, 2000
        stride = s_max * hd * 2
        nbytes = n_panels * length * hd * 2
        fn = lambda: lib.bz_copy_panels(src.ptr, mapped.ptr, n_panels, stride, stride, length * hd * 2,  # noqa: E731
                                        nctas, stream.cuda_stream)
        return fn, nbytes

    if args.once == "panels":
        fn, nb = panels(args.nctas)
        fn()
        torch.cuda.synchronize()
        emit({"case": "panels-once", "bytes": nb})
        return
    if args.once is None:
        for c in (64, 128, 148):
            fn, nb = panels(c)
            ms = timed(fn, stream)
            emit({"case": "copy_panels", "nctas": c, "bytes": nb, "ms": ms, "GBps": nb / ms / 1e6})

    if args.once == "push":
        fn, e = push(args.nctas, 0)
        fn()
        torch.cuda.synchronize()
        emit({"case": "push-once", "ok": check(peer, want, e)})
        return
    if args.once is None:
        for engine, ename in ((0, "vector"), (2, "vec256"), (1, "tma")):
            for c in [int(x) for x in args.ctas.split(",")]:
                fn, e = push(c, engine)
                ms = timed(fn, stream)
                emit({"case": "push", "engine": ename, "nctas": c, "ms": ms, "GBps": payload / ms / 1e6,
                      "ok": check(peer, want, e)})

    # ---- pull: the receiver's SMs read the sender's slab over NVLink (gpu1 <- gpu0) -----------
    if args.once in (None, "pull"):
        spid, sfd, snb = src.export()
        src_on1 = PeerSlab(1, spid, sfd, snb, lay)   # gpu0's slab mapped on gpu1
        stream1 = torch.cuda.Stream(device=1)
        lib1 = cuda_lib(1)

        def pull(nctas, engine):
            e = nxt()

            def fn():
                with torch.cuda.device(1):
                    if engine == "pull":   # bz_pull_tiles
                        lib1.bz_pull_tiles(src_on1.ptr, peer.ptr, peer.flags_ptr, None, None,
                                           peer.tile_off.data_ptr(), 0, lay.ntiles, e, nctas, stream1.cuda_stream)
                    else:                  # bz_push_tiles launched on the receiver (peer source)
                        lib1.bz_push_tiles(src_on1.ptr, ptr_array([peer.ptr]), ptr_array([peer.flags_ptr]), 1,
                                           None, peer.tile_off.data_ptr(), 0, lay.ntiles, e, nctas, engine,
                                           stream1.cuda_stream)
            return fn, e

        if args.once == "pull":
            fn, e = pull(args.nctas, "pull")
            fn()
            torch.cuda.synchronize(1)
            emit({"case": "pull-once", "ok": check(peer, want, e)})
            return
        for engine, ename in (("pull", "bz_pull_tiles"), (0, "vector"), (2, "vec256"), (1, "tma")):
            for c in [int(x) for x in args.ctas.split(",")]:
                fn, e = pull(c, engine)
                ms = timed(fn, stream1)
                emit({"case": "pull", "engine": ename, "nctas": c, "ms": ms, "GBps": payload / ms / 1e6,
                      "ok": check(peer, want, e)})

    # ---- copy-engine hop (no SM moves bytes): tiles per memcpy sweep ---------------------------
    if args.once is None:
        fstream = torch.cuda.Stream(device=0)
        for split in (False, True):
            for tpc in (16, 32, 64, 128):
                e = nxt()
                if split:   # flag kernels on their own stream: copies back to back
                    fn = lambda: lib.bz_push_tiles_ce2(src.ptr, mapped.ptr, mapped.flags_ptr, None,  # noqa: E731
                                                       lay.tile_off.ctypes.data, 0, lay.ntiles, tpc, e,
                                                       stream.cuda_stream, fstream.cuda_stream)
                else:
                    fn = lambda: lib.bz_push_tiles_ce(src.ptr, mapped.ptr, mapped.flags_ptr, None,  # noqa: E731
                                                      lay.tile_off.ctypes.data, 0, lay.ntiles, tpc, e,
                                                      stream.cuda_stream)
                ms = timed(fn, stream)
                emit({"case": "push", "engine": "ce2" if split else "ce", "tiles_per_copy": tpc, "ms": ms,
                      "GBps": payload / ms / 1e6, "ok": check(peer, want, e)})

    # ---- NVLS multicast over gpu0..gpu{G-1} ------------------------------------------------------
    try:
        mc = LocalMc([src] + dsts, 0)
    except Exception as ex:  # noqa: BLE001
        emit({"case": "mc", "supported": False, "error": str(ex)[:300]})
        return

    def mcast(nctas):
        e = nxt()
        fn = lambda: lib.bz_multicast_tiles(src.ptr, mc.ptr, mc.flags_ptr, None, src.tile_off.data_ptr(),  # noqa: E731
                                            0, lay.ntiles, e, nctas, stream.cuda_stream)
        return fn, e

    if args.once == "mc":
        fn, e = mcast(args.nctas)
        fn()
        torch.cuda.synchronize()
        emit({"case": "mc-once", "ok": all(check(d, want, e) for d in dsts)})
        return
    for u in [int(x) for x in args.unrolls.split(",")]:
        os.environ["BZ_MC_UNROLL"] = str(u)
        for c in [int(x) for x in args.ctas.split(",")]:
            fn, e = mcast(c)
            ms = timed(fn, stream)
            emit({"case": "mc", "members": G, "unroll": u, "nctas": c, "ms": ms,
                  "GBps_per_dest": payload / ms / 1e6, "ok": all(check(d, want, e) for d in dsts)})
    os.environ.pop("BZ_MC_UNROLL", None)
    mc.close()


if __name__ == "__main__":
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BZ_WATCHDOG_S", "300")), exit=True)
    t0 = time.time()
    main()
    emit({"case": "done", "wall_s": time.time() - t0})
