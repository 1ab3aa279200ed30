"""GPU parity of the data plane (calls through the C ABI of libblitz.so).

Bit-exactness: every destination slab must equal the source slab byte for byte
after a plan executes (torch.equal on uint8 views, random-bit payloads that
include bf16 NaN/Inf patterns), the tile flags must all carry the epoch, and
the tracker must report every layer loaded.  The payload and fingerprints are
checked against the CPU oracle (oracle/dataplane_ref.py).
"""

import numpy as np
import pytest
import torch

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200._native import cuda_lib
from paper_2412_17246_b200.dataplane import (ENGINE_TMA, ENGINE_VECTOR, DeviceSlab, HostCache,
                                             execute_plan_loopback)
from oracle import dataplane_ref as ref

pytestmark = pytest.mark.gpu


def _plan(sources, targets, group=True, topo="b200-hgx", model=None):
    t = ss.load_topology(topo)
    flows = ss.FlowSet(t)
    model = model or S.model_spec_for(S.LLAMA2_7B)
    req = ss.build_scale_request(model, sources, targets, t, flows)
    return ss.generate_plan(req, t, flows, group=group)


@pytest.fixture(scope="module")
def tiny_layout():
    return S.SlabLayout.for_arch(S.TINY_4L, tile_bytes=256 * 1024)


def test_fill_random_matches_oracle(tiny_layout):
    slab = DeviceSlab(tiny_layout, 0)
    slab.fill_random(seed=1234)
    torch.cuda.synchronize()
    want = ref.random_words(tiny_layout.data_bytes, 1234)
    assert np.array_equal(slab.data.cpu().numpy(), want)
    fp = slab.fingerprints().cpu().numpy().view(np.uint64)
    assert np.array_equal(fp, ref.tile_fingerprints(want, tiny_layout.tile_off))
    slab.close()


def _check_copies(slabs, src, layout, epoch):
    for n, s in slabs.items():
        if n == src:
            continue
        assert torch.equal(s.data, slabs[src].data), f"{n} differs from {src}"
        assert int(s.flags.min()) == epoch and int(s.flags.max()) == epoch
        assert int(s.loaded.item()) == layout.num_layers


@pytest.mark.parametrize("engine", [ENGINE_VECTOR, ENGINE_TMA, 2])
@pytest.mark.parametrize("targets,group", [
    (["gpu1"], True),                                  # C1 1->2
    (["gpu1", "gpu2", "gpu3"], False),                 # 1->4 chain
    ([f"gpu{i}" for i in range(1, 8)], True),          # 1->8 rep + fan-out
    ([f"gpu{i}" for i in range(1, 8)], False),         # 1->8 seven-hop chain
])
def test_loopback_plan_bit_exact(tiny_layout, engine, targets, group):
    plan = _plan(["gpu0"], targets, group=group, model=S.model_spec_for(S.TINY_4L))
    nodes = ["gpu0"] + targets
    slabs = {n: DeviceSlab(tiny_layout, 0) for n in nodes}
    slabs["gpu0"].fill_random(seed=99)
    for epoch in (1, 2):
        if epoch == 2:  # a second transfer must overwrite stale bytes
            for n in targets:
                slabs[n].data.fill_(0xA5)
        execute_plan_loopback(plan, slabs, epoch, engine=engine, nctas=8)
        torch.cuda.synchronize()
        _check_copies(slabs, "gpu0", tiny_layout, epoch)
    for s in slabs.values():
        s.close()


@pytest.mark.parametrize("stage_engine", ["ce", "sm"])
def test_loopback_host_staging_then_fanout(tiny_layout, stage_engine):
    """C5 shape: O(1) host cache -> gpu0 (pcie) -> fan-out gpu4 (nvlink)."""
    plan = _plan(["mem0"], ["gpu0", "gpu4"], model=S.model_spec_for(S.TINY_4L))
    assert [(e.src, e.dst, e.kind) for e in plan.edges] == [("mem0", "gpu0", "pcie")]
    hc = HostCache(tiny_layout)
    hc.tensor.copy_(torch.from_numpy(ref.random_words(tiny_layout.data_bytes, 5)))
    slabs = {n: DeviceSlab(tiny_layout, 0) for n in ("gpu0", "gpu4")}
    execute_plan_loopback(plan, slabs, 1, host_cache=hc, stage_engine=stage_engine, nctas=4)
    torch.cuda.synchronize()
    for n in ("gpu0", "gpu4"):
        assert torch.equal(slabs[n].data.cpu(), hc.tensor), n
        assert int(slabs[n].loaded.item()) == tiny_layout.num_layers
    hc.close()
    for s in slabs.values():
        s.close()


def test_7b_layer_slab_single_hop_bit_exact():
    """Full Llama-2 7B shard (13.48 GB) across one hop on one GPU, fingerprint-checked."""
    lay = S.SlabLayout.for_arch(S.LLAMA2_7B, tile_bytes=1 << 20)
    assert lay.payload_bytes() == 13_476_831_232
    a, b = DeviceSlab(lay, 0), DeviceSlab(lay, 0)
    a.fill_random(seed=7)
    plan = _plan(["gpu0"], ["gpu1"])
    execute_plan_loopback(plan, {"gpu0": a, "gpu1": b}, 1, nctas=64)
    torch.cuda.synchronize()
    assert torch.equal(a.fingerprints(), b.fingerprints())
    # spot-check raw bytes of the first, a middle and the last unit
    for k in (0, lay.num_layers // 2, lay.num_layers - 1):
        o, n = lay.unit_off[k], lay.unit_bytes[k]
        assert torch.equal(a.data[o:o + n], b.data[o:o + n])
    assert int(b.loaded.item()) == 32
    a.close()
    b.close()


def test_wait_layer_gates_a_stream(tiny_layout):
    lib = cuda_lib()
    a, b = DeviceSlab(tiny_layout, 0), DeviceSlab(tiny_layout, 0)
    a.fill_random(seed=3)
    plan = _plan(["gpu0"], ["gpu1"], model=S.model_spec_for(S.TINY_4L))
    copy_stream = torch.cuda.Stream()
    gate_stream = torch.cuda.Stream()
    execute_plan_loopback(plan, {"gpu0": a, "gpu1": b}, 1, stream=copy_stream)
    lib.bz_wait_layer(b.loaded.data_ptr(), tiny_layout.num_layers, gate_stream.cuda_stream)
    with torch.cuda.stream(gate_stream):
        out = b.data[:4096].clone()
    gate_stream.synchronize()
    assert torch.equal(out, a.data[:4096])
    a.close()
    b.close()


def test_handoff_copies_and_counts():
    lib = cuda_lib()
    src = torch.randint(-2**15, 2**15, (2000, 256), dtype=torch.int16, device="cuda")
    dst = torch.zeros_like(src)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.bz_handoff(src.data_ptr(), dst.data_ptr(), src.numel() * 2, flag.data_ptr(), 0, 8,
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(src, dst) and int(flag.item()) == 8


# ---- edge cases: ragged units, single tile, maximum fan-out, empty ranges ------------------


def test_ragged_units_and_tiles_bit_exact():
    """Unit sizes that are not tile multiples (last tile of every unit ragged),
    including a unit smaller than one tile."""
    lay = S.SlabLayout([3 * 4096 + 256, 256, 7 * 4096 - 256, 4096], tile_bytes=4096)
    assert any(int(b - a) < 4096 for a, b in zip(lay.tile_off[:-1], lay.tile_off[1:]))
    slabs = {n: DeviceSlab(lay, 0) for n in ("gpu0", "gpu1", "gpu2")}
    slabs["gpu0"].fill_random(seed=11)
    plan = _plan(["gpu0"], ["gpu1", "gpu2"], group=False, model=S.model_spec_for(S.TINY_4L))
    for engine in (ENGINE_VECTOR, ENGINE_TMA, 2):
        execute_plan_loopback(plan, slabs, engine + 1, engine=engine, nctas=3)
        torch.cuda.synchronize()
        _check_copies(slabs, "gpu0", lay, engine + 1)
    for s in slabs.values():
        s.close()


def test_single_tile_slab():
    lay = S.SlabLayout([512], tile_bytes=1 << 20)
    assert lay.ntiles == 1
    a, b = DeviceSlab(lay, 0), DeviceSlab(lay, 0)
    a.fill_random(seed=2)
    execute_plan_loopback(_plan(["gpu0"], ["gpu1"], model=S.model_spec_for(S.TINY_4L)),
                          {"gpu0": a, "gpu1": b}, 1, nctas=64)
    torch.cuda.synchronize()
    assert torch.equal(a.data, b.data) and int(b.loaded.item()) == 1
    a.close()
    b.close()


def test_max_fanout_star_push_and_empty_range(tiny_layout):
    """One read, BZ_MAX_DST = 8 peer writes per tile; an empty tile range is a no-op."""
    from paper_2412_17246_b200._native import ptr_array
    lib = cuda_lib()
    src = DeviceSlab(tiny_layout, 0)
    src.fill_random(seed=8)
    dsts = [DeviceSlab(tiny_layout, 0) for _ in range(8)]
    s = torch.cuda.current_stream().cuda_stream
    ptrs = ptr_array([d.ptr for d in dsts])
    flags = ptr_array([d.flags_ptr for d in dsts])
    lib.bz_push_tiles(src.ptr, ptrs, flags, 8, None, src.tile_off.data_ptr(), 0, 0, 1, 8, 0, s)
    lib.bz_push_tiles(src.ptr, ptrs, flags, 8, None, src.tile_off.data_ptr(), 0,
                      tiny_layout.ntiles, 1, 8, 0, s)
    torch.cuda.synchronize()
    for d in dsts:
        assert torch.equal(d.data, src.data) and int(d.flags.min()) == 1
        d.close()
    src.close()


def test_preload_kernels_loads_every_module():
    import ctypes
    n = ctypes.c_int()
    cuda_lib().bz_preload_kernels(0, ctypes.byref(n))
    assert n.value >= 20   # push/multicast/stage/track/... + GEMM + decode + glue kernels


def test_push_tile_list_moves_exactly_the_listed_tiles(tiny_layout):
    """Tile-list push (striped host load): listed tiles land bit-exact with their flag,
    unlisted tiles stay untouched; gating on the sender's own flags."""
    from paper_2412_17246_b200._native import ptr_array
    lib = cuda_lib()
    src = DeviceSlab(tiny_layout, 0)
    src.fill_random(seed=12)
    dst = DeviceSlab(tiny_layout, 0)
    dst.data.zero_()
    n = tiny_layout.ntiles
    ids = torch.tensor(list(range(n - 1, -1, -2)), dtype=torch.int32, device="cuda")  # odd-from-top, reversed
    s = torch.cuda.current_stream().cuda_stream
    src.flags.fill_(3)   # the sender's own pieces are staged (epoch 3)
    lib.bz_push_tile_list(src.ptr, ptr_array([dst.ptr]), ptr_array([dst.flags_ptr]), 1, src.flags_ptr,
                          src.tile_off.data_ptr(), ids.data_ptr(), int(ids.numel()), 3, 4, s)
    lib.bz_push_tile_list(src.ptr, ptr_array([dst.ptr]), ptr_array([dst.flags_ptr]), 1, None,
                          src.tile_off.data_ptr(), ids.data_ptr(), 0, 3, 4, s)   # empty list: no-op
    torch.cuda.synchronize()
    listed = set(ids.tolist())
    off = tiny_layout.tile_off
    flags = dst.flags.cpu().tolist()
    for t in range(n):
        a, b = int(off[t]), int(off[t + 1])
        if t in listed:
            assert flags[t] == 3 and torch.equal(dst.data[a:b], src.data[a:b]), t
        else:
            assert flags[t] == 0 and int(dst.data[a:b].count_nonzero()) == 0, t
    from paper_2412_17246_b200._native import BlitzError
    with pytest.raises(BlitzError):   # a non-empty list needs the ids
        lib.bz_push_tile_list(src.ptr, ptr_array([dst.ptr]), ptr_array([dst.flags_ptr]), 1, None,
                              src.tile_off.data_ptr(), None, 4, 3, 4, s)
    src.close()
    dst.close()


def test_bad_arguments_raise():
    from paper_2412_17246_b200._native import BlitzError, ptr_array
    lib = cuda_lib()
    with pytest.raises(BlitzError):
        lib.bz_push_tiles(None, ptr_array([0]), ptr_array([0]), 1, None, None, 0, 1, 1, 8, 0, 0)
    with pytest.raises(BlitzError):  # ndst above BZ_MAX_DST
        lib.bz_push_tiles(1, ptr_array([0] * 9), ptr_array([0] * 9), 9, None, 1, 0, 1, 1, 8, 0, 0)
    with pytest.raises(BlitzError):
        lib.bz_fill_random(1, 17, 0, 0)   # size not a multiple of 16


def test_gate_timeout_fails_loudly():
    """A gate whose flag is never raised gives up after the spin budget (no hung GPU)
    and the next check raises instead of letting results through silently."""
    import ctypes
    from paper_2412_17246_b200.dataplane import gate
    from paper_2412_17246_b200.scaleup import TransferTimeout, check_wait_timeouts
    lib = cuda_lib()
    check_wait_timeouts()                       # absorb anything earlier tests left
    n = ctypes.c_uint64()
    lib.bz_wait_timeouts(ctypes.byref(n), 2_000_000)      # 2 ms budget
    try:
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        gate(flag.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        with pytest.raises(TransferTimeout):
            check_wait_timeouts()
        check_wait_timeouts()                   # counted once
    finally:
        lib.bz_wait_timeouts(ctypes.byref(n), 30_000_000_000)


def test_relay_timeout_withholds_downstream_flags(tiny_layout):
    """A relay whose upstream never publishes must not forward stale bytes: its
    bounded wait gives up, it skips the copy and withholds the downstream flag, so
    the downstream tracker publishes nothing and times out as well."""
    import ctypes
    from paper_2412_17246_b200.scaleup import new_wait_timeouts

    lib = cuda_lib()
    relay, down = DeviceSlab(tiny_layout, 0), DeviceSlab(tiny_layout, 0)
    relay.fill_random(seed=5)
    down.data.fill_(0x5A)
    n = ctypes.c_uint64()
    new_wait_timeouts()                                    # reset the per-device baseline
    lib.bz_wait_timeouts(ctypes.byref(n), 200_000)         # 0.2 ms budget per wait
    try:
        s = torch.cuda.current_stream().cuda_stream
        from paper_2412_17246_b200._native import ptr_array
        # relay flags stay 0 (upstream dead); push epoch 3 downstream
        for engine in (ENGINE_VECTOR, ENGINE_TMA, 2):
            lib.bz_push_tiles(relay.ptr, ptr_array([down.ptr]), ptr_array([down.flags_ptr]), 1,
                              relay.flags_ptr, relay.tile_off.data_ptr(), 0, tiny_layout.ntiles, 3, 8,
                              engine, s)
        # copy-engine relay: gate times out -> flag kernel withholds the release
        lib.bz_push_tiles_ce(relay.ptr, down.ptr, down.flags_ptr, relay.flags_ptr,
                             tiny_layout.tile_off.ctypes.data, 0, tiny_layout.ntiles, 4, 3, s)
        lib.bz_track_layers(down.flags_ptr, down.layer_tile.data_ptr(), tiny_layout.num_layers, 3,
                            down.loaded.data_ptr(), down.stamps.data_ptr(), s)
        torch.cuda.synchronize()
        assert int(down.flags.max()) == 0, "a downstream flag was released for stale bytes"
        assert int(down.loaded.item()) == 0
        assert new_wait_timeouts() > 0
    finally:
        lib.bz_wait_timeouts(ctypes.byref(n), 30_000_000_000)
    relay.close()
    down.close()


def test_copy_engine_hop_with_flag_stream(tiny_layout):
    """bz_push_tiles_ce2 (the copy-engine hop: a relay chain's first hop, the live pair): copies back to back
    on one stream, flag releases on another; bytes and every flag exact, and the copy
    stream joins the flag stream at the end."""
    lib = cuda_lib()
    src, dst = DeviceSlab(tiny_layout, 0), DeviceSlab(tiny_layout, 0)
    src.fill_random(seed=21)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    for epoch, tpc in ((1, 4), (2, 128)):
        lib.bz_push_tiles_ce2(src.ptr, dst.ptr, dst.flags_ptr, None, tiny_layout.tile_off.ctypes.data, 0,
                              tiny_layout.ntiles, tpc, epoch, s1.cuda_stream, s2.cuda_stream)
        s1.synchronize()          # joins s2: every flag released once s1 is done
        assert torch.equal(dst.data, src.data)
        assert int(dst.flags.min()) == epoch and int(dst.flags.max()) == epoch
    src.close()
    dst.close()


def test_pull_kernel_waits_notifies_and_copies_exactly(tiny_layout):
    """bz_pull_tiles (the `auto` engine's source -> leaf hop, launched on the receiver):
    bytes and flags exact; with wait flags it copies only tiles whose flag carries the
    epoch, and notify receives the same releases (loopback on one GPU)."""
    lib = cuda_lib()
    src, dst = DeviceSlab(tiny_layout, 0), DeviceSlab(tiny_layout, 0)
    src.fill_random(seed=33)
    s = torch.cuda.current_stream().cuda_stream
    lib.bz_pull_tiles(src.ptr, dst.ptr, dst.flags_ptr, None, None, dst.tile_off.data_ptr(), 0,
                      tiny_layout.ntiles, 1, 64, s)
    torch.cuda.synchronize()
    assert torch.equal(dst.data, src.data)
    assert int(dst.flags.min()) == 1 and int(dst.flags.max()) == 1
    # relay form: src flags already at epoch 2, a separate notify array receives epoch 2
    src.flags.fill_(2)
    src.fill_random(seed=34)
    notify = torch.zeros(tiny_layout.ntiles, dtype=torch.int32, device="cuda")
    lib.bz_pull_tiles(src.ptr, dst.ptr, dst.flags_ptr, src.flags_ptr, notify.data_ptr(), dst.tile_off.data_ptr(),
                      0, tiny_layout.ntiles, 2, 64, s)
    torch.cuda.synchronize()
    assert torch.equal(dst.data, src.data)
    assert int(dst.flags.min()) == 2 and int(notify.min()) == 2
    src.close()
    dst.close()


def test_gated_copy_engine_relay_chain(tiny_layout):
    """bz_push_tiles_ce2 into a relay, bz_push_tiles_ce_gated out of it (the auto engine's
    relay chain): the relay's copies wait on its own tile flags through gates enqueued on
    a third stream; the leaf ends bit-exact with every flag at the epoch (loopback)."""
    lib = cuda_lib()
    src, relay, leaf = (DeviceSlab(tiny_layout, 0) for _ in range(3))
    src.fill_random(seed=41)
    off = tiny_layout.tile_off.ctypes.data
    s_src, f_src = torch.cuda.Stream(), torch.cuda.Stream()
    s_rel, f_rel, g_rel = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for epoch in (1, 2):
        # the relay's leg first (its gates wait), then the source's leg that feeds it
        lib.bz_push_tiles_ce_gated(relay.ptr, leaf.ptr, leaf.flags_ptr, relay.flags_ptr, off, 0, tiny_layout.ntiles,
                                   4, epoch, s_rel.cuda_stream, f_rel.cuda_stream, g_rel.cuda_stream)
        lib.bz_push_tiles_ce2(src.ptr, relay.ptr, relay.flags_ptr, None, off, 0, tiny_layout.ntiles, 4, epoch,
                              s_src.cuda_stream, f_src.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(leaf.data, src.data) and torch.equal(relay.data, src.data)
        assert int(leaf.flags.min()) == epoch and int(leaf.flags.max()) == epoch
    for x in (src, relay, leaf):
        x.close()
