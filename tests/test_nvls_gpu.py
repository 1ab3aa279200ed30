"""NVLS multicast realisation of ``ScalePlan.nvlink_fanout`` (planner.py:86-87, 245-253).

``k_multicast_tiles`` writes every tile once through a multicast VA bound to the
slabs of a fan-out group; the NVSwitch replicates it.  One process binds slabs on
several of its GPUs (``LocalMulticastGroup``) so the kernel is checked without
torchrun; the multi-process form runs in test_multigpu.py (mgpu_check.py cases
``grouped-nvls`` and ``hostcache-rep-nvls``).
"""

import ctypes

import pytest
import torch

from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200._native import BlitzError, BzMc, cuda_lib
from paper_2412_17246_b200.dataplane import DeviceSlab, HostCache, LocalMulticastGroup

pytestmark = pytest.mark.gpu

LAYOUT = S.SlabLayout.for_arch(S.TINY_4L, tile_bytes=256 * 1024)


def test_one_device_multicast_object():
    """A fan-out group of one GPU has no NVLS form: B200 rejects numDevices=1."""
    lib = cuda_lib(0)
    gmin, grec = ctypes.c_uint64(), ctypes.c_uint64()
    lib.bz_mc_granularity(0, 1, ctypes.byref(gmin), ctypes.byref(grec))
    raw = BzMc()
    try:
        lib.bz_mc_create(1, gmin.value, raw)
    except BlitzError as e:
        assert "CUDA_ERROR_INVALID_VALUE" in str(e) or "NOT_SUPPORTED" in str(e), e
        pytest.skip("cuMulticastCreate rejects numDevices=1 on this B200 (measured: "
                    "CUDA_ERROR_INVALID_VALUE, scripts/nvlink_probe.py); NVLS needs >= 2 GPUs and is "
                    "exercised by test_single_process_multicast_bit_exact and test_multigpu.py")
    lib.bz_mc_free(raw, 0, 0)


@pytest.mark.multigpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NVLS needs >= 2 GPUs")
@pytest.mark.parametrize("relay", [False, True])
def test_single_process_multicast_bit_exact(relay):
    G = min(torch.cuda.device_count(), 4)
    lib = cuda_lib(0)
    for d in range(G):
        cuda_lib(d)
    src = DeviceSlab(LAYOUT, 0)
    dsts = [DeviceSlab(LAYOUT, d) for d in range(1, G)]
    mc = LocalMulticastGroup([src] + dsts, map_device=0)
    hc = None
    try:
        s = torch.cuda.current_stream(0).cuda_stream
        if relay:
            # the writer is itself fed (host cache -> gpu0); it forwards each tile into
            # the group once its own flag says the tile landed (hostcache-rep-nvls)
            tmp = DeviceSlab(LAYOUT, 0)
            tmp.fill_random(seed=31)
            hc = HostCache(LAYOUT)
            hc.tensor.copy_(tmp.data.cpu())
            want = tmp.fingerprints().cpu()
            tmp.close()
        else:
            src.fill_random(seed=31)
            want = src.fingerprints().cpu()
        for epoch in (1, 2):
            for d in dsts:
                with torch.cuda.device(d.device):
                    d.data.fill_(0xA5)
                torch.cuda.synchronize(d.device)
            if relay:
                lib.bz_stage_tiles_ce(hc.ptr, src.ptr, src.flags_ptr, hc.tile_off_host.ctypes.data, 0,
                                      LAYOUT.ntiles, 16, epoch, s)
            lib.bz_multicast_tiles(src.ptr, mc.ptr, mc.flags_ptr, src.flags_ptr if relay else None,
                                   src.tile_off.data_ptr(), 0, LAYOUT.ntiles, epoch, 16, s)
            for d in range(G):
                torch.cuda.synchronize(d)
            for d in dsts:
                assert torch.equal(d.fingerprints().cpu(), want), f"gpu{d.device} differs"
                fl = d.flags.cpu()
                assert int(fl.min()) == epoch and int(fl.max()) == epoch
    finally:
        mc.close()
        if hc is not None:
            hc.close()
        for d in dsts:
            d.close()
        src.close()
