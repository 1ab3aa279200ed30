"""The cache-miss (local storage) load path into HBM (
autoscaler.py:113-117): a slab image streamed with O_DIRECT through pinned
buffers, bit-exact on the GPU, every layer published in order with a stamp."""

import os
import tempfile

import pytest
import torch

from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.dataplane import DeviceSlab
from paper_2412_17246_b200.diskload import DiskSlabLoader, write_slab_image

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("arch", [S.TINY_4L, S.LlamaArch("llama2-7b-l2", 4096, 2, 32, 32, 11008)],
                         ids=["tiny", "7b-width-2l"])
def test_disk_image_loads_bit_exact_layer_by_layer(arch):
    lay = S.SlabLayout.for_arch(arch)
    src, dst = DeviceSlab(lay, 0), DeviceSlab(lay, 0)
    src.fill_random(seed=77)
    want = src.fingerprints().cpu()
    d = tempfile.mkdtemp(dir="/tmp", prefix="bz_disk_")
    path = os.path.join(d, "shard.img")
    try:
        try:
            write_slab_image(src.data, path)
        except OSError as e:
            pytest.skip(f"no O_DIRECT-capable scratch space in /tmp ({e})")
        loader = DiskSlabLoader(lay, path, device=0, chunk=16 << 20)
        for epoch in (1, 2):
            dst.data.fill_(0x5A)
            res = loader.load(dst, epoch)
            assert torch.equal(dst.fingerprints().cpu(), want)
            assert int(dst.loaded.item()) == lay.num_layers
            assert int(dst.flags.min()) == epoch and int(dst.flags.max()) == epoch
            assert res["layer_ms"] == sorted(res["layer_ms"]) and res["layer_ms"][0] > 0
            assert res["ssd_to_gpu_GBps"] > 0
    finally:
        if os.path.exists(path):
            os.unlink(path)
        os.rmdir(d)
        src.close()
        dst.close()
