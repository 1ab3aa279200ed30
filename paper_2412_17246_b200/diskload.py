"""The cache-miss load path: a shard image on local storage streamed into a GPU slab
with per-layer readiness (ServerlessLLM's checkpoint load, autoscaler.py:113-117;
the pool's no-copy case, parampool.py:168-181).

On-disk format: the slab's data region verbatim (load units in order, 256-B aligned,
``slab.SlabLayout``), so a load is one sequential read.  ``checkpoint.py`` converts a
Hugging Face safetensors checkpoint into / out of this layout.

Mechanism: O_DIRECT reads (no page-cache copy) into two pinned staging buffers, each
chunk copied host -> HBM on a side stream while the next chunk is read; as soon as
the bytes of layer unit k have landed, its tile flags are raised and ``loaded`` is
published (in stream order, ``bz_publish_layer``), exactly as for the host-cache
path -- so a scaled instance can start executing the layers that arrived.
"""

from __future__ import annotations

import os
from typing import Optional

import numpy as np
import torch

from ._native import cuda_lib
from .dataplane import DeviceSlab
from .slab import SlabLayout

_ALIGN = 4096  # O_DIRECT: offsets, sizes and buffer addresses multiple of the block size


def write_slab_image(data: torch.Tensor, path: str, chunk: int = 64 << 20) -> int:
    """Write a slab's data region (uint8, host or device) as an image file, padded to
    the O_DIRECT block size.  Returns the bytes written."""
    n = int(data.numel())
    total = (n + _ALIGN - 1) // _ALIGN * _ALIGN
    buf = torch.zeros(chunk, dtype=torch.uint8, pin_memory=True)
    fd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC | getattr(os, "O_DIRECT", 0), 0o644)
    try:
        off = 0
        while off < total:
            m = min(chunk, total - off)
            got = max(0, min(m, n - off))
            buf[:m].zero_()
            if got:
                buf[:got].copy_(data[off:off + got].cpu() if data.is_cuda else data[off:off + got])
            os.write(fd, memoryview(buf.numpy())[:m])
            off += m
        os.fsync(fd)
    finally:
        os.close(fd)
    return total


class DiskSlabLoader:
    """Streams a slab image into a ``DeviceSlab`` with per-layer publish."""

    def __init__(self, layout: SlabLayout, path: str, device: int, chunk: int = 64 << 20):
        if chunk % _ALIGN:
            raise ValueError("chunk must be a multiple of 4096")
        self.layout, self.path, self.device, self.chunk = layout, path, device, chunk
        self.bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.stream = torch.cuda.Stream(device=device)
        self.lib = cuda_lib(device)
        # layer unit k is complete once the read offset passes its end
        self._unit_end = [int(layout.tile_off[layout.layer_tile[k + 1]]) for k in range(layout.num_layers)]

    def load(self, slab: DeviceSlab, epoch: int) -> dict:
        """Read the image into ``slab`` (blocking until the last byte is enqueued and
        copied); returns the per-layer arrival (ms after the first read) and rates."""
        lay = self.layout
        total = lay.data_bytes
        s = self.stream
        with torch.cuda.device(self.device), torch.cuda.stream(s):
            self.lib.bz_publish_layer(slab.loaded.data_ptr(), 0, slab.stamps.data_ptr() + 8 * lay.num_layers,
                                      s.cuda_stream)
        fd = os.open(self.path, os.O_RDONLY | getattr(os, "O_DIRECT", 0))
        done: list[Optional[torch.cuda.Event]] = [None, None]
        off, i, layer = 0, 0, 0
        import time
        t0 = time.perf_counter()
        disk_s = 0.0
        try:
            while off < total:
                b = i % 2
                if done[b] is not None:
                    done[b].synchronize()        # the previous copy out of this buffer finished
                r0 = time.perf_counter()
                n = os.readv(fd, [memoryview(self.bufs[b].numpy())])
                disk_s += time.perf_counter() - r0
                if n <= 0:
                    raise IOError(f"{self.path}: image ends at {off} of {total} bytes")
                n = min(n, total - off)
                with torch.cuda.device(self.device), torch.cuda.stream(s):
                    slab.data[off:off + n].copy_(self.bufs[b][:n], non_blocking=True)
                    off += n
                    # every unit now complete: raise its tile flags, publish it (in order)
                    while layer < lay.num_layers and self._unit_end[layer] <= off:
                        t_lo, t_hi = lay.tiles_of_layer(layer)
                        slab.flags[t_lo:t_hi].fill_(epoch)
                        self.lib.bz_publish_layer(slab.loaded.data_ptr(), layer + 1,
                                                  slab.stamps.data_ptr() + 8 * layer, s.cuda_stream)
                        layer += 1
                    ev = torch.cuda.Event()
                    ev.record(s)
                done[b] = ev
                i += 1
        finally:
            os.close(fd)
        s.synchronize()
        wall = time.perf_counter() - t0
        st = slab.stamps.cpu().tolist()
        return {"layer_ms": [(x - st[lay.num_layers]) / 1e6 for x in st[:lay.num_layers]],
                "bytes": total, "disk_read_GBps": total / disk_s / 1e9, "ssd_to_gpu_GBps": total / wall / 1e9}
