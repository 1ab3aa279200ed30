"""Layer-slab layout of a model shard in HBM (and in the pinned host cache).

The reference describes a model as ``num_layers x bytes_per_layer``
(``parampool.py:25-62``) and streams it layer by layer (``simcore.py:727-733``).
On B200 the shard held by one GPU is ONE contiguous slab laid out in *load
units*: unit 1 = token embedding + block 1, unit k = block k, unit L = block L +
final norm + lm_head (SURVEY.md §7.2 "plan granularity").  Each unit is padded
to 256 B and cut into tiles that never straddle units; tile ``t`` covers
``[tile_off[t], tile_off[t+1])``.  A u32 flag per tile follows the data, so a
single VMM allocation (and a single multicast binding) carries both.

Per-unit bytes of a TP shard are the unit bytes divided by ``tp`` (each rank
holds 1/tp of every matrix), rounded up to the alignment.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ALIGN = 256
FLAG_BYTES = 4
BF16 = 2


@dataclass(frozen=True)
class LlamaArch:
    """Llama-2 family dimensions; parameter bytes per block / embedding in bf16."""

    name: str
    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int = 32000
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    def block_params(self) -> int:
        d = self.d_model
        attn = d * d + 2 * d * self.kv_dim + d * d
        mlp = 3 * d * self.ffn
        return attn + mlp + 2 * d

    def block_bytes(self) -> int:
        return self.block_params() * BF16

    def embed_bytes(self) -> int:
        return self.vocab * self.d_model * BF16

    def total_bytes(self) -> int:
        return self.n_layers * self.block_bytes() + 2 * self.embed_bytes() + self.d_model * BF16

    def unit_bytes(self) -> list[int]:
        """Bytes of each load unit (unit 1 carries the embedding, unit L the head)."""
        units = [self.block_bytes()] * self.n_layers
        units[0] += self.embed_bytes()
        units[-1] += self.d_model * BF16 + self.embed_bytes()
        return units


# SURVEY.md §8d synthetic configs
TINY_4L = LlamaArch("tiny-4l", d_model=256, n_layers=4, n_heads=4, n_kv_heads=4, ffn=688)
LLAMA2_7B = LlamaArch("llama2-7b", 4096, 32, 32, 32, 11008)
LLAMA2_13B = LlamaArch("llama2-13b", 5120, 40, 40, 40, 13824)
LLAMA2_70B = LlamaArch("llama2-70b", 8192, 80, 64, 8, 28672)
ARCHS = {a.name: a for a in (TINY_4L, LLAMA2_7B, LLAMA2_13B, LLAMA2_70B)}


def _align(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


@dataclass
class SlabLayout:
    """Unit/tile geometry of one GPU's shard slab."""

    unit_bytes: list[int]
    tile_bytes: int
    unit_off: list[int] = field(init=False)
    tile_off: np.ndarray = field(init=False)      # int64[ntiles + 1]
    layer_tile: np.ndarray = field(init=False)    # int32[L + 1]
    data_bytes: int = field(init=False)
    flag_offset: int = field(init=False)
    total_bytes: int = field(init=False)

    def __post_init__(self):
        if self.tile_bytes < ALIGN or self.tile_bytes % ALIGN:
            raise ValueError(f"tile_bytes must be a positive multiple of {ALIGN}")
        if not self.unit_bytes or any(u <= 0 for u in self.unit_bytes):
            raise ValueError("unit sizes must be positive")
        offs, tiles, layer_tile = [], [], [0]
        cur = 0
        for u in self.unit_bytes:
            padded = _align(u)
            offs.append(cur)
            n = (padded + self.tile_bytes - 1) // self.tile_bytes
            for i in range(n):
                tiles.append(cur + i * self.tile_bytes)
            cur += padded
            layer_tile.append(len(tiles))
        tiles.append(cur)
        self.unit_off = offs
        self.tile_off = np.asarray(tiles, dtype=np.int64)
        self.layer_tile = np.asarray(layer_tile, dtype=np.int32)
        self.data_bytes = cur
        self.flag_offset = _align(cur, 4096)
        self.total_bytes = self.flag_offset + _align(self.ntiles * FLAG_BYTES, 4096)

    @property
    def num_layers(self) -> int:
        return len(self.unit_bytes)

    @property
    def ntiles(self) -> int:
        return int(self.tile_off.shape[0] - 1)

    def tiles_of_layer(self, k: int) -> tuple[int, int]:
        """Tile range of 0-based unit ``k``."""
        return int(self.layer_tile[k]), int(self.layer_tile[k + 1])

    def payload_bytes(self) -> int:
        """Model bytes carried (without padding)."""
        return int(sum(self.unit_bytes))

    @classmethod
    def for_arch(cls, arch: LlamaArch, tp: int = 1, tile_bytes: int = 1 << 20) -> "SlabLayout":
        return cls([_align((u + tp - 1) // tp) for u in arch.unit_bytes()], tile_bytes)

    @classmethod
    def uniform(cls, num_layers: int, bytes_per_layer: int, tile_bytes: int = 1 << 20) -> "SlabLayout":
        return cls([_align(int(bytes_per_layer))] * num_layers, tile_bytes)


def model_spec_for(arch: LlamaArch, tp: int = 1, **cost):
    """A reference ``ModelSpec`` whose uniform layer size carries the real byte total,
    so modeled estimates and measured transfers describe the same bytes."""
    from .parampool import ModelSpec

    return ModelSpec(name=f"{arch.name}" + (f"-tp{tp}" if tp > 1 else ""),
                     num_layers=arch.n_layers,
                     bytes_per_layer=arch.total_bytes() / arch.n_layers,
                     tp_degree=tp, **cost)
