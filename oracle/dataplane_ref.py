"""CPU restatement of the byte data plane -- TEST INFRASTRUCTURE / CPU BASELINE ONLY.

The reference moves no bytes: a plan edge is ``nbytes / (gbps * eta * 0.125e9)``
seconds (planner.py:227-262, topology.py:57-61) and fan-out is "one intra-host
broadcast" (planner.py:245-253).  Its byte-level meaning is unambiguous: after
a scale-up every target holds a bit-identical copy of the source shard.  This
module states that on the CPU:

* ``random_words`` -- the payload generator of ``bz_fill_random`` (word i =
  splitmix64(seed + i)), so a GPU slab can be checked against bytes made here.
* ``tile_fingerprints`` -- the per-tile fingerprint of ``bz_tile_fingerprints``.
* ``execute_plan_cpu`` -- torch CPU ``copy_`` of each unit along the plan's
  edges (store-and-forward order) and fan-out groups as repeated copies: the
  CPU baseline of BASELINE.md §4 item 2, timed by bench.py's reference arm.

``parity pinned``: the byte semantics (destination == source) are self-pinned
by construction; the plan structure they follow is pinned to the reference's
own outputs (tests/golden/plans.json).
"""

from __future__ import annotations

import time
from typing import Optional

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser (same constants as csrc/dataplane.cu)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def random_words(nbytes: int, seed: int) -> np.ndarray:
    """uint8 payload identical to bz_fill_random(dst, nbytes, seed)."""
    n = nbytes // 8
    with np.errstate(over="ignore"):
        idx = np.arange(n, dtype=np.uint64) + np.uint64(seed)
    return splitmix64(idx).view(np.uint8)


def tile_fingerprints(buf: np.ndarray, tile_off: np.ndarray) -> np.ndarray:
    """sum_i splitmix64(word_i ^ splitmix64(i - tile_start)) per tile, mod 2^64."""
    words = buf.view(np.uint64)
    out = np.zeros(len(tile_off) - 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for t in range(len(tile_off) - 1):
            b, e = int(tile_off[t]) // 8, int(tile_off[t + 1]) // 8
            pos = splitmix64(np.arange(e - b, dtype=np.uint64))
            out[t] = np.sum(splitmix64(words[b:e] ^ pos), dtype=np.uint64)
    return out


def plan_order(plan) -> list[tuple[str, str]]:
    """(sender, receiver) copies in store-and-forward order: chain edges in plan
    order, each fan-out group right after its representative received."""
    copies = []
    for e in plan.edges:
        copies.append((e.src, e.dst))
        for s in plan.nvlink_fanout.get(e.dst, []):
            copies.append((e.dst, s))
    return copies


def execute_plan_cpu(plan, buffers: dict, unit_bounds: list[tuple[int, int]],
                     threads: Optional[int] = None) -> dict:
    """Copy every unit along the plan with torch CPU copy_ (all host threads).

    ``buffers`` maps node -> torch uint8 CPU tensor (sources pre-filled).
    Returns per-destination seconds (time its last unit landed) and totals.
    """
    import torch

    if threads:
        torch.set_num_threads(threads)
    t0 = time.perf_counter()
    done = {}
    for src, dst in plan_order(plan):
        for b, e in unit_bounds:  # layer by layer, like the chain forwards units
            buffers[dst][b:e].copy_(buffers[src][b:e])
        done[dst] = time.perf_counter() - t0
    return done
