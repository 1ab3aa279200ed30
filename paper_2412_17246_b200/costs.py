"""Measured B200 costs for the serving replay (C3: 7B live scaling under a burst).

``simcore.ReferenceCosts`` is the reference's analytic model.  ``MeasuredCosts``
replaces, at the hot-path call sites of the replay, every time the data plane
and the cooperative executor actually determine on B200:

* per-layer arrival of a new instance's weights (``simcore.py:727-733``) and its
  completion (``:735-738``) -- from the tracker stamps of executed plans:
  NVLink hop from a live source, NVLS fan-out, O(1) host-cache staging;
* stop-the-world AllCache load (``autoscaler.py:102-117``) -- measured host staging;
* prefill batch time (``parampool.py:58-59``) -- a least-squares line through
  measured 7B forward passes of the tcgen05 Llama executor;
* the profiled capacity bound (``autoscaler.py:120-126``) from that line;
* decode step time (``parampool.py:61-62``) -- a line through measured KV-cache
  decode steps of the same executor.

* the ServerlessLLM cache-miss load from local storage -- a measured disk ->
  pinned host -> HBM pipeline rate (``calibrate.measure_ssd_load``).

RDMA edges are not executed on this single box; they keep the reference model
and are labelled as such in ``describe()``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

from .simcore import ReferenceCosts


def fit_line(xs: Sequence[float], ys: Sequence[float]) -> tuple[float, float]:
    """Least-squares (alpha, beta) of y = alpha + beta * x."""
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    beta = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx if sxx else 0.0
    return my - beta * mx, beta


@dataclass
class MeasuredCosts(ReferenceCosts):
    """Times measured on B200; ``None`` fields fall back to the reference model."""

    prefill_alpha_ms: Optional[float] = None
    prefill_beta_ms: Optional[float] = None
    nvlink_layer_ms: Optional[list[float]] = None   # arrival of unit k after a 1-hop NVLink scale cmd
    nvlink_hop_fill_ms: float = 0.0                   # extra per chain hop (one tile)
    host_layer_ms: Optional[list[float]] = None       # arrival of unit k from the pinned host cache
    decode_alpha_ms: Optional[float] = None
    decode_beta_ms: Optional[float] = None
    ssd_to_gpu_gbs: Optional[float] = None            # measured disk -> pinned -> HBM rate (GB/s)
    source: dict = field(default_factory=dict)

    name = "b200-measured"

    def prefill_ms(self, model, tokens: int) -> float:
        if self.prefill_alpha_ms is None:
            return super().prefill_ms(model, tokens)
        return self.prefill_alpha_ms + self.prefill_beta_ms * tokens

    def decode_step_ms(self, model, batch: int) -> float:
        if self.decode_alpha_ms is None:
            return super().decode_step_ms(model, batch)
        return self.decode_alpha_ms + self.decode_beta_ms * batch

    def capacity_tokens_per_s(self, model, budget: int) -> float:
        return budget / (self.prefill_ms(model, budget) / 1000.0)

    def _path_kinds(self, plan, node: str) -> list[str]:
        parent = {e.dst: e for e in plan.edges}
        kinds = []
        while node in parent:
            e = parent[node]
            kinds.append(e.kind)
            node = e.src
        return kinds

    def layer_arrival_s(self, plan, node, model, eta) -> list[float]:
        kinds = self._path_kinds(plan, node)
        if kinds and all(k == "nvlink" for k in kinds) and self.nvlink_layer_ms \
                and len(self.nvlink_layer_ms) == model.num_layers:
            extra = (len(kinds) - 1) * self.nvlink_hop_fill_ms
            return [(t + extra) / 1e3 for t in self.nvlink_layer_ms]
        if kinds == ["pcie"] and self.host_layer_ms and len(self.host_layer_ms) == model.num_layers:
            return [t / 1e3 for t in self.host_layer_ms]
        return super().layer_arrival_s(plan, node, model, eta)

    def completion_s(self, plan, est, node, model, eta) -> float:
        fan_rep = {s: rep for rep, sibs in plan.nvlink_fanout.items() for s in sibs}
        if node in fan_rep:
            # NVLS fan-out lands with (not after) the representative on B200
            return self.layer_arrival_s(plan, fan_rep[node], model, eta)[-1]
        kinds = self._path_kinds(plan, node)
        if kinds and (all(k == "nvlink" for k in kinds) or kinds == ["pcie"]):
            return self.layer_arrival_s(plan, node, model, eta)[-1]
        return super().completion_s(plan, est, node, model, eta)

    def _host_load_s(self, model) -> Optional[float]:
        if self.host_layer_ms and len(self.host_layer_ms) == model.num_layers:
            return self.host_layer_ms[-1] / 1e3
        return None

    def stop_the_world_s(self, strategy, model, topo, pool, host_id, now_s, eta) -> float:
        """AllCache and a ServerlessLLM keep-alive hit load from the host cache; a
        ServerlessLLM miss reads the checkpoint from local storage (autoscaler.py:102-117)."""
        host_s = self._host_load_s(model)
        if strategy == "allcache" and host_s is not None:
            return host_s
        if strategy == "sllm":
            hit = pool is not None and host_id is not None and pool.cache_hit(model.name, host_id, now_s)
            if hit and host_s is not None:
                return host_s
            if not hit and self.ssd_to_gpu_gbs:
                return model.shard_bytes / (self.ssd_to_gpu_gbs * 1e9)
        return super().stop_the_world_s(strategy, model, topo, pool, host_id, now_s, eta)

    def describe(self) -> dict:
        return {
            "prefill_ms": ("measured" if self.prefill_alpha_ms is not None else "reference-model"),
            "prefill_alpha_ms": self.prefill_alpha_ms, "prefill_beta_ms": self.prefill_beta_ms,
            "nvlink_layers": "measured" if self.nvlink_layer_ms else "reference-model",
            "host_cache_layers": "measured" if self.host_layer_ms else "reference-model",
            "decode": "measured" if self.decode_alpha_ms is not None else "reference-model",
            "decode_alpha_ms": self.decode_alpha_ms, "decode_beta_ms": self.decode_beta_ms,
            "ssd_load": "measured" if self.ssd_to_gpu_gbs else "reference-model",
            "ssd_to_gpu_GBps": self.ssd_to_gpu_gbs,
            "rdma edges": "reference-model",
            **self.source,
        }
