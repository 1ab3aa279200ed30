"""Measured serving flows in the reference's ``FlowSet``.

The reference accounts a KV-cache P/D transfer as a ``kvcache`` flow registered
at a modeled rate (simcore.py:462-514, ``FlowSet.register``, topology.py:325-406);
the planner then prunes senders that carry serving traffic
(``prune_sources``, planner.py:147-159), and ``build_scale_request`` derates every
node's NVLink out/in bandwidth by the flows on its ports (topology.py:266-292).
``MeasuredFlow`` keeps such a registration in step with a real transfer: the KV
bytes a GPU actually pushed over NVLink in a timed window give the rate the
FlowSet carries, so pruning, per-edge bandwidth and ``plan_is_interference_free``
all see the link occupancy that was measured, not a constant.
"""

from __future__ import annotations

from typing import Optional

from .topology import BYTES_PER_GBPS, CapacityError, FlowSet


def gbps_of(nbytes: float, ms: float) -> float:
    """Rate of ``nbytes`` moved in ``ms`` milliseconds, in the reference's Gbps unit."""
    return nbytes / BYTES_PER_GBPS / (ms / 1e3)


class MeasuredFlow:
    """One live flow ``src -> dst`` registered in ``flows`` at its measured rate."""

    def __init__(self, flows: FlowSet, src: str, dst: str, label: str = "kvcache"):
        self.flows, self.src, self.dst, self.label = flows, src, dst, label
        self.gbps: Optional[float] = None
        self.clamped = False

    def update(self, nbytes: float, ms: float) -> float:
        """Re-register at the rate of the last window (``nbytes`` in ``ms``); a rate above
        what the link / ports still have free is clamped to it.  Returns the Gbps held."""
        rate = gbps_of(nbytes, ms)
        self.release()
        topo = self.flows.topo
        link = topo.link(self.src, self.dst)
        free = min(link.gbps - self.flows.on_link(self.src, self.dst),
                   topo.outcast_bandwidth(self.src, self.flows), topo.incast_bandwidth(self.dst, self.flows))
        self.clamped = rate > free
        rate = min(rate, free)
        if rate <= 0:
            raise CapacityError(f"no capacity left on {self.src} -> {self.dst}")
        self.flows.register(self.src, self.dst, rate, self.label)
        self.gbps = rate
        return rate

    def release(self):
        if self.gbps is not None:
            self.flows.release(self.src, self.dst, self.gbps, self.label)
            self.gbps = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.release()
