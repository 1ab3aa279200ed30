"""Measured serving flows in the FlowSet: the rate a real
KV stream achieved is what pruning, per-edge bandwidth and the interference check
see (planner.py:147-159, 265-285; topology.py:266-292, 325-406)."""

import pytest

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.kvflows import MeasuredFlow, gbps_of


def test_measured_flow_drives_pruning_and_bandwidth():
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    model = S.model_spec_for(S.LLAMA2_7B)
    free = ss.build_scale_request(model, ["gpu0", "gpu1"], ["gpu2", "gpu3"], topo, flows)
    f = MeasuredFlow(flows, "gpu0", "gpu1")
    # 4 x 2 GiB pushed in 12.9 ms -> 666 GB/s -> 5327 Gbps
    g = f.update(4 * (2 << 30), 12.9)
    assert g == pytest.approx(gbps_of(4 * (2 << 30), 12.9)) and not f.clamped
    assert flows.outbound_serving_nodes() == {"gpu0"} and len(flows) == 1
    req = ss.build_scale_request(model, ["gpu0", "gpu1"], ["gpu2", "gpu3"], topo, flows)
    out = {s.node: s.outcast_gbps for s in req.sources}
    out_free = {s.node: s.outcast_gbps for s in free.sources}
    assert out["gpu0"] == pytest.approx(out_free["gpu0"] - g)     # egress derated by the measured rate
    assert out["gpu1"] == pytest.approx(out_free["gpu1"])
    plan = ss.generate_plan(req, topo, flows, group=False, prune=True)
    assert all(e.src != "gpu0" for e in plan.edges)                # the serving sender is pruned
    assert ss.plan_is_interference_free(plan, flows, topo)
    naive = ss.ScalePlan(edges=[ss.planner.PlanEdge("gpu0", "gpu2", 7200.0, "nvlink")], chains=[["gpu0", "gpu2"]])
    assert not ss.plan_is_interference_free(naive, flows, topo)
    # a new window replaces the registration; a rate above the free capacity is clamped
    f.update(4 * (2 << 30), 5.0)
    assert f.clamped and len(flows) == 1 and f.gbps <= topo.link("gpu0", "gpu1").gbps
    f.release()
    assert len(flows) == 0 and flows.outbound_serving_nodes() == set()
