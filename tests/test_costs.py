"""Measured-cost hooks of the serving replay (C3) -- CPU checks.

With ``MeasuredCosts`` left empty the replay must equal the reference model
exactly; with measured curves the hot-path events must come from them."""

import json

import pytest

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import simcore
from paper_2412_17246_b200.calibrate import build_costs, c3_report
from paper_2412_17246_b200.costs import MeasuredCosts, fit_line
from paper_2412_17246_b200.slab import LLAMA2_7B, model_spec_for


def test_fit_line_exact():
    a, b = fit_line([1, 2, 3, 4], [3, 5, 7, 9])
    assert a == pytest.approx(1.0) and b == pytest.approx(2.0)


def _trace():
    return ss.generate_trace("burst", {"rate_per_s": 10, "duration_s": 8, "prompt_tokens": [256, 1024],
                                       "output_tokens": [4, 32],
                                       "bursts": [{"start_s": 2, "duration_s": 2, "multiplier": 5}]}, 2)


def test_empty_measured_costs_equal_reference_model():
    topo = ss.load_topology("b200-hgx-2x8")
    spec = model_spec_for(LLAMA2_7B)
    a = simcore.run_simulation(topo, [spec], _trace(), simcore.SimPolicy())
    b = simcore.run_simulation(topo, [spec], _trace(), simcore.SimPolicy(), costs=MeasuredCosts())
    assert json.dumps(a.summary()) == json.dumps(b.summary())


def test_measured_layer_arrivals_drive_events():
    spec = model_spec_for(LLAMA2_7B)
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    plan = ss.generate_plan(ss.build_scale_request(spec, ["gpu0"], ["gpu1", "gpu2"], topo, flows),
                            topo, flows, group=False)
    nv = [0.6 * (k + 1) for k in range(32)]
    c = MeasuredCosts(nvlink_layer_ms=nv, nvlink_hop_fill_ms=0.01)
    assert c.layer_arrival_s(plan, "gpu1", spec, 0.8) == pytest.approx([t / 1e3 for t in nv])
    assert c.layer_arrival_s(plan, "gpu2", spec, 0.8)[0] == pytest.approx((0.6 + 0.01) / 1e3)
    est = ss.estimate_completion(plan, spec, topo, eta=0.8)
    assert c.completion_s(plan, est, "gpu2", spec, 0.8) == pytest.approx((19.2 + 0.01) / 1e3)
    # rdma edges keep the reference model
    topo2 = ss.load_topology("b200-hgx-2x8")
    f2 = ss.FlowSet(topo2)
    p2 = ss.generate_plan(ss.build_scale_request(spec, ["gpu0"], ["gpu8"], topo2, f2), topo2, f2)
    e2 = ss.estimate_completion(p2, spec, topo2, eta=0.8)
    assert c.completion_s(p2, e2, "gpu8", spec, 0.8) == e2.per_target_completion["gpu8"]


def test_c3_report_shape():
    c = build_costs(prefill={512: 10.0, 2048: 25.0}, host_layer_ms=[8.0 * (k + 1) for k in range(32)])
    r = c3_report(c, strategies=("blitz-live", "allcache"))
    assert "730 requests" in r["trace"]
    for s in ("blitz-live", "allcache"):
        assert set(r["strategies"][s]) == {"modeled", "measured"}
        assert r["strategies"][s]["measured"]["p99_ttft_ms"] > 0


def test_sllm_load_uses_host_on_hit_and_storage_on_miss():
    """autoscaler.py:102-117 with measured rates: a keep-alive hit loads from the
    pinned host cache (the measured host-staging time), a miss from local storage
    (the measured disk -> HBM rate); without measurements the reference model."""
    spec = model_spec_for(LLAMA2_7B)
    topo = ss.load_topology("b200-hgx")
    pool = ss.ParameterPool.init_pool([spec], topo, policy="keep-alive")
    host = pool.cache_refs[spec.name][0].host_id
    c = MeasuredCosts(host_layer_ms=[10.0 * (k + 1) for k in range(spec.num_layers)], ssd_to_gpu_gbs=4.0)
    hit = c.stop_the_world_s("sllm", spec, topo, pool, host, 0.0, 1.0)
    miss = c.stop_the_world_s("sllm", spec, topo, pool, host, 1e6, 1.0)   # keep-alive expired
    assert hit == pytest.approx(0.32)
    assert miss == pytest.approx(spec.shard_bytes / 4e9)
    ref = simcore.ReferenceCosts()
    assert MeasuredCosts().stop_the_world_s("sllm", spec, topo, pool, host, 1e6, 1.0) == \
        ref.stop_the_world_s("sllm", spec, topo, pool, host, 1e6, 1.0)
    assert c.describe()["ssd_load"] == "measured"
