"""the simulator's scale-ups executed in process.

``simscale._scale_via_network`` (the reference's simcore.py:676-750 caller) hands
each plan to ``ExecutedCosts.on_plan``; the data plane moves the bytes and the
replay's ``layer`` / ``transfer`` events (simcore.py:727-738) carry the device
stamps of that execution.  One GPU: stream-ordered loopback; two or more: one
plan GPU per device, hops concurrent over NVLink.
"""

import pytest
import torch

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import simcore
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.inprocess import ExecutedCosts, LocalPlanExecutor

pytestmark = pytest.mark.gpu


def _plan(srcs, tgts, arch=S.TINY_4L, topo="b200-hgx"):
    t = ss.load_topology(topo)
    f = ss.FlowSet(t)
    return ss.generate_plan(ss.build_scale_request(S.model_spec_for(arch), srcs, tgts, t, f), t, f)


def _check(ex, nodes, L):
    assert ex is not None and ex.bit_exact
    for n in nodes:
        a = ex.arrivals_s[n]
        assert len(a) == L and all(x > 0 for x in a) and a == sorted(a)


def test_loopback_execution_is_bit_exact_and_stamped():
    pe = LocalPlanExecutor(S.TINY_4L, [0], tile_bytes=256 * 1024, nctas=8, loopback=True)
    try:
        _check(pe.execute(_plan(["gpu0"], ["gpu1", "gpu2", "gpu3"])), ["gpu1", "gpu2", "gpu3"], 4)
        ex = pe.execute(_plan(["mem0"], ["gpu0", "gpu1"]))
        _check(ex, ["gpu0", "gpu1"], 4)
        hl = pe.host_load()
        _check(hl, ["host-load"], 4)
    finally:
        pe.close()


@pytest.mark.multigpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_device_execution_over_nvlink():
    n = min(torch.cuda.device_count(), 4)
    pe = LocalPlanExecutor(S.TINY_4L, list(range(n)), tile_bytes=256 * 1024, nctas=8)
    try:
        tg = [f"gpu{i}" for i in range(1, n)]
        ex = pe.execute(_plan(["gpu0"], tg))
        assert ex.mode == "devices"
        _check(ex, tg, 4)
    finally:
        pe.close()


def test_simulation_scale_events_are_executed():
    """A short burst replay: every network scale-up the simulator plans is executed
    (bit-exact), and the stop-the-world strategy's loads are real host-cache loads."""
    trace = ss.generate_trace("burst", {"rate_per_s": 20, "duration_s": 14, "prompt_tokens": [512, 2048],
                                        "output_tokens": [16, 64],
                                        "bursts": [{"start_s": 4, "duration_s": 2, "multiplier": 5}]}, seed=1)
    spec = S.model_spec_for(S.TINY_4L)
    topo = ss.load_topology("b200-hgx")
    pe = LocalPlanExecutor(S.TINY_4L, [0], tile_bytes=256 * 1024, nctas=8, loopback=True)
    try:
        for strat, mode in (("blitz-live", "loopback"), ("allcache", "host-load")):
            costs = ExecutedCosts(pe)
            res = simcore.run_simulation(topo, [spec], trace, simcore.SimPolicy(strategy=strat), costs=costs)
            summ = res.summary()
            assert summ["counters"]["scale_ups"] >= 1
            assert costs.executions and all(e.bit_exact for e in costs.executions)
            assert {e.mode for e in costs.executions} == {mode}
            assert summ["ttft_ms"]["p99"] > 0
            d = costs.describe()
            assert d["executed_bit_exact"] and d["executed"].get(mode, 0) == len(costs.executions)
    finally:
        pe.close()
