"""Decision parity: replay the reference's frozen outputs (tests/golden, made by
oracle/gen_golden.py from the reference package itself) through our API and
require exact equality -- plans, chains, fan-out, estimates, live pairs,
layer-ownership splits, ZigZag timelines, throughput ramp, C3 trace."""

import json
import math
from pathlib import Path

import pytest

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200.topology import BYTES_PER_GBPS
from oracle.gen_golden import MODELS, topo_docs

GOLDEN = Path(__file__).parent / "golden"


def _load(name):
    return json.loads((GOLDEN / name).read_text())


def _fin(x):
    if isinstance(x, float) and math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return x


PLAN_CASES = _load("plans.json")
PIPE_CASES = _load("pipelines.json")


def _topo(name):
    doc = topo_docs()[name]
    return ss.load_topology(doc)


@pytest.mark.parametrize("idx", range(len(PLAN_CASES)))
def test_plan_case_matches_reference(idx):
    case = PLAN_CASES[idx]
    topo = _topo(case["topo"])
    flows = ss.FlowSet(topo)
    for src, dst, gbps, label in case["flows"]:
        flows.register(src, dst, gbps, label)
    model = ss.ModelSpec(**MODELS[case["model"]])
    group, prune, eta = case.get("group", True), case.get("prune", True), case.get("eta", 1.0)
    req = ss.build_scale_request(model, case["sources"], case["targets"], topo, flows)
    assert [[s.node, s.outcast_gbps] for s in req.sources] == case["request"]["sources"]
    assert [[t.node, t.incast_gbps, t.outcast_gbps] for t in req.targets] == \
        case["request"]["targets"]
    if "error" in case:
        with pytest.raises(Exception) as info:
            ss.generate_plan(req, topo, flows, group=group, prune=prune)
        assert type(info.value).__name__ == case["error"]
        return
    plan = ss.generate_plan(req, topo, flows, group=group, prune=prune)
    assert [[e.src, e.dst, e.gbps, e.kind] for e in plan.edges] == case["plan"]["edges"]
    assert plan.chains == case["plan"]["chains"]
    assert plan.nvlink_fanout == case["plan"]["fanout"]
    assert {t: plan.depth_of(t) for t in plan.targets()} == case["depth"]
    assert {t: _fin(plan.path_bottleneck(t)) for t in plan.targets()} == case["bottleneck_path"]
    est = ss.estimate_completion(plan, model, topo, eta=eta)
    assert est.per_target_completion == case["completion"]
    assert {str(k): _fin(v) for k, v in est.bottleneck_gbps.items()} == case["chain_bottleneck"]
    assert ss.plan_is_interference_free(plan, flows, topo) == case["interference_free"]
    for node, expected in case["layer_arrivals"].items():
        bw = plan.path_bottleneck(node) * eta * BYTES_PER_GBPS
        d = plan.depth_of(node)
        got = [(d - 1 + k) * model.layer_shard_bytes / bw for k in range(1, model.num_layers + 1)]
        assert got == expected
    pairs = ss.select_live_pairs(plan, est, [f"inst{i}" for i in range(3)], ss.SloProfile(0.25))
    assert [list(p) for p in pairs] == case["live_pairs"]


@pytest.mark.parametrize("idx", range(len(PIPE_CASES)))
def test_pipeline_case_matches_reference(idx):
    case = PIPE_CASES[idx]
    tl = math.inf if case["time_l"] == "inf" else case["time_l"]
    if "error" in case:
        with pytest.raises(Exception) as info:
            ss.configure_pipeline(case["n"], case["L"], tl, weights=case["weights"],
                                  first_layer_offset=case["offset"], c3_form=case["c3_form"])
        assert type(info.value).__name__ == case["error"]
        return
    cfg = ss.configure_pipeline(case["n"], case["L"], tl, weights=case["weights"],
                                first_layer_offset=case["offset"], c3_form=case["c3_form"])
    assert [list(s) for s in cfg.splits] == case["splits"]
    assert cfg.objective() == case["objective"]
    assert cfg.constraint_violations() == case["violations"]
    if "zigzag" in case:
        z = ss.zigzag_schedule(cfg)
        assert [list(x) for x in z.target_intervals] == case["zigzag"]["target"]
        assert [list(x) for x in z.source_intervals] == case["zigzag"]["source"]
        assert z.prefix_done == case["zigzag"]["prefix_done"]
        assert z.finish == case["zigzag"]["finish"]
        assert z.average_latency == case["zigzag"]["average"]
    else:
        with pytest.raises(Exception) as info:
            ss.zigzag_schedule(cfg)
        assert type(info.value).__name__ == case["zigzag_error"]
    if "best_effort" in case:
        be = ss.best_effort_pipeline(case["n"], case["L"], tl, weights=case["weights"])
        assert [list(s) for s in be.splits] == case["best_effort"]
        assert be.objective() == case["best_effort_objective"]


def test_throughput_ramp_matches_reference():
    for L, values in _load("ramp.json").items():
        L = int(L)
        assert [ss.steady_state_throughput(L, k) for k in range(L + 1)] == values


def test_c3_trace_matches_reference(tmp_path):
    trace = ss.generate_trace("burst", {"rate_per_s": 8, "duration_s": 30,
                                        "prompt_tokens": [512, 2048], "output_tokens": [16, 128],
                                        "bursts": [{"start_s": 10, "duration_s": 2,
                                                    "multiplier": 5}]}, seed=1)
    frozen = ss.load_trace(GOLDEN / "c3_burst_trace.jsonl")
    assert trace == frozen


def test_baseline_load_matches_reference():
    for row in _load("baseline_load.json"):
        topo = _topo(row["topo"])
        model = ss.ModelSpec(**MODELS[row["model"]])
        assert ss.baseline_load_time("allcache", model, topo, eta=row["eta"]) == row["allcache"]


def test_fig11_golden():
    """PAPER.md:856 / SURVEY.md §3.3: zigzag splits and finish times for N=6, L=7, time_l=6."""
    cfg = ss.configure_pipeline(6, 7, 6.0)
    assert cfg.splits == [(1, 6), (2, 5), (2, 5), (3, 4), (4, 3), (4, 3)]
    assert cfg.objective() == 17.0
    assert ss.zigzag_schedule(cfg).finish == [7, 12, 17, 21, 24, 27]
    assert ss.best_effort_pipeline(6, 7, 6.0).splits == [(1, 6)] * 6
