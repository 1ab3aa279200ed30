"""Simulator parity: our replay of the hot path's caller reproduces the reference
simulator's summary() (TTFT/TBT percentiles, SLO attainment, counters and every
scale event: plans, chains, fan-out, modeled completions, live targets) and its
utilisation series, value for value, on the frozen cases of oracle/gen_golden.py."""

import json
from pathlib import Path

import pytest

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import simcore
from oracle.gen_golden import MODELS, SIM_CASES, SIM_TRACES, topo_docs

GOLDEN = json.loads((Path(__file__).parent / "golden" / "simulations.json").read_text())


@pytest.mark.parametrize("idx", range(len(GOLDEN)))
def test_simulation_matches_reference(idx):
    case = GOLDEN[idx]
    kind, params, seed = SIM_TRACES[case["trace"]]
    trace = ss.generate_trace(kind, params, seed)
    topo = ss.load_topology(topo_docs()[case["topo"]])
    model = ss.ModelSpec(**MODELS[case["model"]])
    res = simcore.run_simulation(topo, [model], trace, simcore.SimPolicy(strategy=case["strategy"]))
    assert json.loads(json.dumps(res.summary())) == case["summary"]
    assert json.loads(json.dumps(res.series)) == case["series"]


def test_cases_cover_every_strategy():
    assert {c[3] for c in SIM_CASES} == {"blitz-live", "blitz-stop", "allcache", "sllm", "static"}


def test_unsorted_trace_rejected():
    t = [ss.TraceRecord(5.0, 10, 2), ss.TraceRecord(1.0, 10, 2)]
    with pytest.raises(simcore.SimulationError):
        simcore.run_simulation(ss.load_topology("b200-hgx"), [ss.MODEL_PRESETS["llama2-7b"]], t,
                               simcore.SimPolicy())
