"""Generate golden decision vectors by running the REFERENCE package itself.

TEST INFRASTRUCTURE ONLY (oracle/): nothing in the product imports this.

Runs ``scalesim`` from ``/root/reference/pkg/src`` (read-only, this container
only -- the GPU box has no /root/reference) over a deterministic case list and
writes the inputs + reference outputs to ``tests/golden/*.json``.  The parity
tests replay the same inputs through ``paper_2412_17246_b200`` and demand
exact equality (JSON floats round-trip exactly through ``repr``).

Covered reference items:
  a1 build_scale_request    planner.py:288-297
  a2 group_targets          planner.py:121-144
  a3 prune_sources          planner.py:147-159
  a4 generate_plan          planner.py:162-209 (+ _derive_chains 212-224)
  a5 depth_of / path_bottleneck planner.py:95-109
  a6 estimate_completion    planner.py:227-262
  a7 plan_is_interference_free planner.py:265-285
  a12 baseline_load_time    autoscaler.py:102-117
  a13 per-layer arrival model simcore.py:727-733 / default_layer_load_times livescale.py:264-266
  a15 select_live_pairs     livescale.py:379-405
  a16-a18 configure_pipeline / best_effort_pipeline / objective  livescale.py:53-235
  a19 zigzag_schedule       livescale.py:269-346
  a20 steady_state_throughput livescale.py:349-363
  traces.generate_trace (C3 burst trace, traces.py:49-96)

Usage:  python oracle/gen_golden.py      (rewrites tests/golden/)
"""

from __future__ import annotations

import importlib
import json
import math
import random
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def load_reference():
    if not REF_SRC.exists():
        raise SystemExit("reference not present; golden vectors are generated in the build container")
    sys.path.insert(0, str(REF_SRC))
    return importlib.import_module("scalesim")


def _fin(x):
    """JSON cannot hold inf; encode it as a string."""
    if isinstance(x, float) and math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return x


# ---- topologies used by the cases -------------------------------------------------

def topo_docs():
    docs = {
        "b200-hgx": {"hosts": [{"id": 0, "gpus": 8, "host_gpu_gbps": 512.0, "ssd_gpu_gbps": 50.0}],
                     "intra": {"kind": "nvlink", "gbps": 7200.0}, "inter": {"gbps": 400.0}},
        "cluster-A": "cluster-A",
        "cluster-B": "cluster-B",
        "p5.48xlarge": "p5.48xlarge",
        "flat4": {"hosts": [{"id": h, "gpus": 1, "host_gpu_gbps": 10000.0, "ssd_gpu_gbps": 10000.0}
                             for h in range(4)],
                  "intra": {"kind": "none", "gbps": 0}, "inter": {"gbps": 10000.0}},
        "flat6": {"hosts": [{"id": h, "gpus": 1, "host_gpu_gbps": 10000.0, "ssd_gpu_gbps": 10000.0}
                             for h in range(6)],
                  "intra": {"kind": "none", "gbps": 0}, "inter": {"gbps": 10000.0}},
        "shared-nic": {"hosts": [{"id": 0, "gpus": [0, 1, 2, 3], "host_gpu_gbps": 128, "ssd_gpu_gbps": 10,
                                  "nic_groups": [[0, 1], [2, 3]]},
                                 {"id": 1, "gpus": [4, 5, 6, 7], "host_gpu_gbps": 128, "ssd_gpu_gbps": 10,
                                  "nic_groups": [[4, 5], [6, 7]]}],
                       "intra": {"kind": "pcie", "gbps": 256}, "inter": {"gbps": 100}},
        "b200-2x8": {"hosts": [{"id": h, "gpus": 8, "host_gpu_gbps": 512.0, "ssd_gpu_gbps": 50.0}
                                for h in range(2)],
                     "intra": {"kind": "nvlink", "gbps": 7200.0}, "inter": {"gbps": 400.0}},
    }
    return docs


MODELS = {
    "llama2-7b": dict(name="llama2-7b", num_layers=32, bytes_per_layer=437_500_000.0),
    "llama2-70b": dict(name="llama2-70b", num_layers=80, bytes_per_layer=1_750_000_000.0,
                       tp_degree=4),
    # real Llama-2 byte totals, uniform per-layer share (SURVEY.md §7.2 "plan granularity")
    "llama2-7b-real": dict(name="llama2-7b-real", num_layers=32,
                           bytes_per_layer=13_476_831_232 / 32),
    "llama2-13b-tp2": dict(name="llama2-13b-tp2", num_layers=40,
                           bytes_per_layer=26_031_728_640 / 40, tp_degree=2),
    "tiny-4l": dict(name="tiny-4l", num_layers=4, bytes_per_layer=39_096_832 / 4),
}


def plan_cases():
    """Named BASELINE configs (C1-C5 anchors) plus a seeded fuzz over all topologies."""
    cases = [
        # C1 tiny 1->2 on one B200 box
        dict(topo="b200-hgx", model="tiny-4l", sources=["gpu0"], targets=["gpu1"], flows=[]),
        # C2 7B 1->2 / 1->4 / 1->8
        dict(topo="b200-hgx", model="llama2-7b-real", sources=["gpu0"], targets=["gpu1"], flows=[]),
        dict(topo="b200-hgx", model="llama2-7b-real", sources=["gpu0"],
             targets=["gpu1", "gpu2", "gpu3"], flows=[]),
        dict(topo="b200-hgx", model="llama2-7b-real", sources=["gpu0"],
             targets=[f"gpu{i}" for i in range(1, 8)], flows=[]),
        # C4 13B TP=2: anchors of 4 instances, source anchor gpu0
        dict(topo="b200-hgx", model="llama2-13b-tp2", sources=["gpu0"],
             targets=["gpu2", "gpu4", "gpu6"], flows=[]),
        # C5 70B TP=4: host cache -> group anchors gpu0, gpu4
        dict(topo="b200-hgx", model="llama2-70b", sources=["mem0"], targets=["gpu0", "gpu4"],
             flows=[]),
        # cross-host B200 pair with serving traffic
        dict(topo="b200-2x8", model="llama2-7b", sources=["gpu0", "gpu1", "mem0"],
             targets=["gpu8", "gpu9", "gpu10", "gpu3"],
             flows=[["gpu0", "gpu9", 50.0, "kvcache"]]),
    ]
    rng = random.Random(20241217)
    docs = topo_docs()
    nodes = {"b200-hgx": 8, "cluster-A": 32, "cluster-B": 16, "p5.48xlarge": 16, "flat4": 4,
             "flat6": 6, "shared-nic": 8, "b200-2x8": 16}
    hosts = {"b200-hgx": 1, "cluster-A": 4, "cluster-B": 2, "p5.48xlarge": 2, "flat4": 4,
             "flat6": 6, "shared-nic": 2, "b200-2x8": 2}
    for _ in range(220):
        topo = rng.choice(sorted(docs))
        n = nodes[topo]
        gpus = [f"gpu{i}" for i in range(n)]
        rng.shuffle(gpus)
        n_src = rng.randint(1, min(3, n - 1))
        n_tgt = rng.randint(1, min(8, n - n_src))
        srcs = gpus[:n_src]
        tgts = gpus[n_src:n_src + n_tgt]
        if rng.random() < 0.5:
            srcs.append(f"mem{rng.randrange(hosts[topo])}")
        flows = []
        others = gpus[n_src + n_tgt:] + srcs[:1]
        for _k in range(rng.randint(0, 3)):
            a, b = rng.sample(gpus, 2)
            flows.append([a, b, float(rng.choice([5, 10, 15, 25, 50])),
                          rng.choice(["kvcache", "activation", "scale"])])
        cases.append(dict(topo=topo, model=rng.choice(sorted(MODELS)), sources=srcs, targets=tgts,
                          flows=flows, group=rng.random() < 0.7, prune=rng.random() < 0.8,
                          eta=rng.choice([1.0, 0.8, 0.65])))
    return cases


def run_plan_case(ss, case):
    topo = ss.load_topology(topo_docs()[case["topo"]])
    flows = ss.FlowSet(topo)
    registered = []
    for src, dst, gbps, label in case["flows"]:
        try:
            flows.register(src, dst, gbps, label)
            registered.append([src, dst, gbps, label])
        except Exception:  # capacity / missing link: the case records what registered
            pass
    model = ss.ModelSpec(**MODELS[case["model"]])
    group, prune, eta = case.get("group", True), case.get("prune", True), case.get("eta", 1.0)
    out = dict(case, flows=registered)
    req = ss.build_scale_request(model, case["sources"], case["targets"], topo, flows)
    out["request"] = dict(sources=[[s.node, s.outcast_gbps] for s in req.sources],
                          targets=[[t.node, t.incast_gbps, t.outcast_gbps] for t in req.targets])
    try:
        plan = ss.generate_plan(req, topo, flows, group=group, prune=prune)
    except Exception as exc:  # noqa: BLE001 - the exception class is the golden output
        out["error"] = type(exc).__name__
        return out
    est = ss.estimate_completion(plan, model, topo, eta=eta)
    out["plan"] = dict(edges=[[e.src, e.dst, e.gbps, e.kind] for e in plan.edges],
                       chains=plan.chains, fanout=plan.nvlink_fanout)
    out["depth"] = {t: plan.depth_of(t) for t in plan.targets()}
    out["bottleneck_path"] = {t: _fin(plan.path_bottleneck(t)) for t in plan.targets()}
    out["completion"] = est.per_target_completion
    out["chain_bottleneck"] = {str(k): _fin(v) for k, v in est.bottleneck_gbps.items()}
    out["interference_free"] = ss.plan_is_interference_free(plan, flows, topo)
    # per-layer arrival model of the live target (simcore.py:727-733), in seconds
    arrivals = {}
    for e in plan.edges:
        bw = plan.path_bottleneck(e.dst) * eta * ss.topology.BYTES_PER_GBPS
        d = plan.depth_of(e.dst)
        arrivals[e.dst] = [(d - 1 + k) * model.layer_shard_bytes / bw
                           for k in range(1, model.num_layers + 1)]
    out["layer_arrivals"] = arrivals
    over = [f"inst{i}" for i in range(3)]
    pairs = ss.select_live_pairs(plan, est, over, ss.SloProfile(0.25))
    out["live_pairs"] = [list(p) for p in pairs]
    return out


def pipeline_cases():
    rng = random.Random(11)
    cases = []
    for n in (1, 2, 3, 4, 5, 6, 8, 12, 16):
        for L in (1, 3, 4, 7, 8, 32, 40, 80):
            for time_l in (0.0, 0.5, 1.0, 2.0, 6.0, "inf", 0.731):
                cases.append(dict(n=n, L=L, time_l=time_l, weights=None, offset=1,
                                  c3_form="source-prefix"))
    for _ in range(120):
        n = rng.randint(1, 16)
        L = rng.choice([2, 4, 5, 7, 13, 32, 40])
        cases.append(dict(n=n, L=L, time_l=rng.choice([0.25, 0.5, 1.0, 1.5, 3.0, 0.0, 0.73]),
                          weights=[rng.choice([0.5, 1.0, 1.25, 2.0]) * rng.randint(1, 4) / 2
                                   for _ in range(n)],
                          offset=rng.choice([0, 1]),
                          c3_form=rng.choice(["source-prefix", "target-prefix"])))
    return cases


def run_pipeline_case(ss, case):
    tl = math.inf if case["time_l"] == "inf" else case["time_l"]
    out = dict(case)
    try:
        cfg = ss.configure_pipeline(case["n"], case["L"], tl, weights=case["weights"],
                                    first_layer_offset=case["offset"], c3_form=case["c3_form"])
    except Exception as exc:  # noqa: BLE001
        out["error"] = type(exc).__name__
        return out
    out["splits"] = [list(s) for s in cfg.splits]
    out["objective"] = cfg.objective()
    out["violations"] = cfg.constraint_violations()
    try:
        z = ss.zigzag_schedule(cfg)
        out["zigzag"] = dict(target=[list(x) for x in z.target_intervals],
                             source=[list(x) for x in z.source_intervals],
                             prefix_done=z.prefix_done, finish=z.finish,
                             average=z.average_latency)
    except Exception as exc:  # noqa: BLE001
        out["zigzag_error"] = type(exc).__name__
    if case["offset"] == 1 and case["c3_form"] == "source-prefix":
        be = ss.best_effort_pipeline(case["n"], case["L"], tl, weights=case["weights"])
        out["best_effort"] = [list(s) for s in be.splits]
        out["best_effort_objective"] = be.objective()
    return out


SIM_TRACES = {
    "c3-burst": ("burst", {"rate_per_s": 8, "duration_s": 30, "prompt_tokens": [512, 2048],
                           "output_tokens": [16, 128],
                           "bursts": [{"start_s": 10, "duration_s": 2, "multiplier": 5}]}, 1),
    "poisson-small": ("poisson", {"rate_per_s": 6, "duration_s": 12, "prompt_tokens": [128, 1024],
                                  "output_tokens": [2, 48]}, 3),
    "burst-heavy": ("burst", {"rate_per_s": 14, "duration_s": 16, "prompt_tokens": [256, 2048],
                              "output_tokens": [1, 64],
                              "bursts": [{"start_s": 4, "duration_s": 2, "multiplier": 6}]}, 5),
}

SIM_CASES = [
    # (topology doc key, model key, trace key, strategy)
    ("b200-2x8", "llama2-7b", "c3-burst", "blitz-live"),
    ("b200-2x8", "llama2-7b", "c3-burst", "blitz-stop"),
    ("b200-2x8", "llama2-7b", "c3-burst", "allcache"),
    ("b200-2x8", "llama2-7b", "c3-burst", "sllm"),
    ("b200-2x8", "llama2-7b", "c3-burst", "static"),
    ("cluster-A", "llama2-7b", "burst-heavy", "blitz-live"),
    ("cluster-B", "llama2-7b", "burst-heavy", "blitz-live"),
    ("cluster-B", "llama2-7b", "poisson-small", "sllm"),
    ("shared-nic", "llama2-7b", "poisson-small", "blitz-live"),
    ("b200-hgx", "llama2-7b", "burst-heavy", "blitz-live"),
    ("p5.48xlarge", "llama2-70b", "c3-burst", "blitz-live"),
]


def run_sim_cases(ss):
    simcore = importlib.import_module("scalesim.simcore")
    out = []
    for topo_key, model_key, trace_key, strategy in SIM_CASES:
        kind, params, seed = SIM_TRACES[trace_key]
        trace = ss.generate_trace(kind, params, seed)
        topo = ss.load_topology(topo_docs()[topo_key])
        model = ss.ModelSpec(**MODELS[model_key])
        res = simcore.run_simulation(topo, [model], trace, simcore.SimPolicy(strategy=strategy))
        summary = json.loads(json.dumps(res.summary()))
        out.append(dict(topo=topo_key, model=model_key, trace=trace_key, strategy=strategy,
                        summary=summary, series=json.loads(json.dumps(res.series))))
    return out


def decision_workloads(ss, simcore_mod):
    """The reference decision-path items of SURVEY.md §8(d) item 1, as callables
    (used both to time the reference here and our package on the GPU box)."""
    b200 = topo_docs()["b200-hgx"]
    model = ss.ModelSpec(**MODELS["llama2-7b-real"])
    topo = ss.load_topology(b200)
    flows = ss.FlowSet(topo)
    kind, params, seed = SIM_TRACES["c3-burst"]
    trace = ss.generate_trace(kind, {**params, "rate_per_s": 20}, seed)
    topo2 = ss.load_topology(topo_docs()["b200-2x8"])
    targets = [f"gpu{i}" for i in range(1, 8)]

    def plan_1to8():
        req = ss.build_scale_request(model, ["gpu0"], targets, topo, flows)
        plan = ss.generate_plan(req, topo, flows)
        ss.estimate_completion(plan, model, topo, eta=1.0)

    def pipeline(n, L, tl):
        def f():
            cfg = ss.configure_pipeline(n, L, tl)
            ss.zigzag_schedule(cfg)
        return f

    def sim():
        simcore_mod.run_simulation(topo2, [model], trace, simcore_mod.SimPolicy(strategy="blitz-live"))

    return {
        "plan+estimate 1->8 (a1,a4,a6)": plan_1to8,
        "configure_pipeline+zigzag N=16 L=32 time_l=1 (a17,a19)": pipeline(16, 32, 1.0),
        "configure_pipeline+zigzag N=16 L=80 time_l=1 (a17,a19)": pipeline(16, 80, 1.0),
        "run_simulation C3 730 req blitz-live (b200 2x8)": sim,
    }


def time_best(fn, reps=5):
    import time as _t
    best = math.inf
    for _ in range(reps):
        t0 = _t.perf_counter()
        fn()
        best = min(best, _t.perf_counter() - t0)
    return best


def write_timings(ss):
    """Reference decision-path timings next to this package's on the same CPU, same run
    (bench.py reports them beside its on-box timings of our side)."""
    import os
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import paper_2412_17246_b200 as ours
    from paper_2412_17246_b200 import simcore as ours_simcore
    timings = {name: time_best(fn) for name, fn in
               decision_workloads(ss, importlib.import_module("scalesim.simcore")).items()}
    ours_t = {name: time_best(fn) for name, fn in decision_workloads(ours, ours_simcore).items()}
    (OUT / "reference_timings.json").write_text(json.dumps({
        "what": "reference scalesim decision path and this package's, best of 5, single thread (GIL), "
                "same build container, same run",
        "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")
        if os.path.exists("/proc/cpuinfo") else "?",
        "seconds": timings, "ours_seconds": ours_t}, indent=1, sort_keys=True))


def main():
    if "--timings-only" in sys.argv:
        write_timings(load_reference())
        return
    ss = load_reference()
    OUT.mkdir(parents=True, exist_ok=True)
    plans = [run_plan_case(ss, c) for c in plan_cases()]
    (OUT / "plans.json").write_text(json.dumps(plans, sort_keys=True))
    pipes = [run_pipeline_case(ss, c) for c in pipeline_cases()]
    (OUT / "pipelines.json").write_text(json.dumps(pipes, sort_keys=True))
    ramp = {str(L): [ss.steady_state_throughput(L, k) for k in range(0, L + 1)]
            for L in (4, 8, 14, 32)}
    (OUT / "ramp.json").write_text(json.dumps(ramp, sort_keys=True))
    trace = ss.generate_trace("burst", {"rate_per_s": 8, "duration_s": 30,
                                        "prompt_tokens": [512, 2048], "output_tokens": [16, 128],
                                        "bursts": [{"start_s": 10, "duration_s": 2,
                                                    "multiplier": 5}]}, seed=1)
    ss.traces.dump_trace(trace, OUT / "c3_burst_trace.jsonl")
    baselines = []
    for topo_name in ("b200-hgx", "cluster-B", "cluster-A"):
        topo = ss.load_topology(topo_docs()[topo_name])
        for mname in ("llama2-7b", "llama2-70b", "llama2-7b-real"):
            model = ss.ModelSpec(**MODELS[mname])
            for eta in (1.0, 0.8):
                baselines.append(dict(topo=topo_name, model=mname, eta=eta,
                                      allcache=ss.baseline_load_time("allcache", model, topo,
                                                                     eta=eta)))
    (OUT / "baseline_load.json").write_text(json.dumps(baselines, sort_keys=True))
    (OUT / "simulations.json").write_text(json.dumps(run_sim_cases(ss), sort_keys=True))
    write_timings(ss)
    print(f"wrote {len(plans)} plan cases, {len(pipes)} pipeline cases to {OUT}")


if __name__ == "__main__":
    main()
