"""C3 on the real clock (two B200s, one process): a 5x-burst trace served by real
Llama-2 7B prefills; the scale-up is triggered by the reference policy and executed
by the data plane.  Prints one JSON line with p50/p99 TTFT per strategy.

  python scripts/c3_realclock.py [rate_per_s] [duration_s] [n_gpus]
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2412_17246_b200 as ss  # noqa: E402
from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200.realclock import RealClockServer  # noqa: E402


def main():
    rate = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
    duration = float(sys.argv[2]) if len(sys.argv) > 2 else 12.0
    burst_at = duration / 3
    trace = ss.generate_trace("burst", {"rate_per_s": rate, "duration_s": duration, "prompt_tokens": [512, 2048],
                                        "output_tokens": [16, 128],
                                        "bursts": [{"start_s": burst_at, "duration_s": 2, "multiplier": 5}]},
                              seed=1)
    arrivals = [(r.arrival_ms / 1e3, r.prompt_tokens) for r in trace]
    n_gpus = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    srv = RealClockServer(S.LLAMA2_7B, extra_devs=list(range(2, n_gpus)))
    mean_tok = sum(n for _, n in arrivals) / len(arrivals)
    # measured capacity of one instance: mean over the trace's bucket mix
    mean_ms = sum(srv.prefill_ms(n, iters=2) for _, n in arrivals[:64]) / min(64, len(arrivals))
    pre_ms = mean_ms
    capacity = mean_tok / (pre_ms / 1e3)          # prefill tokens/s of one instance, measured
    out = {"n_gpus": n_gpus, "trace": f"burst {rate:g} req/s x {duration:g} s, 5x for 2 s at t={burst_at:g} s, seed 1 "
                    f"({len(arrivals)} requests, mean prompt {mean_tok:.0f} tokens)",
           "model": "llama2-7b (random-init bf16, one request per prefill, prompts padded to 256-token buckets)",
           "instance_capacity_tok_s": capacity, "prefill_ms_at_mean_prompt": pre_ms, "strategies": {}}
    for strat in ("static", "allcache", "live-host", "blitz"):
        r = srv.run(arrivals, strat, capacity)
        out["strategies"][strat] = {k: getattr(r, k) for k in (
            "p50_ttft_ms", "p99_ttft_ms", "mean_ttft_ms", "scale_trigger_s", "scale_ready_s", "load_ms",
            "served", "wall_s", "pair_runs", "instances_added", "all_ready_s")}
        print(f"[c3rc] {strat}: p99 {r.p99_ttft_ms:.1f} ms p50 {r.p50_ttft_ms:.1f} load {r.load_ms} "
              f"added {r.instances_added} all ready at {r.all_ready_s}", flush=True)
    srv.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
