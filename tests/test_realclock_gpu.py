"""Real-clock serving with decode: prefills on the wall
clock, every request then decodes its trace's output tokens in its instance's
continuous batch (per-row device positions), TTFT and TBT observed, not modeled.

One GPU: the new instance shares the GPU with the source and loads from the host
cache (copy engines + in-stream publish -- no kernel waits on another kernel of
the same GPU); more GPUs run the NVLink variants in test_multigpu.py."""

import pytest
import torch

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.realclock import RealClockServer

pytestmark = pytest.mark.gpu


def test_realclock_decode_one_gpu():
    trace = ss.generate_trace("burst", {"rate_per_s": 150, "duration_s": 2, "prompt_tokens": [512, 2048],
                                        "output_tokens": [4, 24],
                                        "bursts": [{"start_s": 0.8, "duration_s": 0.5, "multiplier": 5}]}, seed=4)
    arrivals = [(r.arrival_ms / 1e3, r.prompt_tokens, r.output_tokens) for r in trace]
    srv = RealClockServer(S.TINY_4L, src_dev=0, tgt_dev=0, decode_slots=16, max_new_tokens=32)
    try:
        mean_tok = sum(a[1] for a in arrivals) / len(arrivals)
        for strat in ("static", "allcache"):
            r = srv.run(arrivals, strat, 2.0 * 150 * mean_tok)
            assert r.n == len(arrivals) and r.p99_ttft_ms > 0
            assert r.decode_steps > 0 and r.p99_tbt_ms is not None and r.p99_tbt_ms > 0
            assert r.p50_tbt_ms <= r.p99_tbt_ms
            if strat == "allcache":
                assert r.instances_added == 1 and r.load_ms is not None and r.load_ms > 0
    finally:
        srv.close()
