#!/usr/bin/env python
"""Benchmark of the B200 live-autoscaling data plane (one JSON line on rank 0).

Workloads (BASELINE.json configs):
  N = 1  : O(1) host-cache load of a Llama-2 7B bf16 shard (13.48 GB) into one
           B200 -- plan ``mem0 -> gpu0`` (pcie) from the reference planner,
           copy-engine staging on a side stream + per-layer readiness tracking.
  N >= 2 : live scale-up 1 -> N: the source instance on gpu0 multicasts its
           shard to N-1 new GPUs; plan from ``generate_plan`` (group=True:
           gpu0 -> rep gpu1 over NVLink, the rep's NVLink fan-out realised as a
           pipelined sibling chain -- measured faster than NVLS multimem.st;
           ``--fanout nvls`` selects the multicast realisation).
One step = one complete scale-up (every target holds the bit-exact shard and
its tracker has published every layer).  value = delivered bytes / time
(delivered = shard x number of receiving GPUs), max over ranks.
e2e = the same metric through the public API (planning included) with the
shard starting in the pinned O(1) host cache: ``mem0 -> gpu0`` + NVLink fan-out
to every other GPU, host->device bytes inside the timed region, per-layer
stamps read back to the host.  At N >= 2 the host-fed group loads striped: every
member stages its piece of each layer over its own PCIe link from the one shared
host copy and forwards it over NVLink (``--no-stripe``: the rep's link only).

Beside the headline line (rank 0, same run):
  c3            -- the C3 burst trace replayed through ``simcore`` with the
                   reference's analytic costs and with costs measured here
                   (prefill line, decode line, layer arrivals, host-cache load);
  coop_c1       -- C1: ZigZag prefill while the new slab streams in, then
                   cooperative decode (graph-captured), logits vs the fp32 oracle;
  live_pair     -- N >= 2: two-process ZigZag on 7B while the slab crosses NVLink,
                   then the KV hand-over and the new instance decoding alone;
  ramp          -- N >= 2: pair throughput vs layers resident on the new instance, against
                   the reference's steady_state_throughput;
  c3_realclock  -- N >= 2: the burst served on the wall clock by real 7B prefills on
                   GPUs 0..N-1 (static / AllCache / live-host / NVLink chain scale-up);
  decisions     -- the planner / pipeline / replay calls vs the reference's timings.

``--impl reference`` times the reference's CPU path: the oracle's torch CPU
copies of every layer unit along the same plan (all host threads), rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# stdout carries exactly one JSON line (_emit); main() moves fd 1 onto stderr so
# native libraries' own stdout writes (NCCL's "NCCL version" banner under
# NCCL_DEBUG=WARN/VERSION) cannot land in front of it
_JSON_OUT = sys.stdout


def _emit(line: dict) -> None:
    print(json.dumps(line), file=_JSON_OUT, flush=True)


def _ncu_metrics(name: str) -> dict:
    """{metric: value} of the first kernel in a committed ncu --csv launch list (long format)."""
    import csv
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
    out = {}
    with open(path, newline="") as f:
        rows = [r for r in csv.reader(f) if len(r) >= 15 and r[0] != "ID"]
    for r in rows:
        if r[0] == rows[0][0]:
            out[r[12]] = float(r[14].replace(",", ""))
    return out


def _push_traffic(payload: int):
    """Per-launch DRAM traffic of the dominant mover (k_push_tiles on the sending GPU)
    and its NVLink wire bytes, from the committed single-process 2-GPU ncu capture
    of one 2 GB hop (profiles/r2_ncu_nvlink_push_n2.csv), scaled to this shard."""
    try:
        m = _ncu_metrics("r2_ncu_nvlink_push_n2.csv")
        user = m["nvltx__bytes_data_user.sum"]
        scale = payload / user
        return {"traffic": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) * scale,
                "traffic_source": "ncu, k_push_tiles<0> gpu0->gpu1 hop of 2.0 GB (profiles/r2_ncu_nvlink_push_n2.csv): "
                                  "sender DRAM read+write, scaled to this shard",
                "nvlink_wire_per_user_byte": m["nvltx__bytes.sum"] / user,
                "ncu_nvlink_user_GBps": user / m["gpu__time_duration.sum"],
                "ncu_nvlink_wire_GBps": m["nvltx__bytes.sum"] / m["gpu__time_duration.sum"]}
    except (OSError, KeyError, IndexError, ValueError):
        return {"traffic": None, "traffic_source": None}


def _pull_traffic(payload: int):
    """The same for a pulled hop: the receiver's pull kernel reading the sender's slab
    over NVLink (single-process 2-GPU ncu capture of one 2 GB hop on the receiving GPU,
    profiles/r2_ncu_nvlink_pull_n2.csv), scaled to this shard."""
    try:
        m = _ncu_metrics("r2_ncu_nvlink_pull_n2.csv")
        user = m["nvlrx__bytes_data_user.sum"]
        scale = payload / user
        return {"traffic": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) * scale,
                "traffic_source": "ncu, the pull kernel on gpu1 reading a 2.0 GB hop from gpu0 "
                                  "(profiles/r2_ncu_nvlink_pull_n2.csv): receiver DRAM read+write, scaled",
                "nvlink_wire_per_user_byte": m["nvlrx__bytes.sum"] / user,
                "ncu_nvlink_user_GBps": user / m["gpu__time_duration.sum"],
                "ncu_nvlink_wire_GBps": m["nvlrx__bytes.sum"] / m["gpu__time_duration.sum"]}
    except (OSError, KeyError, IndexError, ValueError, ZeroDivisionError):
        return {"traffic": None, "traffic_source": None}


def _hbm_peak() -> float:
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6545.6


NVLINK_PEAK_GBPS = 770.0     # B200_PROFILING.md: measured peer copy per direction (900 nominal)
NVLINK_NOMINAL_GBPS = 900.0
PCIE_PEAK_GBPS = 63.0        # PCIe Gen5 x16 per direction, nominal
METRIC = "scale-up delivered GB/s (Llama-2 7B bf16 shard into every new B200)"
_T0 = time.perf_counter()


def log(msg: str) -> None:
    print(f"[bench r{os.environ.get('RANK', '0')} +{time.perf_counter() - _T0:7.1f}s] {msg}",
          file=sys.stderr, flush=True)


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="blitz", choices=["blitz", "reference"])
    p.add_argument("--arch", default="llama2-7b")
    p.add_argument("--tp", type=int, default=1, help="GPUs per instance (C4: 13B TP=2, C5: 70B TP=4)")
    p.add_argument("--tile-kib", type=int, default=1024)
    p.add_argument("--nctas", type=int, default=48)
    p.add_argument("--engine", default="auto", choices=["auto", "vector", "vec256", "tma", "ce", "ce2"],
                   help="auto: a source->leaf hop pulled by the receiver's SMs, relay chains on the copy "
                        "engines; ce2: every single-destination hop on the copy engines; "
                        "vector/vec256/tma: the sender's SMs push")
    p.add_argument("--fanout", default="auto", choices=["auto", "nvls", "chain", "star"])
    p.add_argument("--ce2-tiles", type=int, default=0,
                   help="tiles per copy-engine memcpy (0: 256 along an auto relay chain, 128 for ce2)")
    p.add_argument("--no-group", action="store_true", help="plan chains instead of NVLink fan-out")
    p.add_argument("--stage-engine", default="ce", choices=["ce", "sm"])
    p.add_argument("--tiles-per-copy", type=int, default=128,
                   help="tiles per copy-engine memcpy (128 x 1 MiB measured best: 54.8 GB/s)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-stripe", action="store_true",
                   help="host-cache loads over the rep's PCIe link only (no striping over its NVLink group)")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (sweeps only)")
    p.add_argument("--no-c3", action="store_true", help="skip the C3 serving replay")
    p.add_argument("--no-coop", action="store_true", help="skip the C1 cooperative-execution block")
    p.add_argument("--no-live", action="store_true", help="skip the two-GPU live-pair block")
    p.add_argument("--no-realclock", action="store_true",
                   help="skip the real-clock C3 burst on GPUs 0..N-1 (N >= 2)")
    p.add_argument("--live-engine", default="ce", choices=["vector", "ce", "pull"],
                   help="weight hop of the two-GPU live pair (ce: copy engines, no SM on either GPU; "
                        "pull: the target's SMs, which also run its share of the batches)")
    p.add_argument("--live-nctas", type=int, default=48)
    p.add_argument("--live-ce-tiles", type=int, default=128, help="tiles per copy-engine memcpy (--live-engine ce)")
    p.add_argument("--live-repeats", type=int, default=5, help="ZigZag / best-effort runs each (alternating)")
    p.add_argument("--extras", action="store_true",
                   help="at N > 4 also run the live-pair / ramp / real-clock / C3 / C1 blocks")
    p.add_argument("--cpu-sample-units", type=int, default=4)
    p.add_argument("--watchdog-s", type=int, default=900)
    return p.parse_args()


# ---- clocks ------------------------------------------------------------------------------


class ClockSampler:
    """SM clocks + throttle reasons sampled every 10 ms during the timed region.

    NVML (``nvidia_ml_py``) in a thread: the N >= 2 timed regions last ~100 ms, shorter
    than nvidia-smi's start-up, so a polling nvidia-smi often saw none of them.  One
    sample is taken at ``start()`` and one at ``stop()`` so the region always has two.
    nvidia-smi ``-lms 200`` remains the fallback when NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    REASON_BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
                   ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self.samples: list[tuple[float, float, int]] = []   # (sm MHz, max sm MHz, reason bits)
        self.proc = None
        self.nvml = None
        self.handle = None
        self.done = threading.Event()
        self.thread = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.device)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
        return pynvml, h

    def _sample(self):
        n, h = self.nvml, self.handle
        self.samples.append((float(n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)),
                             float(n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)),
                             int(n.nvmlDeviceGetCurrentClocksEventReasons(h))))

    def _poll(self):
        while not self.done.wait(0.01):
            self._sample()

    def start(self):
        try:
            self.nvml, self.handle = self._nvml_handle()
            self._sample()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.nvml is not None:
            self.done.set()
            self.thread.join(timeout=2)
            self._sample()
            sm = [x[0] for x in self.samples]
            reasons = {name for _, _, bits in self.samples for name, b in self.REASON_BITS if bits & b}
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(x[1] for x in self.samples),
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, 10 ms"}
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for name, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi -lms 200"}


# ---- distributed helpers ---------------------------------------------------------------------


def dist_max(values: list[float], world: int) -> list[float]:
    if world == 1:
        return values
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().tolist()


def dist_sum(value: float, world: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t)
    return float(t.item())


# ---- CPU baseline (the oracle restatement; bounded sample) ----------------------------------------


def cpu_copy_baseline(plan, layout, units: int, steps: int = 1) -> dict:
    """Torch CPU copies of the first ``units`` layer units along ``plan`` (all threads)."""
    import torch
    from oracle import dataplane_ref as ref

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    units = max(1, min(units, layout.num_layers))
    nbytes = layout.unit_off[units - 1] + layout.unit_bytes[units - 1]
    nodes = {e.src for e in plan.edges} | set(plan.targets())
    src_nodes = {e.src for e in plan.edges} - set(plan.targets())
    bufs = {}
    seed_buf = torch.from_numpy(ref.random_words((nbytes + 15) // 16 * 16, 5)[:nbytes].copy())
    for n in nodes:
        bufs[n] = seed_buf.clone() if n in src_nodes else torch.empty(nbytes, dtype=torch.uint8)
    bounds = [(layout.unit_off[k], layout.unit_off[k] + layout.unit_bytes[k]) for k in range(units)]
    ref.execute_plan_cpu(plan, bufs, bounds)  # warm (page faults)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        ref.execute_plan_cpu(plan, bufs, bounds)
        times.append(time.perf_counter() - t0)
    for n in plan.targets():
        assert torch.equal(bufs[n], seed_buf), "CPU baseline copy mismatch"
    delivered = sum(layout.unit_bytes[:units]) * len(plan.targets())
    secs = min(times)
    return {"value": delivered / secs / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"layer units 1..{units} of the shard ({delivered / 1e9:.2f} GB delivered "
                      f"to {len(plan.targets())} destination buffer(s)), torch CPU copy_ along "
                      f"the plan edges, best of {steps}",
            "seconds": secs}


# ---- decision path (our API) next to the reference's timings ------------------------------------


def decision_timings() -> dict:
    """SURVEY.md §8(d) item 1 on our API (single thread), with the reference's own
    timings of the same calls (tests/golden/reference_timings.json, measured in the
    build container by oracle/gen_golden.py -- the reference cannot run on the box)."""
    import paper_2412_17246_b200 as ss
    from paper_2412_17246_b200 import simcore
    from paper_2412_17246_b200.slab import LLAMA2_7B, model_spec_for

    model = model_spec_for(LLAMA2_7B)
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    topo2 = ss.load_topology("b200-hgx-2x8")
    trace = ss.generate_trace("burst", {"rate_per_s": 20, "duration_s": 30, "prompt_tokens": [512, 2048],
                                        "output_tokens": [16, 128],
                                        "bursts": [{"start_s": 10, "duration_s": 2, "multiplier": 5}]}, 1)

    def plan_1to8():
        req = ss.build_scale_request(model, ["gpu0"], [f"gpu{i}" for i in range(1, 8)], topo, flows)
        ss.estimate_completion(ss.generate_plan(req, topo, flows), model, topo, eta=1.0)

    def pipeline(n, L):
        return lambda: ss.zigzag_schedule(ss.configure_pipeline(n, L, 1.0))

    work = {
        "plan+estimate 1->8 (a1,a4,a6)": plan_1to8,
        "configure_pipeline+zigzag N=16 L=32 time_l=1 (a17,a19)": pipeline(16, 32),
        "configure_pipeline+zigzag N=16 L=80 time_l=1 (a17,a19)": pipeline(16, 80),
        "run_simulation C3 730 req blitz-live (b200 2x8)":
            lambda: simcore.run_simulation(topo2, [model], trace, simcore.SimPolicy("blitz-live")),
    }
    ref_path = ROOT / "tests" / "golden" / "reference_timings.json"
    ref_doc = json.loads(ref_path.read_text()) if ref_path.exists() else {}
    ref, ours_there = ref_doc.get("seconds", {}), ref_doc.get("ours_seconds", {})
    out = {}
    for name, fn in work.items():
        best = float("inf")
        for _ in range(5):
            t0 = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t0)
        out[name] = {"ours_ms": best * 1e3,
                     "reference_ms": ref[name] * 1e3 if name in ref else None,
                     "ours_ms_same_cpu_as_reference": ours_there[name] * 1e3 if name in ours_there else None}
    return {"calls": out, "ours_timed_on": f"this host, 1 thread, best of 5 ({os.cpu_count()} cores visible)",
            "reference_timed_on": "the build container by oracle/gen_golden.py --timings-only (the reference "
                                  "package is not installed on the GPU box), 1 thread, best of 5, together "
                                  "with ours on the same CPU (ours_ms_same_cpu_as_reference)"}


# ---- C3 on the real clock -------------------------------------------------------------------------


def c3_realclock(arch, n_gpus: int = 2, rate: float = 30.0, duration: float = 9.0) -> dict:
    """The C3 burst (5x for 2 s) served on the wall clock by real prefills: the source
    instance on GPU 0, new instances on GPUs 1..n_gpus-1 added as the reference
    trigger asks; strategies static / allcache (host-cache loads) / live-host /
    blitz (NVLink chain push).  TTFT pass: prefill instances only (the P/D split of
    the paper).  Decode pass (half the rate, so colocated decoding keeps up): every
    instance also decodes its requests' output tokens in a 32-slot continuous batch
    -- p50 / p99 TBT on the wall clock."""
    import paper_2412_17246_b200 as ss
    from paper_2412_17246_b200.realclock import RealClockServer

    def burst(r):
        return ss.generate_trace("burst", {"rate_per_s": r, "duration_s": duration,
                                           "prompt_tokens": [512, 2048], "output_tokens": [16, 128],
                                           "bursts": [{"start_s": duration / 3, "duration_s": 2, "multiplier": 5}]},
                                 seed=1)

    trace = burst(rate)
    arrivals = [(r.arrival_ms / 1e3, r.prompt_tokens) for r in trace]
    srv = RealClockServer(arch, extra_devs=list(range(2, n_gpus)), decode_slots=32, max_new_tokens=128)
    try:
        mean_tok = sum(a[1] for a in arrivals) / len(arrivals)
        pre_ms = sum(srv.prefill_ms(a[1], iters=2) for a in arrivals[:64]) / min(64, len(arrivals))
        capacity = mean_tok / (pre_ms / 1e3)
        keys = ("p50_ttft_ms", "p99_ttft_ms", "mean_ttft_ms", "scale_trigger_s", "scale_ready_s", "load_ms",
                "served", "instances_added", "all_ready_s")
        out = {"trace": f"burst {rate:g} req/s x {duration:g} s, 5x for 2 s at t={duration / 3:g} s, seed 1 "
                        f"({len(arrivals)} requests, mean prompt {mean_tok:.0f} tokens)",
               "served_by": "real prefills (one request each, prompts padded to 256-token buckets, CUDA graphs) "
                            f"on GPUs 0..{n_gpus - 1} (source on GPU 0), host wall clock; trigger = reference "
                            "should_scale_up on a 1 s arrival window vs the measured instance capacity",
               "instance_capacity_tok_s": capacity, "strategies": {}}
        for strat in ("static", "allcache", "live-host", "blitz"):
            r = srv.run(arrivals, strat, capacity)
            out["strategies"][strat] = {k: getattr(r, k) for k in keys}
        # decode pass: colocated continuous-batching decode of every request's output tokens
        dtrace = burst(rate / 2)
        darr = [(r.arrival_ms / 1e3, r.prompt_tokens, r.output_tokens) for r in dtrace]
        dec = {"trace": f"burst {rate / 2:g} req/s x {duration:g} s, 5x for 2 s, seed 1 ({len(darr)} requests, "
                        f"16-128 output tokens each)",
               "served_by": "each instance prefills and then decodes its requests in a 32-slot continuous batch "
                            "(per-row device positions, captured steps over 4/8/16/32 slots, alternating with "
                            "prefills); TBT = host-observed time between a request's tokens",
               "strategies": {}}
        for strat in ("static", "allcache", "blitz"):
            r = srv.run(darr, strat, capacity / 2)
            dec["strategies"][strat] = {k: getattr(r, k) for k in keys + ("p50_tbt_ms", "p99_tbt_ms", "decode_steps")}
        out["with_decode"] = dec
        return out
    finally:
        srv.close()


# ---- C1 cooperative execution (ZigZag) on this GPU vs the CPU fp32 oracle -----------------------


def single_gpu_host_arrivals(layout, device: int, seed: int = 241217, runs: int = 2) -> list:
    """Per-layer arrival times (ms) of one unstriped host-cache load into one GPU: the
    stop-the-world / host-fed load of ONE new instance (C3 scales one at a time, so
    it cannot stripe over sibling GPUs' PCIe links)."""
    import paper_2412_17246_b200 as ss
    from paper_2412_17246_b200.dataplane import DeviceSlab, Fabric, HostCache, ScaleExecutor

    slab = DeviceSlab(layout, device)
    slab.fill_random(seed)
    hc = HostCache(layout)
    hc.tensor.copy_(slab.data.cpu())
    plan = ss.ScalePlan(edges=[ss.planner.PlanEdge("mem0", "gpu0", 512.0, "pcie")], chains=[["mem0", "gpu0"]])
    ex = ScaleExecutor(Fabric(device), plan, slab, {"gpu0": 0}, host_cache=hc)
    best = None
    for _ in range(runs):
        ex.launch()
        ex.synchronize()
        arr = ex.layer_arrivals_ms()
        if best is None or arr[-1] < best[-1]:
            best = arr
    ex.close()
    slab.close()
    hc.close()
    return best


def coop_c1(device: int, n_batches: int = 8, seqs: int = 2, seq_len: int = 1000) -> dict:
    """C1: tiny 4-layer Llama (d=256) scaled 1->2 on one GPU.  The new instance's slab
    streams in from the pinned host cache (copy engines, per-layer publish) while the
    pair serves 8 x 2000-token prefill batches with the configure_pipeline split and
    the zigzag_schedule order; logits vs the fp32 CPU oracle; CPU oracle tokens/s."""
    import torch
    import paper_2412_17246_b200 as ss
    from paper_2412_17246_b200 import slab as S
    from paper_2412_17246_b200.coop import CooperativePair
    from paper_2412_17246_b200.dataplane import DeviceSlab, Fabric, HostCache, ScaleExecutor
    from paper_2412_17246_b200.llama import LlamaExecutor, SlabWeights
    from oracle.forward_ref import forward_fp32, weights_to_cpu_fp32

    arch = S.TINY_4L
    lay = S.SlabLayout.for_arch(arch, tile_bytes=256 * 1024)
    src = DeviceSlab(lay, device)
    w = SlabWeights(arch, lay, src.data)
    w.init_random(seed=0)
    hc = HostCache(lay)
    hc.tensor.copy_(src.data.cpu())
    tgt = DeviceSlab(lay, device)
    fabric = Fabric(device)
    plan = ss.ScalePlan(edges=[ss.planner.PlanEdge("mem0", "gpu0", 512.0, "pcie")],
                        chains=[["mem0", "gpu0"]])
    ex = ScaleExecutor(fabric, plan, tgt, {"gpu0": 0}, host_cache=hc)
    g = torch.Generator().manual_seed(3)
    batches = [torch.randint(0, arch.vocab, (seqs, seq_len), generator=g).to(f"cuda:{device}")
               for _ in range(n_batches)]
    source = LlamaExecutor(w, max_tokens=seqs * seq_len, device=f"cuda:{device}")
    target = LlamaExecutor(SlabWeights(arch, lay, tgt.data), max_tokens=seqs * seq_len,
                           device=f"cuda:{device}")
    # measured time_l = one unit's load time / one block's execution time
    ex.launch()
    ex.synchronize()
    load_ms = ex.layer_arrivals_ms()
    pos = torch.arange(seq_len, dtype=torch.int32, device=f"cuda:{device}").repeat(seqs)
    x = source.embed(batches[0])
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    source.block(0, x, pos, (seqs, seq_len))
    s0.record()
    for _ in range(5):
        source.block(0, x, pos, (seqs, seq_len))
    s1.record()
    s1.synchronize()
    block_ms = s0.elapsed_time(s1) / 5
    unit_ms = (load_ms[-1] - load_ms[0]) / max(1, arch.n_layers - 1) if arch.n_layers > 1 else load_ms[0]
    time_l = max(unit_ms, 1e-6) / block_ms
    cfg = ss.configure_pipeline(n_batches, arch.n_layers, time_l)
    tl = ss.zigzag_schedule(cfg)
    pair = CooperativePair(source, target, tgt.loaded)
    decode_steps = 8
    caches = pair.make_caches(batches, cfg, max_new_tokens=decode_steps)
    ex.launch()                       # untimed warm-up pass (first-use costs of every path)
    pair.run(batches, cfg, tl, caches=caches)
    ex.synchronize()
    ex.launch()                       # fresh transfer: layers arrive while the pair serves
    res = pair.run(batches, cfg, tl, caches=caches)
    ex.synchronize()
    # cooperative decode: same split, each side attends over its own KV blocks
    # (first step eager, the rest one captured two-stream graph per step)
    toks = [lg.argmax(-1) for lg in res.logits]
    gen = [[t] for t in toks]
    step = pair.decode(toks, cfg, caches)
    toks = [lg.argmax(-1) for lg in step.logits]
    for gl, t in zip(gen, toks):
        gl.append(t)
    graph = pair.decode_graph(toks, cfg, caches)
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record()
    for _ in range(decode_steps - 1):
        logits = graph(toks)
        toks = [lg.argmax(-1) for lg in logits]
        for gl, t in zip(gen, toks):
            gl.append(t)
    d1.record()
    d1.synchronize()
    dec_ms = d0.elapsed_time(d1)
    last_logits = [lg.clone() for lg in logits]
    tokens = n_batches * seqs * seq_len
    ref_w = weights_to_cpu_fp32(w)
    torch.set_num_threads(os.cpu_count() or 1)
    from oracle.logit_parity import ParityTally
    # every row of every batch: the prefill logits and the last decode step's (vs a full
    # fp32 recompute over prompt + generated tokens), against the fp32 oracle
    pre, dec = ParityTally(), ParityTally()
    cpu_s = None
    for b in range(n_batches):
        t0 = time.perf_counter()
        want = forward_fp32(arch, ref_w, batches[b].cpu())
        if cpu_s is None:
            cpu_s = time.perf_counter() - t0
        pre.add(res.logits[b], want)
        seq = torch.cat([batches[b].cpu()] + [t.cpu()[:, None] for t in gen[b][:-1]], 1)
        dec.add(last_logits[b], forward_fp32(arch, ref_w, seq))
    out = {"workload": f"C1 tiny-4l d=256, 1->2 on one GPU, {n_batches} x {seqs * seq_len}-token prefill "
                       f"batches served while the new slab streams from the pinned host cache",
           "time_l_measured": time_l, "splits": cfg.splits, "objective": cfg.objective(),
           "pair_ms": res.total_ms, "tokens_per_s": tokens / (res.total_ms / 1e3),
           "handoff_bytes": res.handoff_bytes, "max_rel_err_vs_fp32": pre.max_rel,
           "parity_prefill": pre.summary(), "parity_last_decode_step": dec.summary(),
           "greedy_equal_where_decisive": pre.mismatches == 0 and dec.mismatches == 0,
           "near_tie_rows": pre.ties + dec.ties, "rows": pre.rows + dec.rows,
           "decode": {"steps": decode_steps, "graph_steps_timed": decode_steps - 1, "ms": dec_ms,
                      "tokens_per_s": n_batches * seqs * (decode_steps - 1) / (dec_ms / 1e3),
                      "handoff_bytes_per_step": step.handoff_bytes,
                      "max_rel_err_vs_fp32_last_step": dec.max_rel},
           "cpu_fp32_oracle_tokens_per_s": seqs * seq_len / cpu_s,
           "cpu_cores": os.cpu_count()}
    ex.close()
    hc.close()
    tgt.close()
    src.close()
    return out


def block_cpu_vs_gpu(arch, prefill_ms: dict) -> dict:
    """One Llama block at 2048 tokens (4 x 512): the fp32 CPU oracle (all host threads)
    next to the measured B200 prefill line."""
    import torch
    from oracle.forward_ref import block_fp32

    torch.set_num_threads(os.cpu_count() or 1)
    g = torch.Generator().manual_seed(0)
    d, kv, f = arch.d_model, arch.kv_dim, arch.ffn
    w = {"attn_norm": torch.ones(d), "ffn_norm": torch.ones(d),
         "wqkv": torch.randn(d + 2 * kv, d, generator=g) * 0.02,
         "wo": torch.randn(d, d, generator=g) * 0.02,
         "wgu": torch.randn(2 * f, d, generator=g) * 0.02,
         "wdown": torch.randn(d, f, generator=g) * 0.02}
    x = torch.randn(4, 512, d, generator=g)
    block_fp32(arch, w, x[:, :64])  # warm
    t0 = time.perf_counter()
    block_fp32(arch, w, x)
    cpu_s = time.perf_counter() - t0
    gpu_block_ms = None
    if prefill_ms and 2048 in prefill_ms:
        gpu_block_ms = prefill_ms[2048] / arch.n_layers  # upper bound: includes head / L
    return {"tokens": 2048, "cpu_fp32_ms": cpu_s * 1e3, "cpu_threads": os.cpu_count(),
            "cpu_tokens_per_s": 2048 / cpu_s,
            "gpu_ms_per_block": gpu_block_ms,
            "gpu_tokens_per_s_per_block": 2048 / (gpu_block_ms / 1e3) if gpu_block_ms else None}


# ---- reference arm ------------------------------------------------------------------------------


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    from paper_2412_17246_b200 import slab as S
    from paper_2412_17246_b200.scaleup import plan_for

    arch = S.ARCHS[args.arch]
    layout = S.SlabLayout.for_arch(arch, tile_bytes=args.tile_kib * 1024)
    gpus = [f"gpu{i}" for i in range(world)]
    if world == 1:
        plan, _, _ = plan_for(arch, ["mem0"], ["gpu0"])
        workload = f"{arch.name} O(1) host-cache load mem0->gpu0 (CPU restatement)"
    else:
        plan, _, _ = plan_for(arch, ["gpu0"], gpus[1:], group=not args.no_group)
        workload = f"{arch.name} live scale-up 1->{world} (CPU restatement of the plan's copies)"
    for _ in range(args.warmup):
        cpu_copy_baseline(plan, layout, args.cpu_sample_units, steps=1)
    t0 = time.perf_counter()
    res = cpu_copy_baseline(plan, layout, args.cpu_sample_units, steps=args.steps)
    wall = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["seconds"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload, "sample_units": args.cpu_sample_units},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    _emit(line)


# ---- our arm ----------------------------------------------------------------------------------------


def run_blitz(args):
    import torch
    from paper_2412_17246_b200 import slab as S
    from paper_2412_17246_b200.dataplane import DeviceSlab, Fabric, host_fed_groups, plan_roles
    from paper_2412_17246_b200.scaleup import ScaleUpSession, plan_for, plan_host_cache, rank_plan

    fabric = Fabric.from_env()
    N, rank = fabric.world, fabric.rank
    arch = S.ARCHS[args.arch]
    tp = args.tp
    if N % tp:
        raise SystemExit(f"--tp {tp} must divide the GPU count {N}")
    layout = S.SlabLayout.for_arch(arch, tp=tp, tile_bytes=args.tile_kib * 1024)
    payload = layout.payload_bytes()
    gpus = [f"gpu{i}" for i in range(N)]
    anchors = gpus[::tp]  # InstanceState.node = gpus[0] (simcore.py:142-144)
    node_rank = {g: i for i, g in enumerate(gpus)}
    engine = {"tma": 1, "vec256": 2, "ce": 3, "auto": 4, "ce2": 5}.get(args.engine, 0)
    seed = 241217
    my = gpus[rank]

    def fill_random(host: torch.Tensor):
        tmp = DeviceSlab(layout, fabric.device)
        tmp.fill_random(seed)
        host.copy_(tmp.data.cpu())
        tmp.close()

    def host_cache_for(plan, tag):
        """Pinned O(1) host copy (one /dev/shm region per host-fed group), mapped by the
        ranks that stage from it: the rep, and its NVLink siblings when striped."""
        return plan_host_cache(fabric, layout, plan, node_rank, fill_random,
                               host_stripe=not args.no_stripe, tag=tag)

    if len(anchors) == 1:
        anchor_plan, model, est = plan_for(arch, ["mem0"], anchors, tp=tp)
        workload = (f"{arch.name} bf16 TP={tp} O(1) pinned host-cache load mem0->{anchors} "
                    f"(copy engines), per-layer readiness")
        bound, peak, peak_src = "pcie", PCIE_PEAK_GBPS, "PCIe Gen5 x16 nominal per direction"
    else:
        anchor_plan, model, est = plan_for(arch, ["gpu0"], anchors[1:], group=not args.no_group, tp=tp)
        workload = (f"{arch.name} bf16 TP={tp} live scale-up 1->{len(anchors)} instances: anchor plan "
                    f"{[(e.src, e.dst) for e in anchor_plan.edges]} fan-out {anchor_plan.nvlink_fanout}")
        bound, peak, peak_src = "nvlink", NVLINK_PEAK_GBPS, "B200_PROFILING.md measured peer copy per direction (900 nominal)"
    plan = rank_plan(anchor_plan, tp)
    receivers = len(plan.targets())
    delivered = payload * receivers
    log(f"plan ready: {[(e.src, e.dst) for e in plan.edges]} fanout {plan.nvlink_fanout}")
    hc = host_cache_for(plan, "value")
    log("host cache ready" if hc is not None else "no host cache on this rank")
    sess = ScaleUpSession(fabric, layout, plan, node_rank, host_cache=hc, engine=engine,
                          nctas=args.nctas, fanout_mode=args.fanout, seed=seed,
                          stage_engine=args.stage_engine, tiles_per_copy=args.tiles_per_copy,
                          ce_tiles_per_copy=args.ce2_tiles,
                          host_stripe=not args.no_stripe)

    log("session ready")
    # warm-up (first one verified bit-exact on every receiver)
    ok = True
    for w in range(max(args.warmup, 1)):
        r = sess.run(verify=(w == 0))
        if w == 0:
            ok = bool(r.verified)
    ok_all = dist_sum(0.0 if ok else 1.0, N) == 0.0
    log(f"warm-up done, verified={ok_all}")

    # the achievable PCIe rate on this box: a plain pinned H2D copy (torch, copy
    # engine) of 4 GiB of the same host cache, measured live as the roofline peak
    h2d_ceiling = None
    if bound == "pcie" and hc is not None:
        n = min(4 << 30, hc.tensor.numel())
        scratch = torch.empty(n, dtype=torch.uint8, device=f"cuda:{fabric.device}")
        cs = torch.cuda.Stream(device=fabric.device)
        best = 0.0
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs):
                e0.record(cs)
                scratch.copy_(hc.tensor[:n], non_blocking=True)
                e1.record(cs)
            e1.synchronize()
            best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        del scratch
        h2d_ceiling = best   # secondary denominator; the primary stays PCIe Gen5 x16 nominal
        log(f"h2d ceiling {best:.1f} GB/s")

    clocks = ClockSampler(fabric.device)
    fabric.barrier()
    torch.cuda.synchronize()
    clocks.start()
    steps, kern, first_layer, last_layer = [], [], [], []
    layers_value, layers_host = None, None
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        r = sess.run(time_kernel=True)
        steps.append(r.elapsed_ms)
        kern.append(r.kernel_ms if r.kernel_ms is not None else 0.0)
        if r.layer_ms:
            first_layer.append(r.layer_ms[0])
            last_layer.append(r.layer_ms[-1])
            layers_value = r.layer_ms
    fabric.barrier()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    log(f"timed steps ms={steps} kernel_ms={kern}")
    step_ms = dist_max(steps, N)
    kern_ms = dist_max(kern, N)
    fl = dist_max([statistics.mean(first_layer) if first_layer else 0.0], N)[0]
    launches = dist_sum(float(sess.executor.kernels_per_launch() * args.steps), N)
    ms = statistics.mean(step_ms)
    value = delivered / (ms / 1e3) / 1e9
    dom_kernel_ms = statistics.mean(kern_ms)
    # dominant mover: bytes that cross the bound link per launch = one shard
    achieved = payload / (dom_kernel_ms / 1e3) / 1e9 if dom_kernel_ms > 0 else None
    final_ok = sess.verify(sess.executor.epoch)
    final_all = dist_sum(0.0 if final_ok else 1.0, N) == 0.0

    # ---- e2e: public API, shard starts in pinned host memory ---------------------------------
    e2e = None
    e2e_plan = None
    if not args.no_e2e:
        e2e_anchor, _, _ = plan_for(arch, ["mem0"], anchors, tp=tp)
        e2e_plan = rank_plan(e2e_anchor, tp)
    reuse = e2e_plan is not None and e2e_plan.edges == plan.edges and \
        e2e_plan.nvlink_fanout == plan.nvlink_fanout
    if not reuse:
        sess.close()
        if hc is not None:
            hc.close()
    if e2e_plan is not None:
        log(f"e2e plan {[(e.src, e.dst) for e in e2e_plan.edges]} fanout {e2e_plan.nvlink_fanout}"
            f"{' (same session as value)' if reuse else ''}")
        if reuse:
            hc2, sess2 = hc, sess
        else:
            hc2 = host_cache_for(e2e_plan, "e2e")
            sess2 = ScaleUpSession(fabric, layout, e2e_plan, node_rank, host_cache=hc2, engine=engine,
                                   nctas=args.nctas, fanout_mode=args.fanout, seed=seed,
                                   stage_engine=args.stage_engine, tiles_per_copy=args.tiles_per_copy,
                                   host_stripe=not args.no_stripe)
            for w in range(max(1, min(args.warmup, 2))):
                sess2.run(verify=(w == 0))
        e2e_t = []
        for _ in range(args.steps):
            fabric.barrier()
            t0 = time.perf_counter()
            # the user's call: plan (reference API) + execute + read readiness back
            p, _, _ = plan_for(arch, ["mem0"], anchors, tp=tp)
            p = rank_plan(p, tp)
            assert p.edges == e2e_plan.edges and p.nvlink_fanout == e2e_plan.nvlink_fanout
            r = sess2.run()
            stamps = sess2.slab.stamps.cpu()  # d2h: per-layer arrival stamps
            e2e_t.append(time.perf_counter() - t0)
            if r.layer_ms:
                layers_host = r.layer_ms
        e2e_s = dist_max(e2e_t, N)
        log(f"e2e steps s={e2e_t}")
        # per-GPU last-layer arrival of the last e2e step (host stage vs NVLink stage)
        last_layer = fabric.allgather((my, layers_host[-1] if layers_host else None))
        e2e_ok = dist_sum(0.0 if sess2.verify(sess2.executor.epoch) else 1.0, N) == 0.0
        h2d = payload * tp  # one shard per TP rank crosses PCIe per step
        d2h = int(stamps.numel() * 8) * N
        e2e = {"value": payload * len(e2e_plan.targets()) / statistics.mean(e2e_s) / 1e9,
               "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "workload": f"public API: plan_for(mem0 -> {anchors}, tp={tp}) + ScaleUpSession.run() + "
                           f"stamp readback; plan {[(e.src, e.dst, e.kind) for e in e2e_plan.edges]}"
                           f" fan-out {e2e_plan.nvlink_fanout}",
               "host_stripe": ({rep: len(m) for rep, m in sess2.executor.stripe_groups.items()} or None),
               "last_layer_ms_by_gpu": {n: t for n, t in last_layer if t is not None},
               "bit_exact": e2e_ok}
        sess2.close()
        if hc2 is not None:
            hc2.close()

    # ---- C3: serving replay of the 5x burst with the times measured above -------------------------
    c3 = None
    extras = N <= 4 or args.extras
    if not args.no_c3 and tp == 1 and extras:
        roles_v = plan_roles(plan)
        e2e_roles = plan_roles(e2e_plan) if e2e_plan is not None else {}
        striped = e2e_plan is not None and bool(host_fed_groups(e2e_plan)) and not args.no_stripe
        mine = {"node": my, "value": layers_value, "host": None if striped else layers_host,
                "value_parent": roles_v[my].parent if my in roles_v else None,
                "host_parent": e2e_roles[my].parent if my in e2e_roles else None}
        allm = fabric.allgather(mine)
        if rank == 0:
            nv = next((m["value"] for m in allm if m["value"] and m["value_parent"] == "gpu0"), None)
            host = next((m["host"] for m in allm if m["host"] and (m["host_parent"] or "").startswith("mem")),
                        None)
            if N == 1 and host is None:
                host = layers_value
            if host is None and striped:
                # the e2e load was striped over the group; C3 loads one instance at a time
                log("c3: unstriped single-GPU host load for the host-fed strategies")
                host = single_gpu_host_arrivals(layout, fabric.device)
            from paper_2412_17246_b200.calibrate import (build_costs, c3_report, measure_decode,
                                                         measure_prefill, measure_ssd_load)
            log("c3: measuring prefill and decode")
            pre = measure_prefill(arch, device=fabric.device)
            dec_runs = [measure_decode(arch, device=fabric.device) for _ in range(2)]
            dec = {b: min(r[b] for r in dec_runs) for b in dec_runs[0]}   # per-size best of two passes
            try:
                ssd = measure_ssd_load(device=fabric.device)
            except OSError as e:      # no O_DIRECT-capable scratch space: keep the model
                ssd = {"error": str(e)}
            costs = build_costs(prefill=pre, nvlink_layer_ms=nv, host_layer_ms=host, decode=dec,
                                ssd_gbs=ssd.get("ssd_to_gpu_GBps"),
                                source={"prefill_points_ms": pre, "decode_points_ms": dec,
                                        "decode_context_tokens": 1024, "ssd_probe": ssd,
                                        "measured_in": "this bench run"})
            exe = None
            if N >= 2:
                # the same replay with every network scale-up executed on GPUs 0..N-1 and its
                # layer / transfer events taken from device stamps (inprocess.ExecutedCosts)
                import dataclasses
                from paper_2412_17246_b200.inprocess import ExecutedCosts, LocalPlanExecutor
                exe = ExecutedCosts(LocalPlanExecutor(arch, list(range(N))),
                                    **{f.name: getattr(costs, f.name) for f in dataclasses.fields(costs)})
            c3 = c3_report(costs, executed=exe)
            if exe is not None:
                exe.executor.close()
            c3["block_7b_2048tok"] = block_cpu_vs_gpu(arch, pre)
            # a batch-1 decode step reads every weight once: HBM roofline of the decode GEMMs
            wbytes = arch.total_bytes() - arch.embed_bytes()
            c3["decode_b1_weight_GBps"] = wbytes / (dec[1] / 1e3) / 1e9
            c3["decode_b1_hbm_frac"] = c3["decode_b1_weight_GBps"] / _hbm_peak()
            log(f"c3 done: { {k: v['measured']['p99_ttft_ms'] for k, v in c3['strategies'].items()} }")

    # ---- live pair (N >= 2): ZigZag across two GPUs while the weights stream in ---------------
    # N > 4 (the scaling sweep's 8-GPU point): the headline transfer, e2e and CPU baseline
    # only -- the pair/ramp/real-clock blocks use GPUs 0..3 and are measured at N = 2, 4
    extras = N <= 4 or args.extras
    if not extras:
        log(f"N={N}: live pair / ramp / real-clock C3 / C3 replay / C1 skipped (measured at N <= 4; --extras runs them)")
    live = None
    if N >= 2 and tp == 1 and not args.no_live and extras:
        from paper_2412_17246_b200.livepair import LivePair, summarize
        log("live pair (7B, NVLink hop, ZigZag)")
        lp = LivePair(fabric, arch, n_batches=12, seqs=4, seq_len=500, mode="nvlink",
                      engine={"ce": 5, "vector": 0, "pull": 4}[args.live_engine], nctas=args.live_nctas,
                      repeats=args.live_repeats, ce_tiles_per_copy=args.live_ce_tiles)
        res = lp.run()
        live = summarize(res) if res is not None else None
        log("live pair: KV hand-over to the new instance, which then decodes alone")
        ho = lp.run_handover(lp.cfg, lp.tl)
        if live is not None:
            live["kv_handover"] = ho
        lp.close()
        if live is not None:
            log(f"live pair avg latency {live['avg_latency_ms']}")

    # ---- interference (N == 4): a measured KV flow in the FlowSet prunes the serving sender ----
    interference = None
    if N == 4 and tp == 1 and not args.no_live and extras:
        from paper_2412_17246_b200.interference import run_interference
        log("interference: measured KV flow gpu0 -> gpu1 vs scale-up of gpu2, gpu3")
        try:
            interference = run_interference(fabric, arch)
        except Exception as e:  # report, never sink the bench line
            interference = {"error": f"{type(e).__name__}: {e}"}

    # ---- measured pair-throughput ramp (N >= 2): the executed steady_state_throughput ----------
    ramp = None
    if rank == 0 and N >= 2 and tp == 1 and not args.no_live and extras:
        log("ramp: pair throughput vs layers resident on the new instance (GPUs 0, 1)")
        try:
            from paper_2412_17246_b200.ramp import measure_ramp
            ramp = measure_ramp(arch, batches=12, ks=[0, 4, 8, 12, 16] if arch.n_layers == 32 else None)
        except Exception as e:  # report, never sink the bench line
            ramp = {"error": f"{type(e).__name__}: {e}"}

    # ---- C3 on the real clock (N >= 2): a 5x burst served by real 7B prefills on GPUs 0
    # and 1, the scale-up triggered by the reference policy and executed by the data plane
    realclock = None
    if rank == 0 and N >= 2 and tp == 1 and not args.no_realclock and extras:
        log(f"c3 real clock (GPUs 0..{N - 1})")
        try:
            realclock = c3_realclock(arch, n_gpus=N)
            log(f"c3 real clock p99: { {k: round(v['p99_ttft_ms'], 1) for k, v in realclock['strategies'].items()} }")
        except Exception as e:  # report, never sink the bench line
            realclock = {"error": f"{type(e).__name__}: {e}"}
    fabric.barrier()

    decisions = decision_timings() if rank == 0 else None
    coop = None
    if rank == 0 and not args.no_coop and extras:
        log("c1 cooperative execution")
        coop = coop_c1(fabric.device)
        log(f"c1 done {coop['tokens_per_s']:.0f} tok/s rel_err {coop['max_rel_err_vs_fp32']:.2e}")

    cpu = None
    if rank == 0 and not args.no_cpu:
        log("cpu baseline")
        cpu = cpu_copy_baseline(plan, layout, args.cpu_sample_units, steps=1)
        log(f"cpu baseline {cpu['value']:.2f} GB/s")
        cpu.pop("seconds", None)

    if rank == 0:
        # DRAM traffic of the dominant kernel: the NVLink push kernel (N >= 2); at N=1 the
        # mover is the copy engine (no kernel, no ncu counter): null
        relays = bound == "nvlink" and any(plan_roles(plan)[n].receives and
                                           (plan_roles(plan)[n].children or plan_roles(plan)[n].fanout or
                                            plan_roles(plan)[n].rep is not None) for n in plan.targets())
        # auto pulls source -> leaf hops (the receiver's SMs) and pushes along relay chains
        pulled = bound == "nvlink" and args.engine == "auto" and not relays
        if bound != "nvlink":
            nvl = {"traffic": None, "traffic_source": None}
        else:
            nvl = _pull_traffic(payload) if pulled else _push_traffic(payload)
        traffic, traffic_src = nvl.pop("traffic"), nvl.pop("traffic_source")
        ce_chain = bound == "nvlink" and (args.engine in ("ce", "ce2") or (args.engine == "auto" and relays))
        if ce_chain:
            traffic, traffic_src = None, "copy-engine hops: no SM kernel, invisible to ncu"
            nvl = {}
        mover = ("copy engines (bz_stage_tiles_ce)" if bound == "pcie" else
                 "bz_pull_tiles: each receiver's SMs read the source's slab over NVLink" if pulled else
                 "k_multicast_tiles (NVLS multimem.st) fan-out" if sess.executor.fanout_mode == "nvls" else
                 "copy engines along the chain (bz_push_tiles_ce2 out of the source, bz_push_tiles_ce_gated "
                 "at each relay)" if ce_chain else f"k_push_tiles ({args.engine}) along the chain")
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": workload, "model": arch.name, "tp": tp, "shard_bytes": payload,
                       "receivers": receivers, "tile_bytes": args.tile_kib * 1024,
                       "ntiles": int(layout.ntiles), "nctas": args.nctas,
                       "engine": args.engine, "fanout": sess.executor.fanout_mode,
                       "stage_engine": args.stage_engine,
                       "l2": "inputs (13.48 GB shard) exceed the 126 MB L2; no flush needed",
                       "parallelism": f"1 process per GPU, {N} GPU(s)"},
            "scale_up_ms": ms, "per_dest_GBps": payload / (ms / 1e3) / 1e9,
            "first_layer_ms": fl,
            "modeled_ms_eta1": {k: v * 1e3 for k, v in est.per_target_completion.items()},
            "bit_exact": bool(ok_all and final_all),
            "roofline": {"bound": bound, "mover": mover, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         # one hop moves the shard once across NVLink (push: the sender reads its
                         # HBM and stores to the peer; pull: the receiver loads and writes its HBM)
                         "algorithmic_bytes_per_launch": payload if bound == "nvlink" else None,
                         **nvl,
                         "peak_source": peak_src, "kernel_ms": dom_kernel_ms,
                         "frac_of_nominal": (achieved / (NVLINK_NOMINAL_GBPS if bound == "nvlink"
                                                         else PCIE_PEAK_GBPS)) if achieved else None,
                         # the wire is the real bound: 900 GB/s nominal / the mover's wire bytes per
                         # payload byte from its ncu capture (pull 1.125, push 1.19) -- why a pulled
                         # hop can exceed the recipe's 770 GB/s copy-engine peer copy
                         "protocol_bound_GBps": (NVLINK_NOMINAL_GBPS / nvl["nvlink_wire_per_user_byte"])
                         if bound == "nvlink" and nvl.get("nvlink_wire_per_user_byte") else None,
                         "frac_of_protocol_bound": (achieved * nvl["nvlink_wire_per_user_byte"] / NVLINK_NOMINAL_GBPS)
                         if achieved and bound == "nvlink" and nvl.get("nvlink_wire_per_user_byte") else None,
                         # the box's achievable H2D rate (torch pinned 4 GiB copy, same host cache, this run)
                         "live_h2d_ceiling_GBps": h2d_ceiling,
                         "frac_of_live_h2d_ceiling": (achieved / h2d_ceiling) if (achieved and h2d_ceiling) else None},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "wall_s": wall, "c3": c3, "decisions": decisions, "coop_c1": coop,
            "live_pair": live, "ramp": ramp, "c3_realclock": realclock, "interference": interference,
        }
        _emit(line)
    fabric.barrier()


def main():
    args = parse_args()
    import faulthandler
    faulthandler.dump_traceback_later(args.watchdog_s, exit=True)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_blitz(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    main()
