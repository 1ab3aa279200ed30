"""Scaling side of the serving replay: the control loop and the hot-path callers.

``simcore.Simulation`` mixes this in.  It holds what the data plane replaces on
B200 -- the scale-up through the network (plan, scale flows, live pairs, the
per-layer and completion events of every new instance, simcore.py:676-750),
the layer / transfer events (simcore.py:752-795), the stop-the-world cache
loads (simcore.py:655-674) and the prefill->decode mutation
(simcore.py:628-653) -- plus the control tick that decides when to scale
(simcore.py:560-626).  Times come from the simulation's ``CostModel`` so the
same code replays the reference's analytic model or measured B200 costs.

Event push order and every tie-break follow the reference exactly: the replay
is checked value for value against it (tests/test_simcore_golden.py).
"""

from __future__ import annotations

from collections import deque

from .autoscaler import LoadMetrics, should_scale_up
from .livescale import (LayerLoaded, LiveScaleSession, LoadCompleted, LoadStarted, Phase, SloProfile,
                        mutate_prefill_to_decode, run_transition_protocol, select_live_pairs)
from .parampool import SourceRef
from .planner import build_scale_request, estimate_completion, generate_plan, plan_is_interference_free
from .topology import CapacityError

US_PER_MS = 1000
US_PER_S = 1_000_000

_STOP_THE_WORLD = ("sllm", "allcache")
_NETWORK = ("blitz-live", "blitz-stop")


def _plan_record(now_us: int, strategy: str, plan, est, live_targets, interference_free: bool) -> dict:
    """The ``plan`` scale event of the replay summary (simcore.py:740-750)."""
    rec = {"t_ms": now_us / US_PER_MS, "kind": "plan", "strategy": strategy}
    rec["edges"] = [(e.src, e.dst, round(e.gbps, 3)) for e in plan.edges]
    rec["chains"] = plan.chains
    rec["fanout"] = plan.nvlink_fanout
    rec["completion_s"] = {node: round(sec, 4) for node, sec in sorted(est.per_target_completion.items())}
    rec["live_targets"] = sorted(live_targets)
    rec["interference_free"] = interference_free
    return rec


class ScalingMixin:
    """Control tick, scale up / down, and the load events of new instances."""

    # ---- load signals -----------------------------------------------------------------------

    def _group(self, role: str) -> list:
        return [inst for inst in self.instances.values() if inst.status != "retired" and inst.role == role]

    def _window_rate(self, log: deque) -> float:
        """Tokens per second over the trailing load window (entries are (t_us, tokens))."""
        oldest = self.now_us - int(self.cfg.load_window_s * US_PER_S)
        while log and log[0][0] < oldest:
            log.popleft()
        return sum(tokens for _, tokens in log) / self.cfg.load_window_s

    def _kv_usage(self) -> float:
        decoders = [inst for inst in self.instances.values() if inst.role == "decode"]
        held = sum(r.prompt_tokens for inst in decoders for r in inst.active_decode)
        room = max(1.0, self.cfg.kv_capacity_tokens * max(1, len(self._group("decode"))))
        return min(1.0, held / room)

    # ---- control loop -----------------------------------------------------------------------

    def _on_control_tick(self, _):
        if self.policy.strategy != "static":
            for role, log in (("prefill", self._arrival_log), ("decode", self._decode_log)):
                self._scale_group(role, self._window_rate(log))
        if self._keep_ticking():
            self._push(self.now_us + int(self.cfg.control_interval_ms * US_PER_MS), "control")

    def _scale_group(self, role: str, load: float):
        members = self._group(role)
        metrics = LoadMetrics(window_s=self.cfg.load_window_s, tokens_per_s=load, kvcache_usage=self._kv_usage())
        grow = should_scale_up(metrics, self._policies[role], len(members))
        if grow > 0:
            self._execute_scale_up(role, grow)
        waiting = sum(len(m.queue) + len(m.active_decode) for m in members)
        shrink = self._down[role].observe(self.now_s, metrics, len(members), waiting)
        if shrink > 0:
            self._execute_scale_down(role, shrink)

    # ---- scale up -----------------------------------------------------------------------------

    def _execute_scale_up(self, role: str, count: int):
        strategy = self.policy.strategy
        self.counters["scale_ups"] += 1
        if role == "decode" and strategy in _NETWORK:
            # network strategies first flip idle prefill instances (zero-transfer)
            count = self._mutate_for_decode(count)
            if count <= 0:
                return
        model = self.models[self.default_model]
        fresh = []
        while len(fresh) < count:
            inst = self._allocate(model, role)
            if inst is None:
                break
            fresh.append(inst)
        if not fresh:
            return
        if strategy in _STOP_THE_WORLD:
            self._scale_stop_the_world(fresh, strategy)
        else:
            self._scale_via_network(fresh, live=(role == "prefill" and strategy == "blitz-live"))

    def _flippable(self) -> list:
        return [inst for inst in self._group("prefill")
                if inst.status == "active" and not inst.busy and not inst.queue
                and inst.live_session is None and inst.cooperating_with is None]

    def _mutate_for_decode(self, count: int) -> int:
        """Flip idle prefill instances (keeping one) to decode; every flip asks for
        compensating prefill capacity, scaled through the network.  Returns how many
        decode instances are still missing."""
        missing = count
        while missing > 0:
            spare = self._flippable()
            if len(spare) < 2:
                break
            inst = min(spare, key=lambda i: i.iid)
            flip = mutate_prefill_to_decode(inst)
            self.counters["mutations"] += 1
            self.scale_events.append({"t_ms": self.now_us / US_PER_MS, "kind": "mutate", "instance": inst.iid,
                                      "compensation": flip.compensation.count})
            missing -= 1
            model = self.models[inst.model_name]
            extra = [c for c in (self._allocate(model, "prefill") for _ in range(flip.compensation.count))
                     if c is not None]
            if extra:
                self._scale_via_network(extra, live=(self.policy.strategy == "blitz-live"))
        return missing

    def _load_s(self, strategy: str, model, inst) -> float:
        return self.costs.stop_the_world_s(strategy, model, self.topo, self.pool, inst.host_id, self.now_s,
                                           self.cfg.eta)

    def _scale_stop_the_world(self, fresh: list, strategy: str):
        """Cache baselines: each new instance loads whole before serving (simcore.py:655-674)."""
        model = self.models[self.default_model]
        issue_us = self.now_us + int(self.cfg.scale_cmd_latency_ms * US_PER_MS)
        for inst in fresh:
            if strategy == "sllm":
                hit = self.pool.cache_hit(model.name, inst.host_id, self.now_s)
                self.counters["cache_hits" if hit else "cache_misses"] += 1
            self._push(issue_us + int(round(self._load_s(strategy, model, inst) * US_PER_S)), "transfer",
                       (inst.iid, None))
        self.scale_events.append({"t_ms": self.now_us / US_PER_MS, "kind": strategy,
                                  "targets": [i.iid for i in fresh],
                                  "load_s": [round(self._load_s(strategy, model, i), 3) for i in fresh]})

    def _hold_scale_flows(self, plan) -> dict:
        """Register a scale flow on every plan edge at the bandwidth still free at
        both ends; returns dst -> the registered flow (released when it lands)."""
        held = {}
        for e in plan.edges:
            rate = min(self.topo.outcast_bandwidth(e.src, self.flows),
                       self.topo.incast_bandwidth(e.dst, self.flows), e.gbps)
            if rate <= 0:
                continue
            try:
                self.flows.register(e.src, e.dst, rate, "scale")
            except CapacityError:
                continue
            held[e.dst] = (e.src, e.dst, rate)
        return held

    def _start_live_pairs(self, plan, est, model, targets: dict, issue_us: int) -> set:
        """Pair overloaded prefill instances with new instances of the plan (busiest
        first) and schedule the new instance's per-layer arrivals."""
        candidates = [inst for inst in self._group("prefill")
                      if inst.status == "active" and inst.live_session is None and inst.cooperating_with is None]
        candidates.sort(key=lambda inst: (-inst.queued_tokens(), inst.iid))
        paired = set()
        for src_inst, node in select_live_pairs(plan, est, candidates, SloProfile(self.cfg.live_headroom_s)):
            new = targets.get(node)
            if new is None:
                continue
            session = LiveScaleSession(source_queue=src_inst.queue, target_queue=new.queue,
                                       total_layers=model.num_layers)
            run_transition_protocol(session, LoadStarted())
            new.live_session, src_inst.cooperating_with = session, new.iid
            paired.add(node)
            for k, t_k in enumerate(self.costs.layer_arrival_s(plan, node, model, self.cfg.eta), start=1):
                self._push(issue_us + int(round(t_k * US_PER_S)), "layer", (new.iid, k))
        return paired

    def _scale_via_network(self, fresh: list, live: bool):
        """The hot-path caller (simcore.py:676-750): plan from the live sources,
        hold its flows, pair for live execution, and schedule each new instance's
        completion."""
        model = self.models[self.default_model]
        sources = [ref.node for ref in self.pool.sources_for(model.name, self.now_s)]
        plan = generate_plan(build_scale_request(model, sources, [i.node for i in fresh], self.topo, self.flows),
                             self.topo, self.flows)
        est = estimate_completion(plan, model, self.topo, eta=self.cfg.eta)
        execute = getattr(self.costs, "on_plan", None)
        if execute is not None:
            # executed cost providers (inprocess.ExecutedCosts) move the plan's bytes now;
            # the layer / transfer events below then carry its device stamps
            execute(plan, model)
        self.counters["plans"] += 1
        self.counters["interference_free_plans"] += int(plan_is_interference_free(plan, self.flows, self.topo))
        issue_us = self.now_us + int(self.cfg.scale_cmd_latency_ms * US_PER_MS)
        targets = {inst.node: inst for inst in fresh}
        held = self._hold_scale_flows(plan)
        paired = self._start_live_pairs(plan, est, model, targets, issue_us) if live else set()
        for node, inst in targets.items():
            done_s = self.costs.completion_s(plan, est, node, model, self.cfg.eta)
            self._push(issue_us + int(round(done_s * US_PER_S)), "transfer", (inst.iid, held.get(node)))
        self.scale_events.append(_plan_record(self.now_us, self.policy.strategy, plan, est, paired,
                                              plan_is_interference_free(plan, self.flows, self.topo)))

    # ---- load events ----------------------------------------------------------------------------

    def _on_layer_loaded(self, payload):
        iid, k = payload
        inst = self.instances[iid]
        sess = inst.live_session
        if sess is None or inst.status == "retired" or sess.phase is Phase.FULL_SERVE:
            return
        if k <= sess.loaded_layers:
            return
        run_transition_protocol(sess, LayerLoaded(k))
        inst.loaded_layers = k
        if sess.phase is Phase.PARTIAL_SERVE:
            self._maybe_dispatch_prefill(inst)

    def _end_live_session(self, inst):
        """The new instance is complete: close its live session and release its
        cooperating source(s)."""
        sess = inst.live_session
        if sess.phase is Phase.LOADING:
            run_transition_protocol(sess, LayerLoaded(1))
        run_transition_protocol(sess, LoadCompleted())
        inst.live_session = None
        for other in self.instances.values():
            if other.cooperating_with == inst.iid:
                other.cooperating_with = None
                self._maybe_dispatch_prefill(other)

    def _on_transfer_done(self, payload):
        iid, flow = payload
        if flow is not None:
            try:
                self.flows.release(*flow, "scale")
            except KeyError:
                pass
            self._retry_pending_transfers()
        inst = self.instances[iid]
        if inst.status == "retired":
            return
        inst.status, inst.loaded_layers = "active", inst.total_layers
        if inst.live_session is not None:
            self._end_live_session(inst)
        self.pool.on_deploy(inst.model_name, SourceRef(inst.host_id, inst.gpus[0]), now_s=self.now_s)
        if self.policy.strategy == "sllm":
            self.pool.touch(inst.model_name, inst.host_id, self.now_s)
        (self._maybe_dispatch_prefill if inst.role == "prefill" else self._maybe_step_decode)(inst)

    # ---- scale down -----------------------------------------------------------------------------

    def _execute_scale_down(self, role: str, count: int):
        quiet = [inst for inst in self._group(role)
                 if inst.status == "active" and not (inst.busy or inst.stepping or inst.queue or inst.active_decode)
                 and inst.live_session is None and inst.cooperating_with is None]
        for inst in sorted(quiet, key=lambda i: -i.iid)[:count]:
            inst.status = "retired"
            self.counters["retired"] += 1
            pool = self.free_gpus[inst.host_id]
            pool.extend(inst.gpus)
            pool.sort()
            self.pool.on_reclaim(inst.model_name, SourceRef(inst.host_id, inst.gpus[0]), now_s=self.now_s)
            self.scale_events.append({"t_ms": self.now_us / US_PER_MS, "kind": "retire", "instance": inst.iid,
                                      "role": role})
