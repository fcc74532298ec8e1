"""Decode and prefill entry points, executed on a B200.

Drop-in for ``moesim.pipeline`` (pipeline.py:44-851): same ``Strategy``,
``Timeline``, ``StrategyReport``, ``transfer_budget``, ``simulate_decoding``,
``simulate_prefill`` and ``compare_strategies`` signatures.  Where the
reference advances a discrete-event clock, these functions run the offload
engine: the fp64 gate and cross-layer predictor (K1), the device ARC (K2),
pinned host->HBM copies on a side stream, and the dequant-fused expert FFN
(K3 decode / K4 prefill).  Times in the returned Timeline/StrategyReport are
CUDA-event measurements; the timing-independent decisions (chosen experts,
prediction lists, prefetch/on-demand sets, ARC state) are bit-identical to
the reference's (tests/test_gpu_engine.py).

Extra keyword arguments (not in the reference): ``experts`` (an ExpertStore;
default: synthetic random-init experts for ``cfg``), ``shared_intermediate``
(shared expert width for the default store) and ``return_result`` (also
return the raw engine result with the expert outputs; ``return_result="logs"``
adds the per-step device logs, which cost a D2H copy and host parsing).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .cache import CachePlan, LayeredExpertCache, plan_allocation, zero_plan
from .core import GateTrace, ModelConfig, TimingModel, validate_trace_for
from .errors import InvalidConfig, TraceMismatch
from .predict import CrossLayerDecodePredictor, PrefetchPolicy
from .quant import QuantPolicy

STRATEGY_KINDS = ("fate", "eap", "lod")


@dataclass(frozen=True)
class Strategy:
    """Prefetch / quantization / ordering bundle (pipeline.py:44-104)."""

    kind: str
    prefetch_policy: PrefetchPolicy | None = None
    quant_policy: QuantPolicy | None = None
    reorder_prefill: bool = False
    charge_prediction: bool = False

    def __post_init__(self):
        if self.kind not in STRATEGY_KINDS:
            raise InvalidConfig(f"unknown strategy kind {self.kind!r}")
        if self.kind == "lod" and self.prefetch_policy is not None:
            raise InvalidConfig("lod carries no predictor")

    @classmethod
    def fate(cls, prefetch_policy=None, quant_policy=None, reorder_prefill: bool = True,
             charge_prediction: bool = False) -> "Strategy":
        # quant_policy=None means the default QuantPolicy, as in pipeline.py:78
        return cls("fate", prefetch_policy or PrefetchPolicy("percentile"),
                   quant_policy if quant_policy is not None else QuantPolicy(), reorder_prefill, charge_prediction)

    @classmethod
    def eap(cls, quant_policy=None) -> "Strategy":
        return cls("eap", PrefetchPolicy("topk"), quant_policy, False)

    @classmethod
    def lod(cls) -> "Strategy":
        return cls("lod")

    def prefetch_bits(self) -> int:
        return self.quant_policy.decode_bits if self.quant_policy else 16

    def ondemand_bits(self) -> int:
        return 2 if self.quant_policy else 16

    def cache_bits(self) -> int:
        return self.quant_policy.cache_bits if self.quant_policy else 16


@dataclass(frozen=True)
class TimelineEvent:
    start: float
    end: float
    resource: str
    label: str


@dataclass(frozen=True)
class Timeline:
    events: tuple
    stall_ms: float

    def compute_busy_ms(self) -> float:
        return sum(e.end - e.start for e in self.events if e.resource == "compute")

    def transfer_busy_ms(self) -> float:
        return sum(e.end - e.start for e in self.events if e.resource == "transfer")

    def check_exclusive(self) -> None:
        for res in ("compute", "transfer"):
            spans = sorted((e.start, e.end) for e in self.events if e.resource == res)
            for (s0, e0), (s1, _) in zip(spans, spans[1:]):
                assert s1 >= e0 - 1e-6, f"overlapping {res} events at {s1} < {e0}"


@dataclass(frozen=True)
class StrategyReport:
    strategy: str
    phase: str
    num_tokens: int
    total_ms: float
    ttft_ms: float | None
    tpot_ms: float | None
    tokens_per_s: float
    recall: float
    hit_rate: float
    stall_ms: float
    dequant_count: int
    cache_events: tuple = ()


def transfer_budget(timing: TimingModel, bits: int) -> int:
    """n = floor((t_moe + t_attn + t_gate) / t_expert_io[bits]) (pipeline.py:151-156)."""
    if bits not in timing.t_expert_io:
        raise InvalidConfig(f"no transfer time configured for {bits}-bit experts")
    return math.floor((timing.t_moe + timing.t_attn + timing.t_gate) / timing.t_expert_io[bits])


# ---------------------------------------------------------------------------
# engine plumbing

_STORES: dict = {}
_MAX_STORES = 2      # pinned host pools kept for reuse (each is GBs at model scale)
_MAX_IDLE = 2        # idle engines kept per (store, plan, gates)


def default_store(cfg: ModelConfig, bits, shared_intermediate: int = 0, seed: int = 0):
    """Synthetic random-init experts for cfg, cached per (cfg, bits, shared, seed);
    the least recently used store beyond _MAX_STORES is dropped (engines still
    holding it keep it alive until they close)."""
    from .experts import ExpertStore

    key = (cfg.num_layers, cfg.num_experts, cfg.hidden_dim, cfg.intermediate_dim, tuple(sorted(set(bits))),
           shared_intermediate, seed)
    if key in _STORES:
        _STORES[key] = _STORES.pop(key)  # most recently used last
    else:
        while len(_STORES) >= _MAX_STORES:
            _STORES.pop(next(iter(_STORES)))
        _STORES[key] = ExpertStore(cfg, bits=bits, seed=seed, shared_intermediate=shared_intermediate)
    return _STORES[key]


def release_pools() -> None:
    """Close every idle engine and drop the cached expert stores (their device
    slot pools and pinned host pools are freed once nothing references them)."""
    for engines in _IDLE.values():
        for e in engines:
            e.close()
    _IDLE.clear()
    _STORES.clear()


def knobs_for(strategy: Strategy, plan: CachePlan, n: int):
    from .engine import StrategyKnobs

    pol = strategy.prefetch_policy or PrefetchPolicy("topk")
    qp = strategy.quant_policy
    # a predictor exists only for fate / eap with a prefetch policy: build_decode_predictor
    # returns None otherwise (pipeline.py:330-331), and simulate_prefill's use_cross /
    # use_eap require the policy too (pipeline.py:563-564).  eap: co-activation
    # predictor in K1 (pipeline.py:301-321)
    predicts = strategy.kind in ("fate", "eap") and strategy.prefetch_policy is not None
    return StrategyKnobs(
        use_predictor=predicts, policy="eap" if strategy.kind == "eap" else pol.kind,
        percentile_q=pol.percentile_q, budget_n=n,
        cached_bits=plan.cached_bits, prefetch_bits=strategy.prefetch_bits(), ondemand_bits=strategy.ondemand_bits(),
        prefill_use_predictor=predicts, reorder_prefill=strategy.reorder_prefill,
        p_int2=qp.p_int2 if qp else 0.0, prefill_ondemand_bits=strategy.ondemand_bits() if strategy.kind == "fate" else 16)


def _bits_needed(strategy: Strategy, plan: CachePlan) -> tuple:
    b = {strategy.prefetch_bits(), strategy.ondemand_bits()}
    if strategy.kind == "fate" and strategy.quant_policy is not None:
        b |= {4, 2}
    if sum(plan.per_layer_capacity):
        b.add(plan.cached_bits)
    return tuple(sorted(b))


_IDLE: dict = {}


def _release(key, eng) -> None:
    pool = _IDLE.setdefault(key, [])
    pool.append(eng)
    while len(pool) > _MAX_IDLE:
        pool.pop(0).close()


def bind_engine(cache: LayeredExpertCache | None, plan: CachePlan, cfg: ModelConfig, weights, experts, knobs,
                max_tokens: int):
    """The engine of ``cache`` (created on first use), switched to ``knobs``.

    Engines are pooled per (expert store, plan, gate weights): a fresh
    LayeredExpertCache takes an idle engine, resets its device cache state
    (the reference's ``LayeredExpertCache(plan)``) and returns it to the pool
    when the cache object is garbage collected."""
    import weakref

    from .engine import OffloadEngine

    cache = cache if cache is not None else LayeredExpertCache(plan)
    if cache.engine is None:
        # an engine's slot stride fits the widest format its first strategy needed
        width = max(knobs.cached_bits, knobs.prefetch_bits, knobs.ondemand_bits, knobs.prefill_ondemand_bits)
        key = (id(experts), tuple(plan.per_layer_capacity), id(weights), width)
        idle = [e for e in _IDLE.get(key, []) if e.max_tokens >= max_tokens]
        if idle:
            eng = idle[0]
            _IDLE[key].remove(eng)
            eng.set_strategy(knobs)
            eng.reset_cache()
        else:
            eng = OffloadEngine(cfg, plan.per_layer_capacity, experts, weights, knobs,
                                max_tokens=max(max_tokens, 64))
        cache.bind(eng)
        weakref.finalize(cache, _release, key, eng)
    else:
        eng = cache.engine
        if eng.max_tokens < max_tokens:
            raise InvalidConfig(f"cache engine was built for {eng.max_tokens} tokens, need {max_tokens}")
        eng.set_strategy(knobs)
    return cache, eng


_NO_GATES: dict = {}


def _check_weights(weights, cfg: ModelConfig, strategy: Strategy):
    """The gate weights the engine routes with.  ``None`` is accepted where the
    reference accepts it -- no cross-layer predictor (LoD, EAP, or fate without a
    prefetch policy; pipeline.py:330-334, 570) -- and then stands for an all-zero
    router: every cache decision follows the trace's chosen sets (as in the
    reference, pipeline.py:422) and the expert outputs are combined with the
    uniform routing weight 1/E."""
    if weights is None:
        if strategy.kind == "fate" and strategy.prefetch_policy is not None:
            raise InvalidConfig("cross-layer prediction requires gate weights")
        key = (cfg.num_layers, cfg.num_experts, cfg.hidden_dim)
        if key not in _NO_GATES:
            from .gatesim import GateWeights
            z = np.zeros((cfg.num_experts, cfg.hidden_dim))
            _NO_GATES[key] = GateWeights(matrices=(z,) * cfg.num_layers, temperatures=(1.0,) * cfg.num_layers)
        return _NO_GATES[key]
    if weights.num_layers != cfg.num_layers or weights.matrices[0].shape != (cfg.num_experts, cfg.hidden_dim):
        raise InvalidConfig("gate weights do not match the model geometry")
    return weights


def _resident_counts(logs, caps, L):
    """Resident-set size at each step's decision time, replayed from the step logs."""
    res = [0] * L
    out = []
    for lg in logs:
        l = lg["layer"]
        out.append(res[l])
        inserted = 0 if caps[l] < 1 else sum(1 for e in lg["chosen"] if e not in lg["hits"])
        res[l] = min(caps[l], res[l] + inserted - len(lg["victims"]))
    return out


class RoutingMismatchWarning(UserWarning):
    """The device's fp64 router disagreed with a trace record's ``chosen`` set."""


def _warn_mismatch(stats: dict) -> None:
    # the engine follows record.chosen for every cache decision (pipeline.py:422), as
    # the reference does; a disagreement of the recomputed routing (imported real-model
    # traces, or near-ties) only affects the FFN routing weights, so it is reported
    n = int(stats.get("trace_mismatches", 0))
    if n:
        import warnings
        warnings.warn(f"{n} step(s): the recomputed top-k differs from the trace's chosen set; cache decisions "
                      "follow the trace", RoutingMismatchWarning, stacklevel=3)


def simulate_decoding(trace: GateTrace, strategy: Strategy, plan: CachePlan, timing: TimingModel, cfg: ModelConfig,
                      weights=None, cache: LayeredExpertCache | None = None, predictor=None,
                      collect_cache_events: bool = False, *, experts=None, shared_intermediate: int = 0,
                      return_result: bool = False, _eap_continue: bool = False, engine_tokens: int = 0,
                      dense=None, dense_ctx0: int = 0):
    """Execute decoding of ``trace`` on the GPU (pipeline.py:343-517 semantics).

    ``engine_tokens`` sizes a newly bound engine for at least that many tokens
    (compare_strategies passes the longer of its two traces, so a decode longer
    than the prefill that warmed the cache runs on the same engine).  ``dense``
    (``dense.DenseWeights``) executes the attention block and shared-expert gate in
    every step, token t at context position ``dense_ctx0`` + t.

    Strategy.eap() starts from empty co-activation statistics, as a fresh
    EapDecodePredictor does; compare_strategies passes ``_eap_continue`` so the
    decode continues with the statistics its prefill accumulated (pipeline.py:828-849)."""
    import torch

    if trace.phase != "decoding":
        raise TraceMismatch(f"decoding simulation given a {trace.phase} trace")
    validate_trace_for(trace, cfg)
    if predictor is not None and not isinstance(predictor, CrossLayerDecodePredictor):
        raise InvalidConfig("the B200 engine fuses the cross-layer predictor into its gate kernel; "
                            "custom host predictors are not supported")
    gates = _check_weights(weights, cfg, strategy)
    n = transfer_budget(timing, strategy.prefetch_bits())
    knobs = knobs_for(strategy, plan, n)
    if experts is None:
        experts = default_store(cfg, _bits_needed(strategy, plan), shared_intermediate)
    toks, g, ch = trace.dense_arrays(cfg)
    cache, eng = bind_engine(cache, plan, cfg, gates, experts, knobs, max_tokens=max(len(toks), engine_tokens, 1))
    if dense is not None:
        eng.set_dense(dense, max_ctx=dense_ctx0 + max(len(toks), engine_tokens, 1), ctx0=dense_ctx0)
    # every transfer and kernel in the timeline when the caller collects events (and
    # K3 waits for a step's copies on the stream, so its events are compute alone),
    # else sampled timing and the arrival-gated K3 (engine.OffloadEngine.set_overlap)
    eng.set_copy_timing(1 if collect_cache_events else 8)
    from .engine import overlap_default
    eng.set_overlap(not collect_cache_events and overlap_default())
    if strategy.kind == "eap" and not _eap_continue:
        eng.reset_eap()
    dev = torch.device("cuda", eng.device)
    res = eng.decode(torch.as_tensor(g, device=dev), torch.as_tensor(ch, device=dev), tokens=toks,
                     want_logs=collect_cache_events or return_result == "logs")
    st = res.stats
    if weights is not None:
        _warn_mismatch(st)
    L = cfg.num_layers
    events = []
    stall, timed_steps = 0.0, 0
    for s, (g0, g1, m0, m1) in enumerate(res.step_ms):
        if np.isnan(g1):
            continue  # sampled timing: this step carried no events
        timed_steps += 1
        t, l = toks[s // L], s % L
        events.append(TimelineEvent(g0, g1, "compute", f"gate t{t} L{l}"))
        events.append(TimelineEvent(m0, m1, "compute", f"moe t{t} L{l}"))
        stall += max(0.0, m0 - g1)
    # stall: the compute stream's waits between K1 and K3 (scaled from the timed
    # steps) plus, arrival-gated, the time K3 itself waited for copies
    stall = stall * (len(res.step_ms) / timed_steps if timed_steps else 0.0) + st.get("k3_wait_ms", 0.0)
    kinds = {0: "prefetch", 1: "ondemand"}
    for (c0, c1, kind, step, layer, expert, bits) in res.copies:
        if kind in kinds:
            events.append(TimelineEvent(c0, c1, "transfer", f"{kinds[kind]} t{toks[step] if step < len(toks) else step} "
                                                            f"L{layer} e{expert} {bits}b"))
    events.sort(key=lambda e: (e.start, e.resource, e.end, e.label))
    cache_events = ()
    if collect_cache_events:
        resident = _resident_counts(res.logs, plan.per_layer_capacity, L)
        evs = []
        for s, lg in enumerate(res.logs):
            for e in lg["chosen"]:
                hit = e in lg["hits"] or e in lg["arrived"]
                evs.append({"step": s, "layer": lg["layer"], "expert": e, "outcome": "hit" if hit else "miss",
                            "resident": resident[s]})
        cache_events = tuple(evs)
    total = st["gpu_ms"]
    T = len(toks)
    report = StrategyReport(
        strategy=strategy.kind, phase="decoding", num_tokens=T, total_ms=total, ttft_ms=None, tpot_ms=total / T,
        tokens_per_s=1000.0 * T / total if total > 0 else float("inf"),
        recall=st["recall_sum"] / st["recall_n"] if st["recall_n"] else 0.0,
        hit_rate=(st["cache_hits"] + st["arrival_hits"]) / st["accesses"] if st["accesses"] else 0.0,
        stall_ms=stall, dequant_count=int(st["dequant_count"]), cache_events=cache_events)
    timeline = Timeline(tuple(events), stall)
    if return_result:
        return timeline, report, res
    return timeline, report


def simulate_prefill(trace: GateTrace, strategy: Strategy, plan: CachePlan, timing: TimingModel, cfg: ModelConfig,
                     weights=None, cache: LayeredExpertCache | None = None, eap_stats=None, *, experts=None,
                     shared_intermediate: int = 0, return_result: bool = False, engine_tokens: int = 0):
    """Execute prompt processing of ``trace`` on the GPU (pipeline.py:536-778 semantics)."""
    import torch

    if trace.phase != "prefill":
        raise TraceMismatch(f"prefill simulation given a {trace.phase} trace")
    validate_trace_for(trace, cfg)
    if eap_stats is not None:
        raise InvalidConfig("the B200 engine keeps EAP statistics on the device; pass eap_stats=None "
                            "(compare_strategies shares them between prefill and decode)")
    gates = _check_weights(weights, cfg, strategy)
    n = transfer_budget(timing, strategy.prefetch_bits()) if strategy.prefetch_bits() in timing.t_expert_io else 0
    knobs = knobs_for(strategy, plan, n)
    if experts is None:
        experts = default_store(cfg, _bits_needed(strategy, plan), shared_intermediate)
    toks, g, ch = trace.dense_arrays(cfg)
    cache, eng = bind_engine(cache, plan, cfg, gates, experts, knobs, max_tokens=max(len(toks), engine_tokens, 1))
    if strategy.kind == "eap":
        eng.reset_eap()  # a fresh EapStats (pipeline.py:572-574)
    dev = torch.device("cuda", eng.device)
    Y, st, logs, step_ms, copies = eng.prefill(torch.as_tensor(g, device=dev), torch.as_tensor(ch, device=dev))
    if weights is not None:
        _warn_mismatch(st)
    events = []
    stall = 0.0
    for l, row in enumerate(step_ms):
        events.append(TimelineEvent(row[0], row[1], "compute", f"attn+gate L{l}"))
        events.append(TimelineEvent(row[2], row[3], "compute", f"experts L{l}"))
        stall += max(0.0, row[2] - row[1])
    kinds = {0: "prefetch", 1: "ondemand"}
    for (c0, c1, kind, step, layer, expert, bits) in copies:
        if kind in kinds:
            events.append(TimelineEvent(c0, c1, "transfer", f"{kinds[kind]} t0 L{layer} e{expert} {bits}b"))
    events.sort(key=lambda e: (e.start, e.resource, e.end, e.label))
    total = st["gpu_ms"]
    T = len(toks)
    report = StrategyReport(
        strategy=strategy.kind, phase="prefill", num_tokens=T, total_ms=total, ttft_ms=total, tpot_ms=None,
        tokens_per_s=1000.0 * T / total if total > 0 else float("inf"),
        recall=st["recall_sum"] / st["recall_n"] if st["recall_n"] else 0.0,
        hit_rate=(st["cache_hits"] + st["arrival_hits"]) / st["accesses"] if st["accesses"] else 0.0,
        stall_ms=stall, dequant_count=int(st["dequant_count"]))
    timeline = Timeline(tuple(events), stall)
    if return_result:
        return timeline, report, (Y, st, logs)
    return timeline, report


@dataclass(frozen=True)
class ComparisonRow:
    strategy: str
    phase: str
    budget_bytes: int
    report: StrategyReport
    timeline: Timeline


def shared_cache_bits(strategies: Sequence[Strategy]) -> int:
    for s in strategies:
        if s.quant_policy is not None:
            return s.quant_policy.cache_bits
    return 16


def compare_strategies(cfg: ModelConfig, timing: TimingModel, strategies: Sequence[Strategy], budgets: Sequence[int],
                       prefill_trace: GateTrace | None, decode_trace: GateTrace, weights=None, *, experts=None,
                       shared_intermediate: int = 0) -> list:
    """Every (strategy, budget) over the same traces; decode continues on the prefill-warmed
    cache (pipeline.py:802-851)."""
    if len(strategies) < 2:
        raise InvalidConfig("need at least two strategies to compare")
    if not budgets:
        raise InvalidConfig("need at least one memory budget")
    bits = shared_cache_bits(strategies)
    rows = []
    for budget in budgets:
        shared_plan = plan_allocation(cfg, budget, bits)
        for s in strategies:
            plan = zero_plan(cfg, budget) if s.kind == "lod" else shared_plan
            cache = LayeredExpertCache(plan)
            kw = dict(experts=experts, shared_intermediate=shared_intermediate,
                      engine_tokens=max(decode_trace.num_tokens,
                                        prefill_trace.num_tokens if prefill_trace is not None else 0))
            if prefill_trace is not None:
                tl, rep = simulate_prefill(prefill_trace, s, plan, timing, cfg, weights=weights, cache=cache, **kw)
                rows.append(ComparisonRow(s.kind, "prefill", budget, rep, tl))
            tl, rep = simulate_decoding(decode_trace, s, plan, timing, cfg, weights=weights, cache=cache,
                                        _eap_continue=s.kind == "eap" and prefill_trace is not None, **kw)
            rows.append(ComparisonRow(s.kind, "decoding", budget, rep, tl))
    return rows


def measure_timing_model(engine_result_stats: dict, cfg: ModelConfig, steps: int, copies, t_attn_ms: float = 0.01):
    """A TimingModel measured on this GPU: t_gate/t_moe from the per-step CUDA events,
    t_expert_io from the copy events per bit width, dequant fused (0), and t_attn from
    the dense part's events when the engine executed it (``OffloadEngine.set_dense``),
    else the caller's estimate."""
    io = {}
    for (c0, c1, kind, step, layer, expert, bits) in copies:
        if kind in (0, 1):
            io.setdefault(bits, []).append(c1 - c0)
    t_io = {b: float(np.median(v)) for b, v in io.items()}
    if engine_result_stats.get("dense_ms", 0.0) > 0:
        t_attn_ms = engine_result_stats["dense_ms"] / steps
    # K3's event time less the time it waited for copies (arrival-gated decode)
    t_moe = (engine_result_stats["ffn_ms"] - engine_result_stats.get("k3_wait_ms", 0.0)) / steps
    return TimingModel(t_moe=t_moe, t_attn=t_attn_ms,
                       t_gate=engine_result_stats["gate_ms"] / steps, t_expert_io=t_io, dequant_ms=0.0)
