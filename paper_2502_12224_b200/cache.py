"""Memory-budget planning and the device-resident layered expert cache.

``plan_allocation`` / ``uniform_plan`` / ``zero_plan`` mirror cache.py:19-101
(integer arithmetic that sizes the slot pool).  ``LayeredExpertCache`` keeps
the reference's protocol (``contains``, ``layers[l].resident()``,
``layers[l].access()``, ``seed_resident``; cache.py:182-215) but its state —
ARC lists T1/T2/B1/B2, p, and the expert -> HBM buffer map — lives on the
GPU inside an ``OffloadEngine`` and is updated by kernel K2.  A cache is
bound to an engine the first time ``simulate_decoding`` / ``simulate_prefill``
runs with it; seeds issued before that are applied at binding time.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import Iterable, Sequence

from .core import ModelConfig
from .errors import BudgetTooSmall, InvalidConfig, NoAccesses


@dataclass(frozen=True)
class CachePlan:
    memory_budget: int
    cache_total: int
    per_layer_capacity: tuple
    cached_bits: int

    def bytes_used(self, cfg: ModelConfig) -> int:
        return cfg.dense_bytes + sum(self.per_layer_capacity) * cfg.expert_bytes[self.cached_bits]


def _slots_for_budget(cfg: ModelConfig, memory_budget: int, cached_bits: int) -> int:
    if cached_bits not in cfg.expert_bytes:
        raise InvalidConfig(f"no expert byte size configured for {cached_bits}-bit slots")
    if memory_budget < cfg.dense_bytes:
        raise BudgetTooSmall(f"memory budget {memory_budget} is below the dense footprint {cfg.dense_bytes}")
    return (memory_budget - cfg.dense_bytes) // cfg.expert_bytes[cached_bits]


def plan_allocation(cfg: ModelConfig, memory_budget: int, cached_bits: int = 16) -> CachePlan:
    """Fill layers below the shallow boundary first, split the rest evenly (cache.py:42-74)."""
    total = _slots_for_budget(cfg, memory_budget, cached_bits)
    Lb, E, n = cfg.shallow_boundary_L, cfg.num_experts, cfg.num_layers
    cap = [0] * n
    left = total
    for layer in range(min(Lb, n)):
        if left == 0:
            break
        cap[layer] = min(E, left)
        left -= cap[layer]
    deep = n - Lb
    if left > 0 and deep > 0:
        per = min(E, left // deep)
        spare = left - per * deep if per < E else 0
        for layer in range(Lb, n):
            cap[layer] = per + (1 if layer - Lb < spare else 0)
    return CachePlan(memory_budget, total, tuple(cap), cached_bits)


def uniform_plan(cfg: ModelConfig, memory_budget: int, cached_bits: int = 16) -> CachePlan:
    total = _slots_for_budget(cfg, memory_budget, cached_bits)
    n, E = cfg.num_layers, cfg.num_experts
    per = min(E, total // n)
    spare = total - per * n if per < E else 0
    return CachePlan(memory_budget, total, tuple(per + (1 if l < spare else 0) for l in range(n)), cached_bits)


def zero_plan(cfg: ModelConfig, memory_budget: int = 0) -> CachePlan:
    return CachePlan(memory_budget, 0, (0,) * cfg.num_layers, 16)


class _LayerView:
    """``cache.layers[l]``: the ArcState-like view of one layer on the device."""

    def __init__(self, cache: "LayeredExpertCache", layer: int):
        # a proxy, not a reference: the cache must die by refcount so its
        # pooled engine returns to the pool promptly (pipeline.bind_engine)
        self._c, self.layer = weakref.proxy(cache), layer

    @property
    def capacity(self) -> int:
        return self._c.plan.per_layer_capacity[self.layer]

    def _state(self) -> dict:
        return self._c.engine.arc_state(self.layer)

    @property
    def t1(self):
        return self._state()["t1"]

    @property
    def t2(self):
        return self._state()["t2"]

    @property
    def b1(self):
        return self._state()["b1"]

    @property
    def b2(self):
        return self._state()["b2"]

    @property
    def p_arc(self) -> float:
        return self._state()["p"]

    def resident(self) -> set:
        if self._c.engine is None:
            return set(self._c._pending_seeds.get(self.layer, []))
        return self._c.engine.resident(self.layer)

    def access(self, expert: int) -> bool:
        return self._c._engine_or_raise().access(self.layer, [int(expert)])[0]

    def check_invariants(self) -> None:
        """ArcState.check_invariants (cache.py:118-126) on the device state, plus
        the engine's own invariant: the experts holding a buffer are exactly T1 u T2."""
        st = self._state()
        c = self.capacity
        lists = [st["t1"], st["t2"], st["b1"], st["b2"]]
        total = sum(len(l) for l in lists)
        assert len(st["t1"]) + len(st["t2"]) <= c
        assert len(st["t1"]) + len(st["b1"]) <= c
        assert total <= 2 * c
        assert len(set().union(*map(set, lists))) == total, "ARC lists must be disjoint"
        assert 0.0 <= st["p"] <= c
        assert self._c.engine.resident(self.layer) == set(st["t1"]) | set(st["t2"]), "slot map differs from ARC"


class LayeredExpertCache:
    """Per-layer ARC caches sized by a CachePlan, state on the GPU (cache.py:182-204)."""

    def __init__(self, plan: CachePlan):
        self.plan = plan
        self.engine = None
        self._pending_seeds: dict = {}
        self.layers = [_LayerView(self, l) for l in range(len(plan.per_layer_capacity))]

    def capacity(self, layer: int) -> int:
        return self.plan.per_layer_capacity[layer]

    def _engine_or_raise(self):
        if self.engine is None:
            raise InvalidConfig("this cache is not bound to a device engine yet; run simulate_decoding/"
                                "simulate_prefill with it (or call bind) first")
        return self.engine

    def bind(self, engine) -> None:
        if self.engine is engine:
            return
        if self.engine is not None:
            raise InvalidConfig("cache is already bound to another engine")
        if tuple(int(c) for c in engine.caps) != tuple(self.plan.per_layer_capacity):
            raise InvalidConfig("engine capacities differ from the cache plan")
        self.engine = engine
        for layer, experts in self._pending_seeds.items():
            engine.seed_resident(layer, experts)
        self._pending_seeds.clear()

    def contains(self, layer: int, expert: int) -> bool:
        return int(expert) in self.layers[layer].resident()

    def seed_resident(self, layer: int, experts: Iterable[int]) -> None:
        if self.engine is not None:
            self.engine.seed_resident(layer, [int(e) for e in experts])
            return
        cur = self._pending_seeds.setdefault(layer, [])
        for e in experts:
            if len(cur) >= self.capacity(layer):
                break
            if int(e) not in cur:
                cur.append(int(e))


def arc_access(cache: LayeredExpertCache, layer: int, expert: int) -> bool:
    return cache.layers[layer].access(int(expert))


def update_after_layer(cache: LayeredExpertCache, layer: int, chosen: Iterable[int]) -> None:
    """ARC over the chosen experts in ascending id order (cache.py:212-215), one K2 launch."""
    cache._engine_or_raise().access(layer, sorted(int(x) for x in chosen))


@dataclass
class HitCounters:
    hits: int = 0
    misses: int = 0

    def record(self, hit: bool) -> None:
        if hit:
            self.hits += 1
        else:
            self.misses += 1


def hit_rate(counters: HitCounters) -> float:
    total = counters.hits + counters.misses
    if total == 0:
        raise NoAccesses("no expert accesses recorded")
    return counters.hits / total


def suggest_shallow_boundary(per_layer_recall: Sequence[float], plateau_fraction: float = 0.9) -> int:
    n = len(per_layer_recall)
    if n == 0:
        raise InvalidConfig("recall curve is empty")
    tail = max(1, n // 4)
    thr = plateau_fraction * sum(per_layer_recall[-tail:]) / tail
    return next((l for l, r in enumerate(per_layer_recall) if r >= thr), n)
