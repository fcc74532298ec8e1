"""Prefetch policies, prediction lists and the cross-layer predictor.

Mirrors ``moesim.predict`` (predict.py:21-107, 167-195).  The prediction
itself (``cross_layer_predict``) runs kernel K1 on the GPU: layer l+1's
router applied to layer l's gate input, softmax in fp64, rank order by
(-weight, id) and the nearest-rank percentile prefix.  Inside the decode
engine the same computation is fused into the per-step gate launch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, NamedTuple, Sequence

import numpy as np

from .errors import InvalidConfig, MissingProbes
from .quant import PopularityProfile


@dataclass(frozen=True)
class PrefetchPolicy:
    """``topk``: the predicted top-k.  ``percentile``: every expert strictly above
    the q-th nearest-rank percentile, widened to include the top-k."""

    kind: str = "percentile"
    percentile_q: float = 0.75

    def __post_init__(self):
        if self.kind not in ("topk", "percentile"):
            raise InvalidConfig(f"unknown prefetch policy kind {self.kind!r}")
        if not 0.0 < self.percentile_q < 1.0:
            raise InvalidConfig("percentile_q must lie in (0, 1)")

    def validate_for(self, num_experts: int, top_k: int) -> "PrefetchPolicy":
        if self.kind == "percentile" and (1.0 - self.percentile_q) * num_experts < top_k:
            raise InvalidConfig(f"percentile_q={self.percentile_q} keeps fewer than top_k={top_k} "
                                f"of {num_experts} experts")
        return self


class PrefetchEntry(NamedTuple):
    expert: int
    confidence: float
    bits: int | None


@dataclass(frozen=True)
class PrefetchList:
    """Predicted experts of one layer, highest confidence first."""

    layer: int
    entries: tuple
    cold_start: bool = False

    def __post_init__(self):
        ids = [e.expert for e in self.entries]
        if len(set(ids)) != len(ids):
            raise InvalidConfig("prefetch list has duplicate expert indices")
        conf = [e.confidence for e in self.entries]
        if any(a < b for a, b in zip(conf, conf[1:])):
            raise InvalidConfig("prefetch list must be sorted by confidence descending")

    def experts(self) -> tuple:
        return tuple(e.expert for e in self.entries)

    def expert_set(self) -> frozenset:
        return frozenset(e.expert for e in self.entries)


def nearest_rank_percentile(values, q: float) -> float:
    """Value at rank ceil(q*n) of the ascending sample (predict.py:84-89)."""
    s = np.sort(np.asarray(values))
    r = min(max(int(math.ceil(q * s.shape[0])), 1), s.shape[0])
    return float(s[r - 1])


def cross_layer_predict_batch(gate_in, w, target_layer: int, policy: PrefetchPolicy, top_k: int) -> list:
    """Device K1 over T gate inputs [T, H]: one PrefetchList per row."""
    from . import ops

    routing, order, lens = ops.gate_predict(w.matrices[target_layer], w.temperatures[target_layer], gate_in, top_k,
                                            policy.kind, policy.percentile_q)
    routing, order, lens = routing.cpu().numpy(), order.cpu().numpy(), lens.cpu().numpy()
    out = []
    for t in range(order.shape[0]):
        ids = order[t, :lens[t]]
        out.append(PrefetchList(target_layer, tuple(PrefetchEntry(int(e), float(routing[t, e]), None) for e in ids)))
    return out


def cross_layer_predict(gate_in, w, target_layer: int, policy: PrefetchPolicy, top_k: int) -> PrefetchList:
    """Predict layer target_layer's experts from the previous block's gate input (predict.py:92-107)."""
    h = np.asarray(gate_in, dtype=np.float64)
    if h.ndim != 1 or h.shape[0] != w.matrices[target_layer].shape[1]:
        raise InvalidConfig("hidden vector does not match the gate's hidden dimension")
    return cross_layer_predict_batch(h[None, :], w, target_layer, policy, top_k)[0]


def prefetch_recall(predicted, actual: Iterable[int]) -> float:
    """|predicted & actual| / |actual| (predict.py:167-176)."""
    act = frozenset(int(e) for e in actual)
    if not act:
        raise InvalidConfig("actual expert set must be non-empty")
    pred = predicted.expert_set() if isinstance(predicted, PrefetchList) else frozenset(int(e) for e in predicted)
    return len(pred & act) / len(act)


def prefill_merge(per_token_lists: Sequence[PrefetchList]) -> PopularityProfile:
    """Popularity = number of token lists containing the expert (predict.py:179-195)."""
    if not per_token_lists:
        raise InvalidConfig("cannot merge an empty collection of prefetch lists")
    layers = {pl.layer for pl in per_token_lists}
    if len(layers) != 1:
        raise InvalidConfig(f"prefetch lists target multiple layers: {sorted(layers)}")
    counts: dict = {}
    for pl in per_token_lists:
        for e in pl.expert_set():
            counts[e] = counts.get(e, 0) + 1
    return PopularityProfile.from_counts(layers.pop(), counts)


class CrossLayerDecodePredictor:
    """The decode predictor protocol of pipeline.py:271-298 (issue at gate start)."""

    issue_at_gate_start = True

    def __init__(self, weights, policy: PrefetchPolicy, top_k: int):
        policy.validate_for(weights.matrices[0].shape[0], top_k)
        self.weights, self.policy, self.top_k = weights, policy, top_k

    def predict(self, token: int, source_layer: int, record, chosen=None) -> PrefetchList:
        if record.probe_hidden is None or "gate_in_cur" not in record.probe_hidden:
            raise MissingProbes(f"record (token {token}, layer {source_layer}) lacks gate_in_cur probe")
        return cross_layer_predict(record.probe_hidden["gate_in_cur"], self.weights, source_layer + 1, self.policy,
                                   self.top_k)

    def observe(self, token: int, layer: int, chosen) -> None:
        pass
