"""Gate weights, the device gate, and the synthetic trace workload generator.

* ``GateWeights`` / ``GenConfig`` / ``default_sharpness`` mirror the
  reference's ``moesim.gatesim`` types (gatesim.py:37-103).
* ``gate_forward`` runs the fp64 router on the GPU (kernel K1,
  ``fate_gate_forward`` in include/fate_b200.h): softmax(W_l h / tau_l),
  gatesim.py:113-123.
* ``gen_trace`` is the seeded synthetic WORKLOAD generator
  (gatesim.py:145-240): it produces the gate-input chains the engine replays.
  It is input synthesis, not part of the executed path; it reproduces the
  reference's draw order exactly so the same seed yields byte-identical
  NDJSON (pinned by tests/test_tracegen.py against golden hashes).  The
  routing weights it stores in the trace are computed on the host only so
  the trace file is self-consistent; the engine recomputes routing on the
  device and checks it against the trace.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import GateTrace, ModelConfig, TraceRecord, top_k_set
from .errors import DegenerateGen, InvalidConfig, ZeroVector

# theta(s) = min(1, COEF / s**EXP): share of chain noise inside the consuming
# gate's row space (gatesim.py:29-34).
THETA_COEF = 0.13
THETA_EXP = 2.7


def default_sharpness(num_layers: int, temp_shallow: float = 2.0, temp_deep: float = 0.5) -> tuple:
    if num_layers == 1:
        return (1.0 / temp_shallow,)
    return tuple(1.0 / t for t in np.linspace(temp_shallow, temp_deep, num_layers))


@dataclass(frozen=True)
class GenConfig:
    rho_adjacent: float = 0.888
    rho_within: float | None = None
    layer_sharpness: tuple | None = None
    seed: int = 0
    num_tokens: int = 64
    phase: str = "decoding"

    def resolved_rho_within(self) -> float:
        return float(np.sqrt(self.rho_adjacent)) if self.rho_within is None else self.rho_within

    def resolved_sharpness(self, num_layers: int) -> tuple:
        if self.layer_sharpness is None:
            return default_sharpness(num_layers)
        if len(self.layer_sharpness) != num_layers:
            raise InvalidConfig(f"layer_sharpness has {len(self.layer_sharpness)} entries, expected {num_layers}")
        return tuple(self.layer_sharpness)


@dataclass(frozen=True)
class GateWeights:
    """Per-layer [E, H] fp64 router matrices and temperatures."""

    matrices: tuple
    temperatures: tuple

    def __post_init__(self):
        mats = []
        for m in self.matrices:
            a = np.asarray(m, dtype=np.float64)
            if not np.all(np.isfinite(a)):
                raise InvalidConfig("gate weight matrix has non-finite entries")
            a.flags.writeable = False
            mats.append(a)
        object.__setattr__(self, "matrices", tuple(mats))
        object.__setattr__(self, "temperatures", tuple(float(t) for t in self.temperatures))
        if len(self.matrices) != len(self.temperatures):
            raise InvalidConfig("one temperature per gate matrix required")
        if any(t <= 0 for t in self.temperatures):
            raise InvalidConfig("temperatures must be > 0")

    @property
    def num_layers(self) -> int:
        return len(self.matrices)

    def stacked(self) -> np.ndarray:
        """[L, E, H] contiguous fp64 — the device layout of the router weights."""
        return np.ascontiguousarray(np.stack(self.matrices))


def gate_forward(w: GateWeights, layer: int, hidden) -> np.ndarray:
    """Routing distribution softmax(W_l h / tau_l), computed by kernel K1 on the GPU."""
    h = np.asarray(hidden, dtype=np.float64)
    mat = w.matrices[layer]
    if h.shape[0] != mat.shape[1]:
        raise InvalidConfig(f"hidden vector has dim {h.shape[0]}, gate expects {mat.shape[1]}")
    if not np.all(np.isfinite(h)):
        raise InvalidConfig("hidden vector has non-finite entries")
    from . import ops

    return ops.gate_forward_batch(mat, w.temperatures[layer], h[None, :])[0]


def softmax(z) -> np.ndarray:
    """Host helper kept for API parity (gatesim.py:106-110)."""
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max())
    return e / e.sum()


def cosine_similarity(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise InvalidConfig(f"vector shapes differ: {a.shape} vs {b.shape}")
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na == 0.0 or nb == 0.0:
        raise ZeroVector("cosine similarity of a zero vector is undefined")
    return float(np.dot(a, b) / (na * nb))


def noise_fraction_in_gate_space(sharpness: float) -> float:
    return min(1.0, THETA_COEF / sharpness ** THETA_EXP)


class _Chain:
    """The steered hidden-state walk of gatesim.py:145-167 for one trace."""

    def __init__(self, rng: np.random.Generator, bases: list, thetas: list):
        self.rng, self.bases, self.thetas = rng, bases, thetas

    @staticmethod
    def unit(v: np.ndarray) -> np.ndarray:
        return v / np.linalg.norm(v)

    def step(self, h: np.ndarray, rho: float, layer: int) -> np.ndarray:
        if rho >= 1.0:
            return h
        B, th = self.bases[layer], self.thetas[layer]
        inside = B @ self.rng.standard_normal(B.shape[1])
        outside = self.rng.standard_normal(h.shape[0])
        outside -= B @ (B.T @ outside)
        g = np.sqrt(th) * self.unit(inside) + np.sqrt(1.0 - th) * self.unit(outside)
        g -= np.dot(g, h) * h
        g = self.unit(g)
        return rho * h + np.sqrt(1.0 - rho * rho) * g


def _host_routing(mat: np.ndarray, tau: float, h: np.ndarray) -> np.ndarray:
    z = mat @ h / tau
    e = np.exp(z - z.max())
    return e / e.sum()


def gen_trace(cfg: ModelConfig, gen: GenConfig, weights: GateWeights | None = None):
    """Seeded synthetic decode/prefill trace plus its gate weights (gatesim.py:170-240)."""
    if not 0.0 < gen.rho_adjacent <= 1.0:
        raise InvalidConfig("rho_adjacent must lie in (0, 1]")
    rho_w = gen.resolved_rho_within()
    if not 0.0 < rho_w <= 1.0:
        raise InvalidConfig("rho_within must lie in (0, 1]")
    if rho_w < gen.rho_adjacent - 1e-12:
        raise DegenerateGen(f"rho_within={rho_w:.4f} < rho_adjacent={gen.rho_adjacent:.4f}: "
                            "the across-block step would need cosine > 1")
    rho_x = min(1.0, gen.rho_adjacent / rho_w)
    if gen.num_tokens < 1:
        raise InvalidConfig("num_tokens must be >= 1")
    rng = np.random.default_rng(gen.seed)
    H, E, L = cfg.hidden_dim, cfg.num_experts, cfg.num_layers
    if weights is None:
        sharp = gen.resolved_sharpness(L)
        if any(s <= 0 for s in sharp):
            raise InvalidConfig("sharpness values must be > 0")
        weights = GateWeights(tuple(rng.standard_normal((E, H)) for _ in range(L)),
                              tuple(1.0 / s for s in sharp))
    else:
        if weights.num_layers != L or weights.matrices[0].shape != (E, H):
            raise InvalidConfig("provided gate weights do not match the model geometry")
        sharp = tuple(1.0 / t for t in weights.temperatures)
    bases = [np.linalg.qr(m.T)[0][:, : min(E, H)] for m in weights.matrices]
    chain = _Chain(rng, bases, [noise_fraction_in_gate_space(s) for s in sharp])
    recs = []
    for tok in range(gen.num_tokens):
        attn = chain.unit(rng.standard_normal(H))
        for layer in range(L):
            gin = chain.step(attn, rho_w, layer)
            nxt = chain.step(gin, rho_x, min(layer + 1, L - 1))
            routing = _host_routing(weights.matrices[layer], weights.temperatures[layer], gin)
            recs.append(TraceRecord(tok, layer, top_k_set(routing, cfg.top_k), routing,
                                    {"attn_in_next": nxt, "gate_in_cur": gin, "attn_in_cur": attn}))
            attn = nxt
    return GateTrace(tuple(recs), gen.phase, "synthetic"), weights
