"""OffloadEngine: the Python handle of the C-ABI engine (fate_engine_*).

One engine = one GPU's expert-slot pool + per-layer ARC tables + copy
channel for a given model geometry and cache plan.  Strategy knobs can be
changed between runs (``set_strategy``) while the cache state persists, which
is how ``compare_strategies`` chains prefill into decode (pipeline.py:835-850).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import EngineConfig, PrefillLog, RunStats, StepLog, check, ptr
from .core import ModelConfig
from .errors import InvalidConfig


def overlap_default() -> bool:
    """The decode step protocol engines start with: arrival-gated K3 unless
    FATE_OVERLAP=0.  A waiting K3 holds every SM of its GPU, so processes that
    time-share one GPU (more ranks than devices) should use the stream wait."""
    import os
    return os.environ.get("FATE_OVERLAP", "1") != "0"
from .experts import ExpertStore


@dataclass(frozen=True)
class StrategyKnobs:
    """The subset of pipeline.Strategy the device engine reads."""

    use_predictor: bool = True
    policy: str = "percentile"
    percentile_q: float = 0.75
    budget_n: int = 0
    cached_bits: int = 4
    prefetch_bits: int = 4
    ondemand_bits: int = 2
    prefill_use_predictor: bool = True
    reorder_prefill: bool = True
    p_int2: float = 0.25
    prefill_ondemand_bits: int = 2
    max_inflight: int = 2


@dataclass
class DecodeResult:
    tokens: list
    y: torch.Tensor                 # [T, L, H] fp32 on device
    stats: dict
    logs: list | None               # per-step dicts (timing-independent parity fields)
    step_ms: np.ndarray | None      # [T*L, 4]
    copies: list                    # (start, end, kind, step, layer, expert, bits)


class OffloadEngine:
    def __init__(self, cfg: ModelConfig, capacities, store: ExpertStore, weights, knobs: StrategyKnobs,
                 max_tokens: int = 1024, device: int | None = None):
        self._L = _lib.lib()
        self.cfg, self.store, self.weights = cfg, store, weights
        self.caps = np.ascontiguousarray(np.asarray(capacities, dtype=np.int32))
        if self.caps.shape != (cfg.num_layers,):
            raise InvalidConfig("one capacity per layer required")
        self.knobs = knobs
        self.max_tokens = int(max_tokens)
        self.device = torch.cuda.current_device() if device is None else int(device)
        c = self._config(knobs)
        h = C.c_void_p()
        check(self._L.fate_engine_create(C.byref(c), C.byref(h)), "fate_engine_create")
        self._h = h
        self.set_overlap(overlap_default())
        W = np.ascontiguousarray(np.stack([np.asarray(m, np.float64) for m in weights.matrices]))
        tau = np.ascontiguousarray(np.asarray(weights.temperatures, np.float64))
        if W.shape != (cfg.num_layers, cfg.num_experts, cfg.hidden_dim):
            raise InvalidConfig("gate weights do not match the model geometry")
        check(self._L.fate_engine_set_gate(h, W.ctypes.data, tau.ctypes.data), "fate_engine_set_gate")
        for b in store.bits:
            check(self._L.fate_engine_set_host_pool(h, b, ptr(store.host_pool(b)), store.stride(b)),
                  "fate_engine_set_host_pool")
        if store.shared_intermediate:
            for l in range(cfg.num_layers):
                check(self._L.fate_engine_set_shared(h, l, ptr(store.shared_buffer(l))), "fate_engine_set_shared")

    def _config(self, k: StrategyKnobs) -> EngineConfig:
        cfg = self.cfg
        self._caps_c = self.caps.ctypes.data_as(C.POINTER(C.c_int32))
        return EngineConfig(
            num_layers=cfg.num_layers, num_experts=cfg.num_experts, top_k=cfg.top_k, hidden_dim=cfg.hidden_dim,
            intermediate_dim=cfg.intermediate_dim, shared_intermediate=self.store.shared_intermediate,
            shared_bits=self.store.shared_bits, capacity=self._caps_c, cached_bits=k.cached_bits,
            prefetch_bits=k.prefetch_bits, ondemand_bits=k.ondemand_bits, use_predictor=int(k.use_predictor),
            policy={"percentile": 1, "eap": 2}.get(k.policy, 0), percentile_q=k.percentile_q, budget_n=k.budget_n,
            prefill_use_predictor=int(k.prefill_use_predictor), reorder_prefill=int(k.reorder_prefill),
            p_int2=k.p_int2, prefill_ondemand_bits=k.prefill_ondemand_bits, max_tokens=self.max_tokens,
            max_inflight=k.max_inflight, device=self.device)

    def set_dense(self, dense, max_ctx: int, ctx0: int) -> None:
        """Execute the dense part (``dense.DenseWeights``) in every decode step:
        the K/V cache holds ``max_ctx`` positions per layer, the first ``ctx0`` of
        them a synthetic prompt; decode token t runs at position ctx0 + t."""
        dc = dense.dc
        check(self._L.fate_engine_set_dense(self._h, dc.n_heads, dc.n_kv_heads, dc.head_dim, int(max_ctx), int(ctx0),
                                            dc.eps, dc.rope_theta), "fate_engine_set_dense")
        if getattr(self, "dense", None) is dense and getattr(self, "_dense_ctx", None) == (max_ctx, ctx0):
            return
        self._dense_ctx = (max_ctx, ctx0)
        for l, ly in enumerate(dense.layers):
            check(self._L.fate_engine_set_dense_layer(self._h, l, ptr(ly["wqkv"]), ptr(ly["bqkv"]), ptr(ly["norm"]),
                                                      ptr(ly["wo"]), ptr(ly["shared_gate"])),
                  "fate_engine_set_dense_layer")
        self.dense = dense  # the engine reads these buffers on every step

    def set_copy_timing(self, stride: int) -> None:
        """Time every stride-th transfer of timed runs (default 8; 1: every one, 0: none)."""
        check(self._L.fate_engine_set_copy_timing(self._h, int(stride)), "fate_engine_set_copy_timing")

    def set_overlap(self, on: bool) -> None:
        """Decode: K3 launched behind K1 and gated per expert on its copy (default),
        or the compute stream waits for all of a step's copies first."""
        check(self._L.fate_engine_set_overlap(self._h, int(bool(on))), "fate_engine_set_overlap")

    def set_strategy(self, knobs: StrategyKnobs) -> None:
        c = self._config(knobs)
        check(self._L.fate_engine_set_strategy(self._h, C.byref(c)), "fate_engine_set_strategy")
        self.knobs = knobs

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.fate_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- cache protocol (cache.py:182-215) ----------------------------------
    def reset_cache(self) -> None:
        check(self._L.fate_engine_reset_cache(self._h), "fate_engine_reset_cache")

    def reset_eap(self) -> None:
        """EAP co-activation statistics back to empty (a fresh EapStats, predict.py:110-130)."""
        check(self._L.fate_engine_reset_eap(self._h), "fate_engine_reset_eap")

    def resident(self, layer: int) -> set:
        out = (C.c_int32 * self.cfg.num_experts)()
        check(self._L.fate_engine_resident(self._h, layer, out), "fate_engine_resident")
        return {e for e in range(self.cfg.num_experts) if out[e]}

    def access(self, layer: int, experts) -> list:
        ex = np.ascontiguousarray(np.asarray(list(experts), dtype=np.int32))
        hits = np.zeros(len(ex), dtype=np.int32)
        check(self._L.fate_engine_access(self._h, layer, ex.ctypes.data_as(C.POINTER(C.c_int32)), len(ex),
                                         hits.ctypes.data_as(C.POINTER(C.c_int32))), "fate_engine_access")
        return [bool(h) for h in hits]

    def set_expert_sources(self, bits: int, ptrs) -> None:
        """Expert-sharded mode: misses of width ``bits`` copy from ptrs[l*E + e]
        (device or peer buffers; 0 keeps the host copy).  ``None`` clears."""
        if ptrs is None:
            check(self._L.fate_engine_set_expert_sources(self._h, bits, None), "fate_engine_set_expert_sources")
            return
        n = self.cfg.num_layers * self.cfg.num_experts
        if len(ptrs) != n:
            raise InvalidConfig(f"expected {n} source pointers, got {len(ptrs)}")
        arr = (C.c_void_p * n)(*[int(p) or None for p in ptrs])
        check(self._L.fate_engine_set_expert_sources(self._h, bits, arr), "fate_engine_set_expert_sources")

    def seed_resident(self, layer: int, experts) -> None:
        ex = np.ascontiguousarray(np.asarray(list(experts), dtype=np.int32))
        check(self._L.fate_engine_seed_resident(self._h, layer, ex.ctypes.data_as(C.POINTER(C.c_int32)), len(ex)),
              "fate_engine_seed_resident")

    def arc_state(self, layer: int) -> dict:
        E = self.cfg.num_experts
        arrs = [(C.c_int32 * E)() for _ in range(4)]
        lens = (C.c_int32 * 4)()
        p = C.c_double()
        check(self._L.fate_engine_arc_state(self._h, layer, *arrs, lens, C.byref(p)), "fate_engine_arc_state")
        return {"t1": list(arrs[0][:lens[0]]), "t2": list(arrs[1][:lens[1]]), "b1": list(arrs[2][:lens[2]]),
                "b2": list(arrs[3][:lens[3]]), "p": p.value}

    # -- runs ---------------------------------------------------------------
    def decode(self, gate_in: torch.Tensor, chosen: torch.Tensor | None, tokens=None, want_logs: bool = False,
               timed: bool = True) -> DecodeResult:
        """Decode T tokens whose gate inputs are already on the device ([T, L, H] fp64)."""
        cfg = self.cfg
        T = gate_in.shape[0]
        if T > self.max_tokens:
            raise InvalidConfig(f"{T} tokens exceed the engine's max_tokens={self.max_tokens}")
        dev = gate_in.device
        y = torch.empty((T, cfg.num_layers, cfg.hidden_dim), dtype=torch.float32, device=dev)
        log = None
        if want_logs:
            log = torch.zeros((T * cfg.num_layers, C.sizeof(StepLog)), dtype=torch.uint8, device=dev)
        st = RunStats()
        torch.cuda.current_stream().synchronize()
        check(self._L.fate_engine_decode(self._h, ptr(gate_in), ptr(chosen), T, ptr(y), ptr(log),
                                         C.byref(st) if timed else None), "fate_engine_decode")
        logs = _parse_step_logs(log, cfg) if want_logs else None
        step_ms, copies = self.timeline() if timed else (None, [])
        return DecodeResult(list(range(T)) if tokens is None else list(tokens), y, st.as_dict(), logs, step_ms,
                            copies)

    def prefill(self, gate_in: torch.Tensor, chosen: torch.Tensor | None, timed: bool = True):
        cfg = self.cfg
        T = gate_in.shape[0]
        if T > self.max_tokens:
            raise InvalidConfig(f"{T} tokens exceed the engine's max_tokens={self.max_tokens}")
        Y = torch.empty((cfg.num_layers, T, cfg.hidden_dim), dtype=torch.float32, device=gate_in.device)
        logs = (PrefillLog * cfg.num_layers)()
        st = RunStats()
        torch.cuda.current_stream().synchronize()
        check(self._L.fate_engine_prefill(self._h, ptr(gate_in), ptr(chosen), T, ptr(Y), logs,
                                          C.byref(st) if timed else None), "fate_engine_prefill")
        step_ms, copies = self.timeline() if timed else (None, [])
        return Y, st.as_dict(), [_parse_prefill_log(lg) for lg in logs], step_ms, copies

    def timeline(self):
        counts = (C.c_int32 * 2)()
        check(self._L.fate_engine_timeline(self._h, None, 0, None, None, 0, counts), "fate_engine_timeline")
        ns, nc = counts[0], counts[1]
        sm = np.zeros((max(ns, 1), 4))
        cm = np.zeros((max(nc, 1), 2))
        meta = np.zeros((max(nc, 1), 5), dtype=np.int32)
        check(self._L.fate_engine_timeline(self._h, sm.ctypes.data, ns, cm.ctypes.data, meta.ctypes.data, nc, counts),
              "fate_engine_timeline")
        copies = [(float(cm[i, 0]), float(cm[i, 1]), *[int(v) for v in meta[i]]) for i in range(nc)]
        return sm[:ns], copies


def _parse_step_logs(log: torch.Tensor, cfg: ModelConfig) -> list:
    raw = log.cpu().numpy()
    out = []
    k = cfg.top_k
    for s in range(raw.shape[0]):
        lg = StepLog.from_buffer_copy(raw[s].tobytes())
        rec = {"token": s // cfg.num_layers, "layer": s % cfg.num_layers,
               "chosen": list(lg.chosen[:k]), "src_bits": list(lg.src_bits[:k]),
               "hits": [lg.chosen[i] for i in range(k) if lg.hit[i]],
               "ondemand": list(lg.ondemand[:lg.n_ondemand]), "victims": list(lg.victims[:lg.n_victims]),
               "arrived": [lg.chosen[i] for i in range(k) if lg.arrived[i]],
               "routing": list(lg.routing[:k]), "fmt_bits": list(lg.fmt_bits[:k]), "mismatch": lg.mismatch}
        if lg.n_pred >= 0:
            rec["pred"] = list(lg.pred[:lg.n_pred])
            rec["prefetch"] = list(lg.prefetch[:lg.n_prefetch])
        out.append(rec)
    return out


def _parse_prefill_log(lg: PrefillLog) -> dict:
    g = lambda name, n: list(getattr(lg, name)[:n])  # noqa: E731
    return {"pred_order": g("pred_order", lg.n_pred), "pred_counts": g("pred_counts", lg.n_pred),
            "prefetch": list(zip(g("prefetch", lg.n_prefetch), g("prefetch_bits", lg.n_prefetch))),
            "actives": g("actives", lg.n_active), "counts": g("counts", lg.n_active),
            "resident": g("resident", lg.n_resident), "planned": g("planned", lg.n_planned),
            "ondemand": g("ondemand", lg.n_ondemand), "src_bits": g("src_bits", lg.n_active),
            "victims": g("victims", lg.n_victims), "started": g("started", lg.n_started),
            "mismatch": lg.mismatch}
