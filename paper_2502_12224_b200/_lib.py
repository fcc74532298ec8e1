"""ctypes binding of libfate_b200.so (include/fate_b200.h).

The library is the product: there is no CPU fallback.  ``lib()`` raises
DeviceError when the .so is missing or no CUDA device is visible; every
wrapper checks the returned status and raises the matching SimError.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError, raise_for

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfate_b200.so")

MAX_EXPERTS = 256
MAX_TOPK = 16
HEADER_BYTES = 256

c_int, c_i64, c_dbl, c_vp = C.c_int, C.c_int64, C.c_double, C.c_void_p
P_i32 = C.POINTER(C.c_int32)


class EngineConfig(C.Structure):
    _fields_ = [
        ("num_layers", c_int), ("num_experts", c_int), ("top_k", c_int), ("hidden_dim", c_int),
        ("intermediate_dim", c_int), ("shared_intermediate", c_int), ("shared_bits", c_int),
        ("capacity", P_i32), ("cached_bits", c_int), ("prefetch_bits", c_int), ("ondemand_bits", c_int),
        ("use_predictor", c_int), ("policy", c_int), ("percentile_q", c_dbl), ("budget_n", c_int),
        ("prefill_use_predictor", c_int), ("reorder_prefill", c_int), ("p_int2", c_dbl),
        ("prefill_ondemand_bits", c_int), ("max_tokens", c_int), ("max_inflight", c_int), ("device", c_int),
    ]


K_, E_ = MAX_TOPK, MAX_EXPERTS


class StepLog(C.Structure):
    _fields_ = [
        ("chosen", C.c_int32 * K_), ("src_bits", C.c_int32 * K_), ("hit", C.c_int32 * K_),
        ("ondemand", C.c_int32 * K_), ("victims", C.c_int32 * K_),
        ("n_ondemand", C.c_int32), ("n_victims", C.c_int32), ("n_pred", C.c_int32), ("n_prefetch", C.c_int32),
        ("arrived", C.c_int32 * K_), ("pred", C.c_int32 * E_), ("prefetch", C.c_int32 * E_),
        ("routing", C.c_float * K_), ("fmt_bits", C.c_int32 * K_), ("mismatch", C.c_int32), ("pad", C.c_int32),
    ]


class PrefillLog(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_pred", "n_prefetch", "n_active", "n_resident", "n_planned",
                                          "n_ondemand", "n_victims", "n_started")] + [
        (n, C.c_int32 * E_) for n in ("pred_order", "pred_counts", "prefetch", "prefetch_bits", "actives", "counts",
                                     "resident", "planned", "ondemand", "src_bits", "victims", "started")] + [
        ("mismatch", C.c_int32), ("pad", C.c_int32)]


class RunStats(C.Structure):
    _fields_ = [
        ("gpu_ms", c_dbl), ("ffn_ms", c_dbl), ("gate_ms", c_dbl),
        ("steps", c_i64), ("accesses", c_i64), ("cache_hits", c_i64), ("arrival_hits", c_i64),
        ("dequant_count", c_i64), ("prefetch_issued", c_i64), ("ondemand_issued", c_i64),
        ("transfers_done", c_i64), ("transfers_dropped", c_i64), ("h2d_bytes", c_i64),
        ("copy_busy_ms", c_dbl), ("recall_sum", c_dbl), ("recall_n", c_i64), ("trace_mismatches", c_i64),
        ("ffn_bytes", c_i64), ("ffn_flops", c_dbl), ("near_ties", c_i64), ("d2d_bytes", c_i64),
        ("error", C.c_int32), ("pad", C.c_int32), ("dense_ms", c_dbl), ("k3_wait_ms", c_dbl),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_ if name != "pad"}


# name -> (restype, argtypes); the exported symbol set of include/fate_b200.h
SIGNATURES = {
    "fate_version": (c_int, []),
    "fate_last_error": (C.c_char_p, []),
    "fate_device_count": (c_int, [P_i32]),
    "fate_quant_pack": (c_int, [c_vp, c_i64, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fate_quant_pack64": (c_int, [c_vp, c_i64, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fate_dequant": (c_int, [c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp]),
    "fate_dequant64": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp]),
    "fate_pack_expert": (c_int, [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp]),
    "fate_expert_buffer_bytes": (c_i64, [c_int, c_int, c_int]),
    "fate_gate_forward": (c_int, [c_vp, c_dbl, c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_int, c_int, c_dbl, c_vp]),
    "fate_ffn_decode": (c_int, [c_vp, c_int, c_int, C.POINTER(c_vp), C.POINTER(C.c_float), c_vp, c_vp, c_vp]),
    "fate_k3_profile": (c_int, [c_vp]),
    "fate_k4_profile": (c_int, [c_vp]),
    "fate_engine_set_expert_sources": (c_int, [c_vp, c_int, c_vp]),
    "fate_ipc_get_handle": (c_int, [c_vp, c_vp, C.POINTER(c_i64)]),
    "fate_ipc_open_handle": (c_int, [c_vp, C.POINTER(c_vp)]),
    "fate_ipc_close": (c_int, [c_vp]),
    "fate_host_register": (c_int, [c_vp, c_i64]),
    "fate_dense_step": (c_int, [c_int, c_int, c_int, c_int, C.c_float, C.c_float] + [c_vp] * 10 + [c_int]
                        + [c_vp] * 8),
    "fate_host_unregister": (c_int, [c_vp]),
    "fate_engine_set_copy_timing": (c_int, [c_vp, c_int]),
    "fate_engine_set_overlap": (c_int, [c_vp, c_int]),
    "fate_channel_create": (c_int, [c_int, c_int, C.POINTER(c_vp)]),
    "fate_channel_destroy": (c_int, [c_vp]),
    "fate_channel_enqueue": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_i64, C.POINTER(c_i64)]),
    "fate_channel_promote": (c_int, [c_vp]),
    "fate_channel_drop_stale": (c_int, [c_vp, c_int, c_int, C.POINTER(c_int)]),
    "fate_channel_pump": (c_int, [c_vp]),
    "fate_channel_wait": (c_int, [c_vp, c_i64, c_vp]),
    "fate_channel_find": (c_int, [c_vp, c_int, c_int, c_int, C.POINTER(c_int), C.POINTER(c_i64)]),
    "fate_channel_pending": (c_int, [c_vp, C.POINTER(c_i64), c_int, C.POINTER(c_int), C.POINTER(c_int)]),
    "fate_engine_set_dense": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_int, C.c_float, C.c_float]),
    "fate_engine_set_dense_layer": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fate_ffn_decode_timed": (c_int, [c_vp, c_int, c_int, c_int, C.POINTER(c_vp), C.POINTER(C.c_float), c_vp, c_int,
                                      c_vp, C.POINTER(C.c_float)]),
    "fate_k1_profile": (c_int, [c_vp]),
    "fate_ffn_prefill": (c_int, [c_vp, c_int, c_int, c_int, C.POINTER(c_vp), c_vp, c_vp, P_i32, c_vp, c_vp]),
    "fate_engine_create": (c_int, [C.POINTER(EngineConfig), C.POINTER(c_vp)]),
    "fate_engine_destroy": (c_int, [c_vp]),
    "fate_engine_set_strategy": (c_int, [c_vp, C.POINTER(EngineConfig)]),
    "fate_engine_timeline": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_int, P_i32]),
    "fate_engine_set_gate": (c_int, [c_vp, c_vp, c_vp]),
    "fate_engine_reset_eap": (c_int, [c_vp]),
    "fate_engine_set_host_pool": (c_int, [c_vp, c_int, c_vp, c_i64]),
    "fate_engine_set_shared": (c_int, [c_vp, c_int, c_vp]),
    "fate_engine_reset_cache": (c_int, [c_vp]),
    "fate_engine_seed_resident": (c_int, [c_vp, c_int, P_i32, c_int]),
    "fate_engine_resident": (c_int, [c_vp, c_int, P_i32]),
    "fate_engine_access": (c_int, [c_vp, c_int, P_i32, c_int, P_i32]),
    "fate_engine_arc_state": (c_int, [c_vp, c_int, P_i32, P_i32, P_i32, P_i32, P_i32, C.POINTER(c_dbl)]),
    "fate_engine_decode": (c_int, [c_vp, c_vp, c_vp, c_int, c_vp, c_vp, C.POINTER(RunStats)]),
    "fate_engine_prefill": (c_int, [c_vp, c_vp, c_vp, c_int, c_vp, C.POINTER(PrefillLog), C.POINTER(RunStats)]),
}

_LIB = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the library and bind every declared symbol (no device check)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise DeviceError(f"{path} is not built; run `python -m paper_2502_12224_b200.build` "
                          "(no CPU fallback exists for the offload engine)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def lib() -> C.CDLL:
    """The loaded library, after checking a CUDA device is usable."""
    L = load()
    n = C.c_int32(0)
    st = L.fate_device_count(C.byref(n))
    if st != 0 or n.value < 1:
        raise DeviceError("no CUDA device visible to libfate_b200 (the B200 path has no CPU fallback): "
                          + L.fate_last_error().decode())
    return L


def check(status: int, what: str) -> None:
    if status != 0:
        detail = load().fate_last_error().decode(errors="replace")
        raise_for(status, what, detail)


def ptr(t) -> int:
    """Raw device/host pointer of a torch tensor (or 0 for None)."""
    return 0 if t is None else int(t.data_ptr())
