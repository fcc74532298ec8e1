"""Standalone device ops over torch tensors (each one call into the C ABI).

torch supplies device memory and streams; every computation here runs in
libfate_b200.so kernels.  These back the reference-API mirrors
(``gate_forward``, ``cross_layer_predict``, ``quantize``) and the tests.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr


def _stream() -> int:
    return int(torch.cuda.current_stream().cuda_stream)


def device() -> torch.device:
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def gate_predict(W, tau: float, h, top_k: int, policy: str = "topk", q: float = 0.75):
    """K1 on T vectors: (routing [T,E] f64, order [T,E] i32, list_len [T] i32), torch on device."""
    L = _lib.lib()
    dev = device()
    Wd = torch.as_tensor(np.ascontiguousarray(W, dtype=np.float64)).to(dev)
    hd = torch.as_tensor(np.ascontiguousarray(np.atleast_2d(h), dtype=np.float64)).to(dev)
    T, H = hd.shape
    E = Wd.shape[0]
    routing = torch.empty((T, E), dtype=torch.float64, device=dev)
    order = torch.empty((T, E), dtype=torch.int32, device=dev)
    lens = torch.empty((T,), dtype=torch.int32, device=dev)
    check(L.fate_gate_forward(ptr(Wd), float(tau), ptr(hd), T, E, H, ptr(routing), ptr(order), ptr(lens), top_k,
                              1 if policy == "percentile" else 0, float(q), _stream()), "fate_gate_forward")
    return routing, order, lens


def gate_forward_batch(W, tau: float, h) -> np.ndarray:
    routing, _, _ = gate_predict(W, tau, h, 1)
    return routing.cpu().numpy()


def quant_pack(w: torch.Tensor, bits: int, group: int = 64, want64: bool = False):
    """K5: (codes u8, sz f32 [groups,2], scale64, zero64) for a device tensor (fp32 or fp64)."""
    L = _lib.lib()
    n = w.numel()
    n_groups = max(1, -(-n // group))
    codes = torch.empty((-(-n * bits // 8),), dtype=torch.uint8, device=w.device)
    sz = torch.empty((n_groups, 2), dtype=torch.float32, device=w.device)
    s64 = torch.empty((n_groups,), dtype=torch.float64, device=w.device) if want64 else None
    z64 = torch.empty((n_groups,), dtype=torch.float64, device=w.device) if want64 else None
    wc = w.contiguous().reshape(-1)
    fn = L.fate_quant_pack64 if wc.dtype == torch.float64 else L.fate_quant_pack
    if wc.dtype not in (torch.float64, torch.float32):
        wc = wc.float()
    check(fn(ptr(wc), n, bits, group, ptr(codes), ptr(sz), ptr(s64), ptr(z64), _stream()), "fate_quant_pack")
    return codes, sz, s64, z64


def dequant(codes: torch.Tensor, sz: torch.Tensor, n: int, bits: int, group: int = 64) -> torch.Tensor:
    L = _lib.lib()
    out = torch.empty((n,), dtype=torch.float32, device=codes.device)
    check(L.fate_dequant(ptr(codes), ptr(sz), n, bits, group, ptr(out), _stream()), "fate_dequant")
    return out


def dequant64(codes: torch.Tensor, s64: torch.Tensor, z64: torch.Tensor, n: int, bits: int,
              group: int = 64) -> torch.Tensor:
    L = _lib.lib()
    out = torch.empty((n,), dtype=torch.float64, device=codes.device)
    check(L.fate_dequant64(ptr(codes), ptr(s64), ptr(z64), n, bits, group, ptr(out), _stream()), "fate_dequant64")
    return out


def expert_buffer_bytes(H: int, I: int, bits: int) -> int:
    v = _lib.load().fate_expert_buffer_bytes(H, I, bits)
    if v < 0:
        from .errors import InvalidConfig
        raise InvalidConfig(f"no packed layout for H={H}, I={I}, bits={bits}")
    return int(v)


def pack_expert(w1: torch.Tensor, w3: torch.Tensor, w2: torch.Tensor, bits: int, layer: int = 0, expert: int = 0,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """Pack (w1 [I,H], w3 [I,H], w2 [H,I]) fp32 into one self-describing device buffer."""
    L = _lib.lib()
    I, H = w1.shape
    nb = expert_buffer_bytes(H, I, bits)
    if out is None:
        out = torch.empty((nb,), dtype=torch.uint8, device=w1.device)
    check(L.fate_pack_expert(ptr(w1.contiguous()), ptr(w3.contiguous()), ptr(w2.contiguous()), H, I, bits, layer,
                             expert, ptr(out), _stream()), "fate_pack_expert")
    return out


def ffn_decode(x: torch.Tensor, bufs: list, weights) -> torch.Tensor:
    """K3 standalone: y = sum_j w_j FFN_j(x) over packed expert buffers (device uint8 tensors)."""
    L = _lib.lib()
    H = x.numel()
    n = len(bufs)
    arr = (C.c_void_p * n)(*[ptr(b) for b in bufs])
    w = (C.c_float * n)(*[float(v) for v in weights])
    total_I = 0
    for b in bufs:
        hdr = b[:_lib.HEADER_BYTES].view(torch.int32).cpu()
        total_I += int(hdr[5])
    scratch = torch.empty((total_I,), dtype=torch.float32, device=x.device)
    y = torch.empty((H,), dtype=torch.float32, device=x.device)
    check(L.fate_ffn_decode(ptr(x.contiguous()), H, n, arr, w, ptr(scratch), ptr(y), _stream()), "fate_ffn_decode")
    return y


def ffn_decode_timed(x: torch.Tensor, sets: list, weights, iters: int = 50):
    """K3 launched `iters` times back to back cycling over expert `sets` (lists of
    packed buffers of equal length); returns (y, mean kernel ms from CUDA events)."""
    L = _lib.lib()
    H = x.numel()
    n, ns = len(sets[0]), len(sets)
    flat = [b for s in sets for b in s]
    arr = (C.c_void_p * len(flat))(*[ptr(b) for b in flat])
    w = (C.c_float * n)(*[float(v) for v in weights])
    y = torch.empty((H,), dtype=torch.float32, device=x.device)
    ms = C.c_float(0.0)
    check(L.fate_ffn_decode_timed(ptr(x.contiguous()), H, n, ns, arr, w, ptr(y), iters, _stream(), C.byref(ms)),
          "fate_ffn_decode_timed")
    return y, float(ms.value)


def ffn_prefill(X: torch.Tensor, bufs: list, tok_lists: list, tok_weights: list) -> torch.Tensor:
    """K4 standalone: Y[t] = sum over experts e of w_{t,e} FFN_e(X[t]) for token lists per expert."""
    L = _lib.lib()
    T, H = X.shape
    n = len(bufs)
    arr = (C.c_void_p * n)(*[ptr(b) for b in bufs])
    off = np.zeros(n + 1, dtype=np.int32)
    for j, t in enumerate(tok_lists):
        off[j + 1] = off[j] + len(t)
    idx = torch.as_tensor(np.concatenate([np.asarray(t, np.int32) for t in tok_lists]) if n else np.zeros(0, np.int32),
                          device=X.device)
    tw = torch.as_tensor(np.concatenate([np.asarray(w, np.float32) for w in tok_weights]) if n else np.zeros(0, np.float32),
                         device=X.device)
    Y = torch.zeros((T, H), dtype=torch.float32, device=X.device)
    offc = (C.c_int32 * (n + 1))(*off.tolist())
    check(L.fate_ffn_prefill(ptr(X.contiguous()), T, H, n, arr, ptr(idx), ptr(tw), offc, ptr(Y), _stream()),
          "fate_ffn_prefill")
    return Y


def dense_step(dims: dict, layer: dict, kv: torch.Tensor, h_prev: torch.Tensor, y_prev, gate_in, pos: int) -> dict:
    """One dense step (attention block + shared-expert gate) on the device,
    ``fate_dense_step``; returns the intermediate vectors (for numerics tests)."""
    L = _lib.lib()
    H, nh, nkv, hd = dims["H"], dims["n_heads"], dims["n_kv_heads"], dims["head_dim"]
    dev = h_prev.device
    out = {k: torch.empty(n, dtype=torch.float32, device=dev) for k, n in
           (("h", H), ("qkv", (nh + 2 * nkv) * hd), ("q", nh * hd), ("o", nh * hd), ("a", H),
            ("part_o", 128 * nh * hd), ("part_ml", 128 * nh * 2), ("gate", 1))}
    gw = layer.get("shared_gate")
    check(L.fate_dense_step(H, nh, nkv, hd, dims.get("eps", 1e-6), dims.get("rope_theta", 1e6), ptr(layer["wqkv"]),
                            ptr(layer.get("bqkv")), ptr(layer["norm"]), ptr(layer["wo"]), ptr(kv), ptr(gw),
                            ptr(out["gate"]) if gw is not None else None, ptr(h_prev), ptr(y_prev), ptr(gate_in), pos,
                            ptr(out["h"]), ptr(out["qkv"]), ptr(out["q"]), ptr(out["o"]), ptr(out["a"]),
                            ptr(out["part_o"]), ptr(out["part_ml"]), _stream()), "fate_dense_step")
    return out
