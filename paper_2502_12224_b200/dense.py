"""The dense part of a decode step on the device: the
attention block (RMSNorm, QKV projection, RoPE, K/V cache, decode attention,
output projection + residual) and the shared-expert gate, which the reference
charges as the constants ``t_attn`` / ``t_gate`` (core.py:79-83,
pipeline.py:418, 484).  ``DenseWeights`` holds random-init weights of a model's
attention geometry on the GPU; ``OffloadEngine.set_dense`` makes every decode
step execute them (csrc/dense.cu) before the gate."""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from .core import ModelConfig
from .errors import InvalidConfig


@dataclass(frozen=True)
class DenseConfig:
    n_heads: int
    n_kv_heads: int
    head_dim: int = 128
    qkv_bias: bool = False
    shared_gate: bool = False   # Qwen1.5-MoE's sigmoid shared_expert_gate
    eps: float = 1e-6
    rope_theta: float = 1e6

    @classmethod
    def qwen_moe(cls) -> "DenseConfig":    # Qwen1.5-MoE-A2.7B: 16 x 128 MHA, q/k/v bias, gated shared expert
        return cls(16, 16, 128, qkv_bias=True, shared_gate=True, eps=1e-6, rope_theta=1e6)

    @classmethod
    def deepseek_moe(cls) -> "DenseConfig":  # DeepSeek-MoE-16B: 16 x 128 MHA
        return cls(16, 16, 128, eps=1e-6, rope_theta=1e4)

    @classmethod
    def mixtral(cls) -> "DenseConfig":       # Mixtral-8x7B: 32 query heads, 8 K/V heads (GQA)
        return cls(32, 8, 128, eps=1e-5, rope_theta=1e6)


class DenseWeights:
    """Per layer: Wqkv [(nh + 2 nkv) hd, H] and Wo [H, nh hd] in bf16, the q/k/v
    bias, RMSNorm weight and shared-expert gate in fp32, drawn from a seeded CUDA
    generator (random init: no checkpoints in this environment)."""

    def __init__(self, cfg: ModelConfig, dc: DenseConfig, seed: int = 0, device=None, init_scale: float = 0.02):
        if dc.n_heads * dc.head_dim > 4 * cfg.hidden_dim or dc.n_heads % dc.n_kv_heads:
            raise InvalidConfig("dense geometry does not fit the model")
        self.cfg, self.dc = cfg, dc
        dev = device or torch.device("cuda", torch.cuda.current_device())
        H, nh, nkv, hd = cfg.hidden_dim, dc.n_heads, dc.n_kv_heads, dc.head_dim
        nq = (nh + 2 * nkv) * hd
        self.layers = []
        for l in range(cfg.num_layers):
            g = torch.Generator(device=dev).manual_seed(seed * 1_000_003 + 77_000_000 + l)
            r = lambda *s: torch.randn(*s, generator=g, device=dev)  # noqa: E731
            self.layers.append({
                "wqkv": (r(nq, H) * init_scale).to(torch.bfloat16),
                "bqkv": r(nq) * 0.1 if dc.qkv_bias else None,
                "norm": 1.0 + 0.1 * r(H),
                "wo": (r(H, nh * hd) * (init_scale / math.sqrt(cfg.num_layers))).to(torch.bfloat16),
                "shared_gate": r(H) * init_scale if dc.shared_gate else None,
            })

    def device_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for ly in self.layers for t in ly.values() if t is not None)
