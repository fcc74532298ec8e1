"""The dense part of a decode step against a plain PyTorch
fp64 reference on the same bf16 weights and bf16 K/V cache: RMSNorm + QKV GEMV,
RoPE, K/V append, split-context decode attention (MHA and GQA), output
projection + residual, and the shared-expert gate.  fp32 accumulation:
rel-L2 <= 1e-4 per stage."""
import math

import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm())


@pytest.mark.parametrize("H,nh,nkv,hd,ctx0,bias,gate", [(2048, 16, 16, 128, 300, True, True),
                                                         (4096, 32, 8, 128, 70, False, False),
                                                         (256, 4, 2, 64, 1, True, False)])
def test_dense_step_matches_torch(H, nh, nkv, hd, ctx0, bias, gate):
    import torch
    from paper_2502_12224_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(H + nh)
    dev = "cuda"
    nq = (nh + 2 * nkv) * hd
    r = lambda *s: torch.randn(*s, generator=g, device=dev)  # noqa: E731
    layer = {"wqkv": (r(nq, H) * 0.02).to(torch.bfloat16), "wo": (r(H, nh * hd) * 0.02).to(torch.bfloat16),
             "norm": 1.0 + 0.1 * r(H), "bqkv": 0.1 * r(nq) if bias else None,
             "shared_gate": 0.02 * r(H) if gate else None}
    max_ctx = ctx0 + 4
    kv = (0.5 * r(max_ctx, 2, nkv * hd)).to(torch.bfloat16)
    kv0 = kv.clone()
    h_prev, y_prev = r(H), r(H) * 0.3
    gate_in = torch.randn(H, generator=g, device=dev, dtype=torch.float64) / math.sqrt(H)
    dims = {"H": H, "n_heads": nh, "n_kv_heads": nkv, "head_dim": hd, "eps": 1e-6, "rope_theta": 1e6}
    pos = ctx0
    out = ops.dense_step(dims, layer, kv, h_prev, y_prev, gate_in, pos)
    # ---- fp64 reference
    d = lambda t: t.double()  # noqa: E731
    h = d(h_prev) + d(y_prev)
    xn = h * torch.rsqrt((h * h).mean() + 1e-6) * d(layer["norm"])
    qkv = d(layer["wqkv"]) @ xn + (d(layer["bqkv"]) if bias else 0.0)
    assert _rel(out["h"], h) < 1e-6 and _rel(out["qkv"], qkv) < TOL
    q, k, v = qkv[:nh * hd].view(nh, hd), qkv[nh * hd:(nh + nkv) * hd].view(nkv, hd), qkv[(nh + nkv) * hd:].view(nkv, hd)
    half = hd // 2
    inv = torch.tensor([1e6 ** (-2.0 * i / hd) for i in range(half)], dtype=torch.float64, device=dev)
    ang = pos * inv
    cs, sn = torch.cos(ang), torch.sin(ang)

    def rope(x):
        x0, x1 = x[:, :half], x[:, half:]
        return torch.cat([x0 * cs - x1 * sn, x1 * cs + x0 * sn], dim=1)
    qr, kr = rope(q), rope(k)
    assert _rel(out["q"], qr.reshape(-1)) < TOL
    # the appended K/V row is the bf16 rounding of the roped k and of v; earlier rows untouched
    assert torch.equal(kv[:pos], kv0[:pos])
    assert _rel(kv[pos, 0].float(), kr.reshape(-1)) < 1e-2 and _rel(kv[pos, 1].float(), v.reshape(-1)) < 1e-2
    K = d(kv[:pos + 1, 0]).view(pos + 1, nkv, hd)
    V = d(kv[:pos + 1, 1]).view(pos + 1, nkv, hd)
    grp = nh // nkv
    o = torch.empty(nh, hd, dtype=torch.float64, device=dev)
    for hh in range(nh):
        s = (K[:, hh // grp] @ qr[hh]) / math.sqrt(hd)
        o[hh] = torch.softmax(s, 0) @ V[:, hh // grp]
    assert _rel(out["o"], o.reshape(-1)) < TOL
    a = h + d(layer["wo"]) @ o.reshape(-1)
    assert _rel(out["a"], a) < TOL
    if gate:
        sg = torch.sigmoid((d(layer["shared_gate"]) * (math.sqrt(H) * gate_in)).sum())
        assert abs(float(out["gate"][0]) - float(sg)) < 1e-5
