"""GPU parity of the individual kernels against the CPU oracle (run with -m gpu).

K5 packing must be bit-exact; K1 ids/orders bit-exact; K3 within the stated
fp32 tolerance of the fp64 oracle on identical dequantized weights.
"""

import numpy as np
import pytest

from golden_util import golden, tiny_traces
from oracle import fate_oracle as O

pytestmark = pytest.mark.gpu

# K3 tolerance (fp32 accumulation vs the fp64 oracle on the same dequantized weights)
K3_REL_L2 = 2e-5
K3_MAX_ABS_REL = 1e-4


def _torch():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a visible CUDA device"
    return torch


def test_quant_pack_matches_reference_goldens():
    torch = _torch()
    from paper_2502_12224_b200 import ops
    for case in golden()["quant"]:
        x = torch.tensor(case["x"], dtype=torch.float64, device="cuda")
        codes, sz, s64, z64 = ops.quant_pack(x, case["bits"], want64=True)
        assert codes.cpu().numpy().tolist() == case["codes"]
        assert s64.cpu().numpy().tolist() == case["scales"]
        assert z64.cpu().numpy().tolist() == case["zeros"]


@pytest.mark.parametrize("bits", [8, 4, 2])
def test_quant_pack_fp32_random(bits):
    torch = _torch()
    from paper_2502_12224_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(bits)
    w = torch.randn((1408, 2048), generator=g, device="cuda") * 0.02
    w.view(-1)[1000:1200] = 0.5  # constant groups
    codes, sz, s64, z64 = ops.quant_pack(w, bits, want64=True)
    ref_codes, ref_s, ref_z = O.quantize(w.cpu().numpy().astype(np.float64), bits)
    np.testing.assert_array_equal(codes.cpu().numpy(), ref_codes)
    np.testing.assert_array_equal(s64.cpu().numpy(), ref_s)
    np.testing.assert_array_equal(z64.cpu().numpy(), ref_z)
    np.testing.assert_array_equal(sz.cpu().numpy()[:, 0], ref_s.astype(np.float32))
    np.testing.assert_array_equal(sz.cpu().numpy()[:, 1], ref_z.astype(np.float32))


@pytest.mark.parametrize("policy", ["topk", "percentile"])
def test_gate_ids_bit_exact_tiny(policy):
    _torch()
    from paper_2502_12224_b200 import ops
    tr = tiny_traces()
    W, taus, g = tr["gate_w"], tr["taus"], tr["dec_gate_in"]
    T, L, H = g.shape
    for l in range(L):
        routing, order, lens = ops.gate_predict(W[l], taus[l], g[:, l], 2, policy)
        order, lens = order.cpu().numpy(), lens.cpu().numpy()
        for t in range(T):
            w = O.gate_routing(W[l], taus[l], g[t, l])
            want = O.predicted_list(w, policy, 0.75, 2)
            assert order[t, :lens[t]].tolist() == want
            assert sorted(order[t, :2].tolist()) == tr["dec_chosen"][t, l].tolist()
        np.testing.assert_allclose(routing.cpu().numpy()[0], O.gate_routing(W[l], taus[l], g[0, l]), rtol=1e-13)


def _expert(torch, H, I, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn(s, generator=g, device="cuda") * 0.02 for s in ((I, H), (I, H), (H, I))]


@pytest.mark.parametrize("bits", [16, 8, 4, 2])
def test_pack_expert_layout(bits):
    torch = _torch()
    from paper_2502_12224_b200 import ops
    H, I = 256, 512
    w1, w3, w2 = _expert(torch, H, I, 3)
    buf = ops.pack_expert(w1, w3, w2, bits, layer=2, expert=5).cpu().numpy()
    assert buf.size - 256 == O.expert_bytes(3 * H * I, bits)
    u = O.unpack_buffer(buf, H, I, bits)
    assert u["header"] == {"bits": bits, "layer": 2, "expert": 5, "H": H, "I": I}
    for j, w in zip("132", (w1, w3, w2)):
        if bits == 16:
            np.testing.assert_array_equal(u["w" + j].astype(np.float32),
                                          w.cpu().to(torch.bfloat16).float().numpy())
        else:
            codes, s, z = O.quantize(w.cpu().numpy().astype(np.float64), bits)
            np.testing.assert_array_equal(u["codes" + j], codes)


@pytest.mark.parametrize("H,I,bits_list", [(256, 512, [4, 2]), (2048, 1408, [4, 4, 2, 4]), (2048, 1408, [16]),
                                            (4096, 1024, [8, 2]), (2048, 5632, [4, 2])])
def test_ffn_decode_numerics(H, I, bits_list):
    torch = _torch()
    from paper_2502_12224_b200 import ops
    bufs, ws, refs = [], [], []
    for j, b in enumerate(bits_list):
        w1, w3, w2 = _expert(torch, H, I, 100 + j)
        buf = ops.pack_expert(w1, w3, w2, b)
        bufs.append(buf)
        ws.append(0.1 + 0.2 * j)
        refs.append(O.unpack_buffer(buf.cpu().numpy(), H, I, b))
    x = (torch.randn(H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))).float()
    y = ops.ffn_decode(x, bufs, ws).cpu().numpy().astype(np.float64)
    xd = x.cpu().numpy().astype(np.float64)
    want = sum(w * O.ffn_swiglu(xd, r["w1"], r["w3"], r["w2"]) for w, r in zip(ws, refs))
    rel = np.linalg.norm(y - want) / np.linalg.norm(want)
    assert rel <= K3_REL_L2, rel
    assert np.max(np.abs(y - want)) <= K3_MAX_ABS_REL * np.max(np.abs(want))
