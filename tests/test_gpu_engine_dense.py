"""The engine with the dense part on: every decode step runs
the attention block and the shared-expert gate before the gate kernel.  The
schedule stays bit-exact against the reference (the dense part feeds the
residual stream, not the trace-driven router), the shared expert is weighted by
sigmoid(w . x), and the run reports the dense time it measured."""
import math

import numpy as np
import pytest

from golden_util import config_traces, golden
from oracle import fate_oracle as O

pytestmark = pytest.mark.gpu


def test_decode_with_dense_part_schedule_and_outputs():
    import torch
    from paper_2502_12224_b200.dense import DenseConfig, DenseWeights
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden()["schedules"]["tiny"]
    want = e["decode_cold"]
    cfg, dec, pre, w = config_traces("tiny")
    store = ExpertStore(cfg, bits=(4, 2), seed=0, shared_intermediate=512)
    eng = OffloadEngine(cfg, e["plan"], store, w, StrategyKnobs(budget_n=want["n"]), max_tokens=64)
    dc = DenseConfig(n_heads=4, n_kv_heads=2, head_dim=64, qkv_bias=True, shared_gate=True)
    dense = DenseWeights(cfg, dc, seed=0)
    T = 16
    eng.set_dense(dense, max_ctx=200 + T, ctx0=200)
    _, g, ch = dec.dense_arrays(cfg)
    res = eng.decode(torch.as_tensor(g[:T], device="cuda"), torch.as_tensor(ch[:T], device="cuda"), want_logs=True)
    for got, ref in zip(res.logs, want["steps"][:T * cfg.num_layers]):
        assert (got["chosen"], got.get("pred"), got["hits"], got["ondemand"], got["victims"]) == \
               (ref["chosen"], ref.get("pred"), ref["hits"], ref["ondemand"], ref["victims"])
    assert res.stats["dense_ms"] > 0 and res.stats["gpu_ms"] > res.stats["dense_ms"]
    # y of one step: routed experts + sigmoid(w_sg . x) * shared expert
    H, I = cfg.hidden_dim, cfg.intermediate_dim
    lg = res.logs[6]
    t, l = lg["token"], lg["layer"]
    x = (np.sqrt(H) * g[t, l]).astype(np.float32).astype(np.float64)
    r = O.gate_routing(w.matrices[l], w.temperatures[l], g[t, l])
    sh = O.unpack_buffer(store.shared_buffer(l).cpu().numpy(), H, 512, 16)
    sg = dense.layers[l]["shared_gate"].double().cpu().numpy()
    gate = 1.0 / (1.0 + math.exp(-float(sg @ (np.sqrt(H) * g[t, l]))))
    want_y = np.float32(gate) * O.ffn_swiglu(x, sh["w1"], sh["w3"], sh["w2"])
    for ex, b in zip(lg["chosen"], lg["fmt_bits"]):
        d = O.unpack_buffer(store.packed(l, ex, b).numpy(), H, I, b)
        want_y = want_y + np.float32(r[ex]) * O.ffn_swiglu(x, d["w1"], d["w3"], d["w2"])
    y = res.y[t, l].cpu().numpy().astype(np.float64)
    assert np.linalg.norm(y - want_y) / np.linalg.norm(want_y) < 2e-5
    eng.close()
