"""Prefill engine parity (run with -m gpu).

Which of a layer's prefetches had started by its block end is timing
dependent (pipeline.py:682); the engine reports that set per layer, and
every other field must then match the oracle bit for bit: prediction
profile and order, INT2/INT4 bit map, prefetch list, actives and counts,
resident set, on-demand order, ARC victims, final ARC state, recall and
dequant_count.  Expert outputs are checked against the fp64 oracle.
"""

import numpy as np
import pytest

from golden_util import config_traces, golden
from oracle import fate_oracle as O

pytestmark = pytest.mark.gpu

# K4 runs on tcgen05 with bf16 operands (token rows and dequantized weights
# rounded to bf16) and fp32 accumulation: stated tolerance against the fp64
# oracle on the same packed weights.
Y_REL_L2 = 1e-2


def _setup(name, shared=0, n=15):
    import torch
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden()["schedules"][name]
    cfg, dec, pre, w = config_traces(name)
    store = ExpertStore(cfg, bits=(4, 2), seed=0, shared_intermediate=shared)
    eng = OffloadEngine(cfg, e["plan"], store, w, StrategyKnobs(budget_n=n), max_tokens=max(64, pre.num_tokens))
    return cfg, dec, pre, w, store, eng, e


def _check_prefill(logs, oracle):
    for l, (g, o) in enumerate(zip(logs, oracle["layers"])):
        assert g["mismatch"] == 0, l
        if "pred_order" in o:
            assert g["pred_order"] == o["pred_order"], l
            assert g["pred_counts"] == o["pred_counts"], l
            assert [tuple(x) for x in g["prefetch"]] == [tuple(x) for x in o["prefetch"]], l
        assert g["actives"] == o["actives"], l
        assert g["counts"] == o["counts"], l
        assert g["resident"] == o["resident"], l
        assert sorted(g["planned"]) == sorted(o["planned"]), l
        assert g["ondemand"] == o["ondemand"], l
        assert g["src_bits"] == o["src_bits"], l
        assert g["victims"] == o["victims"], l


@pytest.mark.parametrize("name", ["tiny", "dsk"])
def test_prefill_then_decode_chain(name):
    import torch
    cfg, dec, pre, w, store, eng, e = _setup(name)
    mats, taus = np.stack(w.matrices), np.array(w.temperatures)
    _, gp, chp = pre.dense_arrays(cfg)
    Y, st, logs, step_ms, copies = eng.prefill(torch.as_tensor(gp, device="cuda"), torch.as_tensor(chp, device="cuda"))
    started = {l: set(lg["started"]) for l, lg in enumerate(logs)}
    arcs = [O.Arc(c) for c in e["plan"]]
    ora = O.prefill_schedule(gp, chp.tolist(), mats, taus, e["plan"], cfg.top_k, O.StrategyKnobs(), 4,
                             started=started, arcs=arcs)
    _check_prefill(logs, ora)
    for l in range(cfg.num_layers):
        assert eng.arc_state(l) == ora["arcs"][l]
    assert st["recall_sum"] / st["recall_n"] == pytest.approx(ora["recall"], abs=1e-12)
    assert st["dequant_count"] == ora["dequant_count"]
    assert st["trace_mismatches"] == 0
    # decode continues on the prefill-warmed cache (pipeline.py:835-850)
    _, gd, chd = dec.dense_arrays(cfg)
    n = golden()["schedules"][name]["decode_warm"]["n"]
    res = eng.decode(torch.as_tensor(gd, device="cuda"), torch.as_tensor(chd, device="cuda"), want_logs=True)
    ord_ = O.decode_schedule(gd, chd.tolist(), mats, taus, e["plan"], cfg.top_k, n, O.StrategyKnobs(), 4, arcs=arcs)
    for g, o in zip(res.logs, ord_["steps"]):
        assert (g["chosen"], g.get("pred"), g.get("prefetch"), g["hits"], g["ondemand"], g["victims"]) == \
               (o["chosen"], o.get("pred"), o.get("prefetch"), o["hits"], o["ondemand"], o["victims"])
    for l in range(cfg.num_layers):
        assert eng.arc_state(l) == ord_["arcs"][l]
    eng.close()


@pytest.mark.parametrize("name", ["tiny", "qwen"])
def test_eap_prefill_then_decode_chain(name):
    """EAP baseline through prefill and the chained decode (pipeline.py:828-849):
    the co-activation statistics the prefill accumulates on the device carry
    into the decode; both phases bit-exact against the oracle given the
    measured started sets, and the decode against the reference's own log
    when every prefetch had started (as in the reference's timeline)."""
    import torch
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden()["schedules"][name]
    cfg, dec, pre, w = config_traces(name)
    n = e["decode_eap_warm"]["n"]
    kn = StrategyKnobs(budget_n=n, policy="eap", prefetch_bits=16, ondemand_bits=16, cached_bits=4,
                       prefill_ondemand_bits=16, reorder_prefill=False, p_int2=0.0)
    store = ExpertStore(cfg, bits=(16, 4), seed=0)
    eng = OffloadEngine(cfg, e["plan"], store, w, kn, max_tokens=max(64, pre.num_tokens))
    eng.reset_eap()
    mats, taus = np.stack(w.matrices), np.array(w.temperatures)
    _, gp, chp = pre.dense_arrays(cfg)
    Y, st, logs, step_ms, copies = eng.prefill(torch.as_tensor(gp, device="cuda"), torch.as_tensor(chp, device="cuda"))
    started = {l: set(lg["started"]) for l, lg in enumerate(logs)}
    arcs = [O.Arc(c) for c in e["plan"]]
    kno = O.StrategyKnobs(kind="eap", quant=False, policy_kind="topk", reorder_prefill=False)
    counts = np.zeros((cfg.num_layers - 1, cfg.num_experts, cfg.num_experts), dtype=np.int64)
    ora = O.prefill_schedule(gp, chp.tolist(), mats, taus, e["plan"], cfg.top_k, kno, 4, started=started, arcs=arcs,
                             eap_counts=counts)
    _check_prefill(logs, ora)
    for l in range(cfg.num_layers):
        assert eng.arc_state(l) == ora["arcs"][l]
    assert st["dequant_count"] == ora["dequant_count"]
    assert st["trace_mismatches"] == 0
    _, gd, chd = dec.dense_arrays(cfg)
    res = eng.decode(torch.as_tensor(gd, device="cuda"), torch.as_tensor(chd, device="cuda"), want_logs=True)
    ord_ = O.decode_schedule(gd, chd.tolist(), mats, taus, e["plan"], cfg.top_k, n, kno, 4, arcs=arcs,
                             eap_counts=counts)
    for g, o in zip(res.logs, ord_["steps"]):
        assert (g["chosen"], g.get("pred"), g.get("prefetch"), g["hits"], g["ondemand"], g["victims"]) == \
               (o["chosen"], o.get("pred"), o.get("prefetch"), o["hits"], o["ondemand"], o["victims"])
    for l in range(cfg.num_layers):
        assert eng.arc_state(l) == ord_["arcs"][l]
    want_started = {l: set(x["started"]) for l, x in enumerate(e["prefill_eap"]["layers"])}
    if started == want_started:
        want = e["decode_eap_warm"]
        for g, wst in zip(res.logs, want["steps"]):
            assert (g.get("pred"), g.get("prefetch"), g["hits"], g["ondemand"], g["victims"]) == \
                   (wst.get("pred"), wst.get("prefetch"), wst["hits"], wst["ondemand"], wst["victims"])
    eng.close()


def test_prefill_outputs_match_fp64_oracle():
    import torch
    cfg, dec, pre, w, store, eng, e = _setup("tiny", shared=512)
    _, gp, chp = pre.dense_arrays(cfg)
    Y, st, logs, _, _ = eng.prefill(torch.as_tensor(gp, device="cuda"), torch.as_tensor(chp, device="cuda"))
    Y = Y.cpu().numpy().astype(np.float64)
    H, I = cfg.hidden_dim, cfg.intermediate_dim
    worst = 0.0
    for l, lg in enumerate(logs):
        assert lg["resident"] == []  # cold cache: every layer's data came over the channel
        bits_of = dict(zip(lg["actives"], lg["src_bits"]))
        sh = O.unpack_buffer(store.shared_buffer(l).cpu().numpy(), H, 512, 16)
        deq = {a: O.unpack_buffer(store.packed(l, a, bits_of[a]).numpy(), H, I, bits_of[a]) for a in lg["actives"]}
        for t in range(gp.shape[0]):
            x = (np.sqrt(H) * gp[t, l]).astype(np.float32).astype(np.float64)
            r = O.gate_routing(w.matrices[l], w.temperatures[l], gp[t, l])
            want = O.ffn_swiglu(x, sh["w1"], sh["w3"], sh["w2"])
            for a in chp[t, l]:
                d = deq[int(a)]
                want = want + np.float32(r[a]) * O.ffn_swiglu(x, d["w1"], d["w3"], d["w2"])
            worst = max(worst, np.linalg.norm(Y[l, t] - want) / np.linalg.norm(want))
    print(f"prefill Y worst rel-L2 vs fp64 oracle: {worst:.3e}")
    assert worst <= Y_REL_L2, worst
    eng.close()


def test_ffn_prefill_standalone():
    import torch
    from paper_2502_12224_b200 import ops
    H, I = 256, 512
    g = torch.Generator(device="cuda").manual_seed(5)
    bufs, refs = [], []
    for j, b in enumerate((4, 2, 16)):
        ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in ((I, H), (I, H), (H, I))]
        buf = ops.pack_expert(*ws, b)
        bufs.append(buf)
        refs.append(O.unpack_buffer(buf.cpu().numpy(), H, I, b))
    X = torch.randn((40, H), generator=g, device="cuda")
    toks = [[0, 3, 5, 39], list(range(0, 40, 2)), [7]]
    wts = [[0.5, 0.25, 1.0, 2.0], [0.1] * 20, [3.0]]
    Y = ops.ffn_prefill(X, bufs, toks, wts).cpu().numpy()
    Xd = X.cpu().numpy().astype(np.float64)
    want = np.zeros((40, H))
    for r, tl, wl in zip(refs, toks, wts):
        for t, wv in zip(tl, wl):
            want[t] += wv * O.ffn_swiglu(Xd[t], r["w1"], r["w3"], r["w2"])
    rel = np.linalg.norm(Y - want) / np.linalg.norm(want)
    print(f"ffn_prefill rel-L2 vs fp64 oracle: {rel:.3e}")
    assert rel <= Y_REL_L2, rel


def test_ffn_prefill_qwen_shape_multi_tile():
    # Qwen expert geometry, token lists longer than one 128-token tile, mixed widths
    import torch
    from paper_2502_12224_b200 import ops
    H, I = 2048, 1408
    g = torch.Generator(device="cuda").manual_seed(11)
    bufs, refs = [], []
    for b in (4, 2, 16, 8):
        ws = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in ((I, H), (I, H), (H, I))]
        buf = ops.pack_expert(*ws, b)
        bufs.append(buf)
        refs.append(O.unpack_buffer(buf.cpu().numpy(), H, I, b))
    T = 300
    X = torch.randn((T, H), generator=g, device="cuda")
    rng = np.random.default_rng(3)
    toks = [sorted(rng.choice(T, size=n, replace=False).tolist()) for n in (300, 130, 17, 1)]
    wts = [rng.uniform(0.05, 1.0, size=len(tl)).tolist() for tl in toks]
    Y = ops.ffn_prefill(X, bufs, toks, wts).cpu().numpy().astype(np.float64)
    Xd = X.cpu().numpy().astype(np.float64)
    want = np.zeros((T, H))
    for r, tl, wl in zip(refs, toks, wts):
        h1, h3 = Xd[tl] @ r["w1"].T, Xd[tl] @ r["w3"].T
        a = h1 / (1.0 + np.exp(-h1)) * h3
        want[tl] += np.asarray(wl)[:, None] * (a @ r["w2"].T)
    rel = np.linalg.norm(Y - want) / np.linalg.norm(want)
    print(f"ffn_prefill qwen-shape rel-L2 vs fp64 oracle: {rel:.3e}")
    assert rel <= Y_REL_L2, rel
    # every listed token row got its contribution (no dropped tiles)
    row_rel = np.linalg.norm(Y - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-30)
    assert row_rel.max() <= 5 * Y_REL_L2, row_rel.max()
