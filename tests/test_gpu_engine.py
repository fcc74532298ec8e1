"""End-to-end parity of the device engine against the oracle (run with -m gpu).

Timing-independent fields of every decode step must be bit-exact: chosen
ids, predicted list entries[:n], prefetch-issued set, cache-hit flags,
on-demand set, ARC victims, source bits, final ARC state, recall and
dequant_count.  Expert outputs are checked against the fp64 oracle on the
same dequantized copies the GPU used (source bits per step).
"""

import numpy as np
import pytest

from golden_util import config_traces, golden, tiny_traces
from oracle import fate_oracle as O

pytestmark = pytest.mark.gpu

Y_REL_L2 = 2e-5


def _engine(name, n, knobs_kw=None, bits=(4, 2), shared=0, max_tokens=128):
    import torch
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden()["schedules"][name]
    cfg, dec, pre, w = config_traces(name)
    store = ExpertStore(cfg, bits=bits, seed=0, shared_intermediate=shared)
    kn = StrategyKnobs(budget_n=n, **(knobs_kw or {}))
    eng = OffloadEngine(cfg, e["plan"], store, w, kn, max_tokens=max_tokens)
    return cfg, dec, pre, w, store, eng


def _dev_trace(trace, cfg):
    import torch
    toks, g, ch = trace.dense_arrays(cfg)
    return torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda"), g, ch


def _compare_steps(logs, want, n_pred_layers=True):
    assert len(logs) == len(want["steps"])
    for g, w in zip(logs, want["steps"]):
        key = (g["token"], g["layer"])
        assert g["mismatch"] == 0, key
        assert g["chosen"] == w["chosen"], key
        assert g.get("pred") == w.get("pred"), key
        assert g.get("prefetch") == w.get("prefetch"), key
        assert g["hits"] == w["hits"], key
        assert g["ondemand"] == w["ondemand"], key
        assert g["victims"] == w["victims"], key
        if "src_bits" in w:
            assert g["src_bits"] == w["src_bits"], key


@pytest.mark.parametrize("name", ["tiny", "qwen", "mixtral"])
def test_decode_schedule_bit_exact(name):
    cfg, dec, pre, w, store, eng = _engine(name, n=15)
    gd, chd, g, ch = _dev_trace(dec, cfg)
    res = eng.decode(gd, chd, want_logs=True)
    want = golden()["schedules"][name]["decode_cold"]
    oracle = O.decode_schedule(g, ch.tolist(), np.stack(w.matrices), np.array(w.temperatures), golden()["schedules"][name]["plan"],
                               cfg.top_k, want["n"], O.StrategyKnobs(), 4)
    _compare_steps(res.logs, oracle)
    _compare_steps(res.logs, want)  # and directly against the reference's own log
    for l in range(cfg.num_layers):
        assert eng.arc_state(l) == want["arcs"][l]
    st = res.stats
    assert st["trace_mismatches"] == 0
    assert st["dequant_count"] == want["report"]["dequant_count"]
    assert st["recall_sum"] / st["recall_n"] == pytest.approx(want["report"]["recall"], abs=1e-12)
    assert st["prefetch_issued"] == want["transfers"]["prefetch"]
    assert st["ondemand_issued"] == want["transfers"]["ondemand"]
    assert st["cache_hits"] == sum(len(s["hits"]) for s in want["steps"])
    eng.close()


def test_decode_n0_and_topk_variants():
    e = golden()["schedules"]["tiny"]
    for variant, kw in (("decode_cold_n0", {}), ("decode_cold_topk", {"policy": "topk"})):
        want = e[variant]
        cfg, dec, pre, w, store, eng = _engine("tiny", n=want["n"], knobs_kw=kw)
        gd, chd, g, ch = _dev_trace(dec, cfg)
        res = eng.decode(gd, chd, want_logs=True)
        _compare_steps(res.logs, want)
        for l in range(cfg.num_layers):
            assert eng.arc_state(l) == want["arcs"][l]
        eng.close()


@pytest.mark.parametrize("name", ["tiny", "qwen"])
def test_decode_eap_baseline(name):
    """EAP baseline (pipeline.py:301-321) in K1: co-activation observe + scored
    top-k prediction, 16-bit prefetch / on-demand, against the oracle and the
    reference's own EAP log."""
    e = golden()["schedules"][name]
    want = e["decode_eap"]
    kw = {"policy": "eap", "prefetch_bits": 16, "ondemand_bits": 16, "cached_bits": 4,
          "prefill_use_predictor": False}
    cfg, dec, pre, w, store, eng = _engine(name, n=want["n"], knobs_kw=kw, bits=(16, 4))
    gd, chd, g, ch = _dev_trace(dec, cfg)
    res = eng.decode(gd, chd, want_logs=True)
    oracle = O.decode_schedule(g, ch.tolist(), np.stack(w.matrices), np.array(w.temperatures), e["plan"],
                               cfg.top_k, want["n"], O.StrategyKnobs(kind="eap", quant=False, policy_kind="topk"), 4)
    _compare_steps(res.logs, oracle)
    _compare_steps(res.logs, want)
    for l in range(cfg.num_layers):
        assert eng.arc_state(l) == want["arcs"][l]
    st = res.stats
    assert st["dequant_count"] == want["report"]["dequant_count"]
    assert st["recall_sum"] / st["recall_n"] == pytest.approx(want["report"]["recall"], abs=1e-12)
    assert st["prefetch_issued"] == want["transfers"]["prefetch"]
    assert st["ondemand_issued"] == want["transfers"]["ondemand"]
    eng.close()


def test_simulate_decoding_eap_public_api():
    """The drop-in call a moesim user makes: pipeline.simulate_decoding with
    Strategy.eap() reproduces the reference's timing-independent report fields."""
    from golden_util import PAPER_TIMING
    from paper_2502_12224_b200 import cache, core, pipeline
    e = golden()["schedules"]["tiny"]
    want = e["decode_eap"]["report"]
    cfg, dec, pre, w = config_traces("tiny")
    budget = cfg.dense_bytes + 12 * cfg.expert_bytes[4]
    plan = cache.plan_allocation(cfg, budget, 4)
    assert list(plan.per_layer_capacity) == e["plan"]
    tl, rep = pipeline.simulate_decoding(dec, pipeline.Strategy.eap(), plan, core.TimingModel(**PAPER_TIMING), cfg,
                                         weights=w)
    assert rep.strategy == "eap"
    assert rep.dequant_count == want["dequant_count"]
    assert rep.recall == pytest.approx(want["recall"], abs=1e-12)


def test_compare_strategies_fate_eap_lod():
    """The reference harness call (pipeline.py:802-851) on the GPU engine: per
    strategy a prefill on a fresh cache, then decode on the warmed one; EAP's
    statistics carry from its prefill into its decode.  Recall is timing-
    independent, so it must equal the reference's chained decode."""
    from golden_util import PAPER_TIMING
    from paper_2502_12224_b200 import core, pipeline
    e = golden()["schedules"]["tiny"]
    cfg, dec, pre, w = config_traces("tiny")
    budget = cfg.dense_bytes + 12 * cfg.expert_bytes[4]
    strategies = [pipeline.Strategy.fate(), pipeline.Strategy.eap(), pipeline.Strategy.lod()]
    rows = pipeline.compare_strategies(cfg, core.TimingModel(**PAPER_TIMING), strategies, [budget], pre, dec, weights=w)
    got = {(r.strategy, r.phase): r.report for r in rows}
    assert set(got) == {(k, ph) for k in ("fate", "eap", "lod") for ph in ("prefill", "decoding")}
    assert got[("fate", "decoding")].recall == pytest.approx(e["decode_warm"]["report"]["recall"], abs=1e-12)
    assert got[("eap", "decoding")].recall == pytest.approx(e["decode_eap_warm"]["report"]["recall"], abs=1e-12)
    assert got[("lod", "decoding")].recall == 0.0


def test_decode_outputs_match_fp64_oracle():
    """y[t, l] = sum_e w_e FFN_e(sqrt(H) * gate_in) with each expert dequantized
    from the copy the GPU actually used (src_bits), plus the shared expert."""
    cfg, dec, pre, w, store, eng = _engine("tiny", n=15, shared=512)
    gd, chd, g, ch = _dev_trace(dec, cfg)
    res = eng.decode(gd, chd, want_logs=True)
    y = res.y.cpu().numpy().astype(np.float64)
    H, I = cfg.hidden_dim, cfg.intermediate_dim
    cache = {}

    def deq(l, e, bits):
        if (l, e, bits) not in cache:
            cache[(l, e, bits)] = O.unpack_buffer(store.packed(l, e, bits).numpy(), H, I, bits)
        return cache[(l, e, bits)]

    shared = [O.unpack_buffer(store.shared_buffer(l).cpu().numpy(), H, 512, 16) for l in range(cfg.num_layers)]
    worst = 0.0
    for s, lg in enumerate(res.logs[:64]):
        t, l = lg["token"], lg["layer"]
        x = (np.sqrt(H) * g[t, l]).astype(np.float32).astype(np.float64)
        r = O.gate_routing(w.matrices[l], w.temperatures[l], g[t, l])
        want = O.ffn_swiglu(x, shared[l]["w1"], shared[l]["w3"], shared[l]["w2"])
        for e, bits in zip(lg["chosen"], lg["fmt_bits"]):
            # a slot filled by an INT2 on-demand load stays INT2 (tagged slot bits)
            d = deq(l, e, bits)
            want = want + np.float32(r[e]) * O.ffn_swiglu(x, d["w1"], d["w3"], d["w2"])
        got = y[t, l]
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        worst = max(worst, rel)
    assert worst <= Y_REL_L2, worst
    eng.close()


@pytest.mark.parametrize("name", ["tiny", "qwen"])
def test_expert_sharded_sources_same_decisions_and_outputs(name):
    # expert-sharded peer-fetch mode with one rank: every expert is
    # homed on this GPU, so misses are HBM-to-HBM copies instead of host fetches;
    # every trace decision and every output must be identical to the host run
    import torch
    from paper_2502_12224_b200.replicas import ExpertShards
    cfg, dec, pre, w, store, eng = _engine(name, n=15, shared=0)
    gd, chd, g, ch = _dev_trace(dec, cfg)
    T = min(gd.shape[0], 16)
    ref = eng.decode(gd[:T], chd[:T], want_logs=True)
    ref_arcs = [eng.arc_state(l) for l in range(cfg.num_layers)]
    shards = ExpertShards(store, bits=(4, 2), rank=0, world_size=1)
    assert shards.device_bytes == sum(store.host_pool(b).numel() for b in (4, 2))
    eng.reset_cache()
    shards.attach(eng)
    got = eng.decode(gd[:T], chd[:T], want_logs=True)
    # every byte now comes from device memory; how many queued prefetches were
    # dropped as stale before starting is timing dependent (pipeline.py:247-253)
    assert got.stats["h2d_bytes"] == 0 and got.stats["d2d_bytes"] > 0
    assert got.stats["ondemand_issued"] == ref.stats["ondemand_issued"]
    assert got.stats["prefetch_issued"] == ref.stats["prefetch_issued"]
    for a, b in zip(got.logs, ref.logs):
        assert (a["chosen"], a.get("pred"), a.get("prefetch"), a["hits"], a["ondemand"], a["victims"]) == \
               (b["chosen"], b.get("pred"), b.get("prefetch"), b["hits"], b["ondemand"], b["victims"])
    assert torch.equal(got.y, ref.y)
    assert [eng.arc_state(l) for l in range(cfg.num_layers)] == ref_arcs
    shards.detach(eng)
    eng.reset_cache()
    back = eng.decode(gd[:T], chd[:T])
    assert back.stats["d2d_bytes"] == 0 and back.stats["h2d_bytes"] > 0
    shards.close()
    eng.close()


@pytest.mark.parametrize("name,n", [("qwen", 15), ("qwen", 0), ("mixtral", 15)])
def test_arrival_gated_k3_same_decisions_and_outputs(name, n):
    # the default decode protocol launches K3 right behind K1 and gates each
    # expert on its copy's generation mark; the stream-wait protocol starts K3
    # once every copy of the step landed.  Decisions, ARC state and every output
    # bit must be identical (prefetched experts still in flight included, n = 15)
    import torch
    cfg, dec, pre, w, store, eng = _engine(name, n=n, shared=512 if name == "qwen" else 0)
    gd, chd, g, ch = _dev_trace(dec, cfg)
    T = min(gd.shape[0], 24)
    eng.set_overlap(False)
    ref = eng.decode(gd[:T], chd[:T], want_logs=True)
    ref_arcs = [eng.arc_state(l) for l in range(cfg.num_layers)]
    assert ref.stats["k3_wait_ms"] == 0.0
    eng.set_overlap(True)
    eng.reset_cache()
    got = eng.decode(gd[:T], chd[:T], want_logs=True)
    for a, b in zip(got.logs, ref.logs):
        assert (a["chosen"], a.get("pred"), a.get("prefetch"), a["hits"], a["ondemand"], a["victims"],
                a["src_bits"]) == \
               (b["chosen"], b.get("pred"), b.get("prefetch"), b["hits"], b["ondemand"], b["victims"], b["src_bits"])
    assert torch.equal(got.y, ref.y)
    assert [eng.arc_state(l) for l in range(cfg.num_layers)] == ref_arcs
    assert got.stats["ondemand_issued"] > 0 and got.stats["k3_wait_ms"] > 0.0
    eng.close()
