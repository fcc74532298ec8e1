"""Pin the CPU oracle (oracle/fate_oracle.py) to the reference's own outputs.

Every vector here was produced by running the reference ``moesim`` package
(tests/golden/make_golden.py).  If these pass, the oracle is a faithful
restatement and can be trusted as the checker for the GPU path.
"""

import numpy as np
import pytest

from golden_util import PAPER_TIMING, config_traces, golden, tiny_traces
from oracle import fate_oracle as O


def test_spec_known_answers():
    k = golden()["kat"]
    np.testing.assert_array_equal(O.softmax64(np.array([2.0, 1.0, 0.0, -1.0])), np.array(k["softmax"]))
    w = np.array(k["percentile_60"]["w"])
    assert O.nearest_rank_threshold(w, 0.75) == k["percentile_60"]["thr"]
    assert O.predicted_list(w, "percentile", 0.75, 4) == k["percentile_60"]["list"]
    assert len(k["percentile_60"]["list"]) == 15
    assert O.plan_capacities(24, 60, 3, 300) == k["plan_300"]
    assert O.plan_capacities(24, 60, 3, 100) == k["plan_100"]
    assert O.plan_capacities(24, 60, 3, 1500) == k["plan_1500"]
    for c, seq, key in ((2, [0, 1, 0, 2, 0], "arc_c2"), (1, [0, 0], "arc_c1")):
        a = O.Arc(c)
        assert [a.access(x)[0] for x in seq] == k[key]
    codes, sc, zr = O.quantize(np.array([0.0, 1.0, 2.0, 3.0]), 2, group=4)
    assert codes.tolist() == k["quant_2bit"]["codes"] == [228]
    codes, sc, zr = O.quantize(np.full(10, 0.37), 4, group=4)
    assert codes.tolist() == k["quant_const"]["codes"]
    np.testing.assert_array_equal(O.dequantize(codes, sc, zr, 4, (10,), group=4), k["quant_const"]["deq"])
    assert O.pack_codes(np.arange(16, dtype=np.uint8), 4).tolist() == k["pack4_0_15"]
    assert O.transfer_budget(13, 9, 2, 6) == k["transfer_budget"] == 4
    assert O.transfer_budget(13, 9, 2, 1.6) == k["transfer_budget_paper"]
    bits = O.assign_bits_prefill(list(range(8)), 0.25)
    assert {str(e): b for e, b in bits.items()} == k["assign_bits_8"]
    counts, order = O.popularity([[1, 2]] * 3)
    assert {str(e): c for e, c in counts.items()} == k["prefill_merge"]["counts"]
    assert order == k["prefill_merge"]["ordering"]
    assert sorted(O.top_k(np.full(5, 0.2), 2)) == k["topk_ties"]


def test_quantize_byte_exact():
    for case in golden()["quant"]:
        x = np.array(case["x"]).reshape(case["shape"])
        codes, sc, zr = O.quantize(x, case["bits"])
        assert codes.tolist() == case["codes"]
        assert sc.tolist() == case["scales"]
        assert zr.tolist() == case["zeros"]
        deq = O.dequantize(codes, sc, zr, case["bits"], x.shape)
        assert np.all(np.abs(deq - x) <= np.repeat(sc, 64)[: x.size].reshape(x.shape) / 2 + 1e-15)


def test_arc_sequences():
    for case in golden()["arc"]:
        a = O.Arc(case["c"])
        hits = [a.access(x)[0] for x in case["seq"]]
        assert hits == case["hits"]
        f = case["final"]
        assert (a.t1, a.t2, a.b1, a.b2, a.p) == (f["t1"], f["t2"], f["b1"], f["b2"], f["p"])


def _knobs(**kw):
    return O.StrategyKnobs(**kw)


def _check_decode(got, want):
    assert len(got["steps"]) == len(want["steps"])
    for g, w in zip(got["steps"], want["steps"]):
        assert g["chosen"] == w["chosen"]
        assert g.get("pred") == w.get("pred"), (g["token"], g["layer"])
        assert g.get("prefetch") == w.get("prefetch"), (g["token"], g["layer"])
        assert g["ondemand"] == w["ondemand"], (g["token"], g["layer"])
        assert g["hits"] == w["hits"], (g["token"], g["layer"])
        assert g["victims"] == w["victims"], (g["token"], g["layer"])
    assert got["arcs"] == want["arcs"]
    assert got["recall"] == pytest.approx(want["report"]["recall"], abs=1e-12)
    assert got["dequant_count"] == want["report"]["dequant_count"]
    n_pref = sum(len(s.get("prefetch", [])) for s in got["steps"])
    n_od = sum(len(s["ondemand"]) for s in got["steps"])
    assert (n_pref, n_od) == (want["transfers"]["prefetch"], want["transfers"]["ondemand"])


def _arrays(trace, cfg):
    _, g, ch = trace.dense_arrays(cfg)
    return g, ch.tolist()


@pytest.mark.parametrize("variant", ["decode_cold", "decode_cold_n0", "decode_cold_topk", "decode_lod", "decode_eap"])
def test_tiny_decode_schedule(variant):
    e = golden()["schedules"]["tiny"]
    tr = tiny_traces()
    mats, taus = tr["gate_w"], tr["taus"]
    want = e[variant]
    kind = {"decode_lod": "lod", "decode_eap": "eap"}.get(variant, "fate")
    knobs = _knobs(kind=kind, quant=kind == "fate",
                   policy_kind="topk" if variant.endswith("topk") or kind == "eap" else "percentile")
    caps = [0] * 4 if kind == "lod" else e["plan"]
    got = O.decode_schedule(tr["dec_gate_in"], tr["dec_chosen"].tolist(), mats, taus, caps, 2, want["n"],
                            knobs, 16 if kind == "lod" else 4)
    _check_decode(got, want)


def test_qwen_eap_decode_schedule():
    """EAP baseline (pipeline.py:301-321) on the Qwen shape: co-activation stats
    accumulate over tokens, so later steps exercise the scored (non-cold) path."""
    from golden_util import config_traces
    e = golden()["schedules"]["qwen"]
    want = e["decode_eap"]
    cfg, dec, pre, w = config_traces("qwen")
    g, ch = _arrays(dec, cfg)
    got = O.decode_schedule(g, ch, np.stack(w.matrices), np.array(w.temperatures), e["plan"], cfg.top_k, want["n"],
                            _knobs(kind="eap", quant=False, policy_kind="topk"), 4)
    _check_decode(got, want)


def test_tiny_canary_values():
    """SURVEY §8c drift canaries, measured with the reference."""
    d = golden()["schedules"]["tiny"]["decode_cold"]
    assert d["steps"][0]["chosen"] == [2, 6]
    assert d["transfers"] == {"prefetch": 334, "ondemand": 142}
    assert d["report"]["dequant_count"] == 512
    assert abs(d["report"]["hit_rate"] - 0.722656) < 1e-6


def _check_prefill(got, want):
    for g, w in zip(got["layers"], want["layers"]):
        assert [list(x) for x in g.get("prefetch", [])] == w["prefetch_for_next"], g["layer"]
        assert [[e, 2] for e in g["ondemand"]] == w["ondemand"], g["layer"]
        assert g["victims"] == w["victims"], g["layer"]
    assert got["arcs"] == want["arcs"]
    assert got["recall"] == pytest.approx(want["report"]["recall"], abs=1e-12)
    assert got["dequant_count"] == want["report"]["dequant_count"]


@pytest.mark.parametrize("name", ["tiny", "qwen", "dsk", "mixtral"])
def test_prefill_then_decode_schedule(name):
    """compare_strategies chaining: prefill on a cold cache, decode on the warmed one."""
    e = golden()["schedules"][name]
    cfg, dec, pre, w = config_traces(name)
    mats, taus = np.stack(w.matrices), np.array(w.temperatures)
    arcs = [O.Arc(c) for c in e["plan"]]
    want = e["prefill_cold"]
    started = {l: set(x["started"]) for l, x in enumerate(want["layers"])}
    gp, chp = _arrays(pre, cfg)
    got = O.prefill_schedule(gp, chp, mats, taus, e["plan"], cfg.top_k, _knobs(), 4, started=started, arcs=arcs)
    _check_prefill(got, want)
    gd, chd = _arrays(dec, cfg)
    wd = e["decode_warm"]
    got = O.decode_schedule(gd, chd, mats, taus, e["plan"], cfg.top_k, wd["n"], _knobs(), 4, arcs=arcs)
    _check_decode(got, wd)


@pytest.mark.parametrize("name", ["tiny", "qwen"])
def test_eap_prefill_then_decode_schedule(name):
    """EAP chaining (pipeline.py:828-849): prefill and decode share one EapStats."""
    e = golden()["schedules"][name]
    cfg, dec, pre, w = config_traces(name)
    mats, taus = np.stack(w.matrices), np.array(w.temperatures)
    arcs = [O.Arc(c) for c in e["plan"]]
    kn = _knobs(kind="eap", quant=False, policy_kind="topk", reorder_prefill=False)
    counts = np.zeros((cfg.num_layers - 1, cfg.num_experts, cfg.num_experts), dtype=np.int64)
    want = e["prefill_eap"]
    started = {l: set(x["started"]) for l, x in enumerate(want["layers"])}
    gp, chp = _arrays(pre, cfg)
    got = O.prefill_schedule(gp, chp, mats, taus, e["plan"], cfg.top_k, kn, 4, started=started, arcs=arcs,
                             eap_counts=counts)
    for g, wl in zip(got["layers"], want["layers"]):
        assert [list(x) for x in g.get("prefetch", [])] == wl["prefetch_for_next"], g["layer"]
        assert [[x, 16] for x in g["ondemand"]] == wl["ondemand"], g["layer"]
        assert g["victims"] == wl["victims"], g["layer"]
    assert got["arcs"] == want["arcs"]
    assert got["recall"] == pytest.approx(want["report"]["recall"], abs=1e-12)
    assert got["dequant_count"] == want["report"]["dequant_count"]
    gd, chd = _arrays(dec, cfg)
    wd = e["decode_eap_warm"]
    got = O.decode_schedule(gd, chd, mats, taus, e["plan"], cfg.top_k, wd["n"], kn, 4, arcs=arcs, eap_counts=counts)
    _check_decode(got, wd)


@pytest.mark.parametrize("name", ["qwen", "dsk", "mixtral"])
def test_decode_schedule_model_shapes(name):
    e = golden()["schedules"][name]
    cfg, dec, pre, w = config_traces(name)
    gd, chd = _arrays(dec, cfg)
    got = O.decode_schedule(gd, chd, np.stack(w.matrices), np.array(w.temperatures), e["plan"], cfg.top_k,
                            e["decode_cold"]["n"], _knobs(), 4)
    _check_decode(got, e["decode_cold"])
