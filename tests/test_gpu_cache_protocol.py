"""The public cache protocol on the device (reference cache.py:182-215):
a LayeredExpertCache bound to the engine answers contains / layers[l].resident /
layers[l].access / seed_resident / update_after_layer exactly like the reference's
ArcState replayed by the oracle, keeps the ARC invariants (check_invariants), and
the drop-in calls the reference accepts (weights=None for LoD, a decode longer than
the prefill that warmed the cache) run on the engine."""
import numpy as np
import pytest

from golden_util import PAPER_TIMING, config_traces, golden
from oracle import fate_oracle as O

pytestmark = pytest.mark.gpu


def _bound_cache():
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import LayeredExpertCache, plan_allocation
    from paper_2502_12224_b200.core import TimingModel
    cfg, dec, pre, w = config_traces("tiny")
    plan = plan_allocation(cfg, cfg.dense_bytes + 12 * cfg.expert_bytes[4], 4)
    cache = LayeredExpertCache(plan)
    # a short decode binds the engine (and leaves a warm, reference-exact state)
    P.simulate_decoding(dec, P.Strategy.fate(), plan, TimingModel(**PAPER_TIMING), cfg, weights=w, cache=cache)
    return cfg, plan, cache, golden()["schedules"]["tiny"]["decode_cold"]["arcs"]


def test_bound_cache_protocol_matches_oracle():
    from paper_2502_12224_b200.cache import arc_access, update_after_layer
    cfg, plan, cache, arcs = _bound_cache()
    # state after the decode: the reference's final ARC lists
    ora = []
    for l in range(cfg.num_layers):
        lv = cache.layers[l]
        assert (lv.t1, lv.t2, lv.b1, lv.b2, lv.p_arc) == (arcs[l]["t1"], arcs[l]["t2"], arcs[l]["b1"], arcs[l]["b2"],
                                                          arcs[l]["p"])
        lv.check_invariants()
        a = O.Arc(plan.per_layer_capacity[l])
        a.t1, a.t2, a.b1, a.b2, a.p = list(lv.t1), list(lv.t2), list(lv.b1), list(lv.b2), lv.p_arc
        ora.append(a)
    rng = np.random.default_rng(5)
    for _ in range(200):
        l = int(rng.integers(0, cfg.num_layers))
        if rng.random() < 0.5:
            e = int(rng.integers(0, cfg.num_experts))
            assert cache.contains(l, e) == (e in ora[l].resident())
            assert arc_access(cache, l, e) == ora[l].access(e)[0]
        else:
            chosen = rng.choice(cfg.num_experts, size=cfg.top_k, replace=False).tolist()
            update_after_layer(cache, l, chosen)
            for e in sorted(chosen):
                ora[l].access(int(e))
        lv = cache.layers[l]
        assert (lv.t1, lv.t2, lv.b1, lv.b2) == (ora[l].t1, ora[l].t2, ora[l].b1, ora[l].b2)
        assert lv.p_arc == ora[l].p
        assert lv.resident() == ora[l].resident()
        lv.check_invariants()


def test_seed_resident_before_and_after_binding():
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import LayeredExpertCache, plan_allocation
    from paper_2502_12224_b200.core import TimingModel
    cfg, dec, pre, w = config_traces("tiny")
    plan = plan_allocation(cfg, cfg.dense_bytes + 12 * cfg.expert_bytes[4], 4)
    cache = LayeredExpertCache(plan)
    cache.seed_resident(1, [3, 5, 7])  # pending until bound; capacity of layer 1 is 2
    assert cache.layers[1].resident() == {3, 5}
    P.simulate_decoding(dec, P.Strategy.fate(), plan, TimingModel(**PAPER_TIMING), cfg, weights=w, cache=cache)
    for l in range(cfg.num_layers):
        cache.layers[l].check_invariants()


def test_lod_without_gate_weights_and_long_decode_after_prefill():
    # LoD accepts weights=None as in the reference (no predictor): decisions follow the
    # trace's chosen sets; and compare_strategies sizes the engine for the longer trace
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import zero_plan
    from paper_2502_12224_b200.core import TimingModel
    cfg, dec, pre, w = config_traces("tiny")
    want = golden()["schedules"]["tiny"]["decode_lod"]
    tl, rep = P.simulate_decoding(dec, P.Strategy.lod(), zero_plan(cfg), TimingModel(**PAPER_TIMING), cfg,
                                  weights=None)
    assert rep.dequant_count == want["report"]["dequant_count"] and rep.recall == 0.0
    with pytest.raises(Exception):
        P.simulate_decoding(dec, P.Strategy.fate(), zero_plan(cfg), TimingModel(**PAPER_TIMING), cfg, weights=None)
    from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
    longdec, _ = gen_trace(cfg, GenConfig(seed=4, num_tokens=100, phase="decoding"), weights=w)
    budget = cfg.dense_bytes + 12 * cfg.expert_bytes[4]
    rows = P.compare_strategies(cfg, TimingModel(**PAPER_TIMING), [P.Strategy.fate(), P.Strategy.lod()], [budget],
                                pre, longdec, weights=w)
    assert {(r.strategy, r.phase) for r in rows} == {(k, ph) for k in ("fate", "lod") for ph in ("prefill", "decoding")}
    P.release_pools()
