"""Trace parity at the configurations the bench measures (run with -m gpu).

The golden schedules come from running the reference (tests/golden/make_golden_big.py):
* BASELINE configs[1] exactly as bench.py runs it (Qwen shape, 360 INT4 slots,
  256 tokens, n = 0, cold): every step's chosen / hits / on-demand / victims /
  source widths and the final ARC state of all 24 layers;
* configs[2] (DeepSeek shape, 512-token prefill, 448 slots, cold) chained into
  a 32-token decode on the warmed cache;
* configs[3] (Mixtral shape, 64 tokens) at every budget of the sweep;
* the LoD baseline (tiny and Qwen);
* K2 on the 400 reference ARC sequences (capacities 0-8, ghost hits, p).
"""

import numpy as np
import pytest

from golden_util import big_traces, golden, golden_big
from oracle import fate_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _free_pinned():
    # the stores here pin 12-45 GB of host memory each; hand it back between tests
    yield
    import gc

    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch._C._host_emptyCache()


def _steps_equal(logs, want, fields=("chosen", "hits", "ondemand", "victims")):
    assert len(logs) == len(want)
    for g, w in zip(logs, want):
        key = (g["token"], g["layer"])
        assert g["mismatch"] == 0, key
        for f in fields:
            assert g[f] == w[f], (key, f)
        assert g.get("pred") == w.get("pred"), key
        assert g.get("prefetch") == w.get("prefetch"), key


def _src_bits(logs, want, ondemand_bits, cached_bits):
    # the reference's source width: ondemand_bits for on-demand loads, the cached /
    # prefetched width otherwise (pipeline.py:441-466)
    for g, w in zip(logs, want):
        exp = [ondemand_bits if e in w["ondemand"] else cached_bits for e in w["chosen"]]
        assert g["src_bits"] == exp, (g["token"], g["layer"])


def _dev(trace, cfg):
    import torch
    _, g, ch = trace.dense_arrays(cfg)
    return torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")


def test_bench_config_decode_trace_exact():
    """configs[1] as bench.py measures it: 6,144 decode steps bit-exact against the reference."""
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import CachePlan
    from paper_2502_12224_b200.engine import OffloadEngine
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden_big()["qwen_bench"]
    want = e["decode_cold"]
    cfg, dec, w = big_traces("qwen_bench")
    store = ExpertStore(cfg, bits=(4, 2), seed=0, shared_intermediate=5632)
    plan = CachePlan(0, sum(e["plan"]), tuple(e["plan"]), 4)
    eng = OffloadEngine(cfg, e["plan"], store, w, P.knobs_for(P.Strategy.fate(), plan, want["n"]), max_tokens=256)
    gd, chd = _dev(dec, cfg)
    res = eng.decode(gd, chd, want_logs=True)
    _steps_equal(res.logs, want["steps"])
    _src_bits(res.logs, want["steps"], 2, 4)
    assert [eng.arc_state(l) for l in range(cfg.num_layers)] == want["arcs"]
    st = res.stats
    assert st["trace_mismatches"] == 0
    assert st["ondemand_issued"] == want["transfers"]["ondemand"]
    assert st["prefetch_issued"] == want["transfers"]["prefetch"] == 0
    assert st["dequant_count"] == want["report"]["dequant_count"]
    assert st["cache_hits"] / st["accesses"] == pytest.approx(want["report"]["hit_rate"], abs=1e-12)
    eng.close()


def test_dsk_prefill512_then_decode():
    """configs[2]: the 512-token prefill.  Timing-independent fields against the
    reference's own log (prediction list + bit map, victims, final ARC state);
    on-demand and residency against the oracle given the measured started set;
    then the chained decode against the reference's log."""
    import torch
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden_big()["dsk_prefill512"]
    cfg, pre, dec, w = big_traces("dsk_prefill512")
    store = ExpertStore(cfg, bits=(4, 2), seed=0)
    wd = e["decode_warm"]
    eng = OffloadEngine(cfg, e["plan"], store, w, StrategyKnobs(budget_n=wd["n"]), max_tokens=512)
    gp, chp = _dev(pre, cfg)
    Y, st, logs, _, _ = eng.prefill(gp, chp)
    ref = e["prefill_cold"]
    for l, (g, r) in enumerate(zip(logs, ref["layers"])):
        assert g["mismatch"] == 0, l
        assert [list(x) for x in g["prefetch"]] == r["prefetch_for_next"], l
        assert g["victims"] == r["victims"], l
    assert [eng.arc_state(l) for l in range(cfg.num_layers)] == ref["arcs"]
    assert st["recall_sum"] / st["recall_n"] == pytest.approx(ref["report"]["recall"], abs=1e-12)
    started = {l: set(lg["started"]) for l, lg in enumerate(logs)}
    mats, taus = np.stack(w.matrices), np.array(w.temperatures)
    _, gpn, chpn = pre.dense_arrays(cfg)
    ora = O.prefill_schedule(gpn, chpn.tolist(), mats, taus, e["plan"], cfg.top_k, O.StrategyKnobs(), 4,
                             started=started, arcs=[O.Arc(c) for c in e["plan"]])
    for l, (g, o) in enumerate(zip(logs, ora["layers"])):
        assert (g["actives"], g["counts"], g["resident"], g["ondemand"], g["src_bits"]) == \
               (o["actives"], o["counts"], o["resident"], o["ondemand"], o["src_bits"]), l
    assert st["dequant_count"] == ora["dequant_count"]
    # decode on the warmed cache: state-derived, so equal to the reference's log
    gd, chd = _dev(dec, cfg)
    res = eng.decode(gd, chd, want_logs=True)
    _steps_equal(res.logs, wd["steps"])
    assert [eng.arc_state(l) for l in range(cfg.num_layers)] == wd["arcs"]
    assert res.stats["recall_sum"] / res.stats["recall_n"] == pytest.approx(wd["report"]["recall"], abs=1e-12)
    eng.close()


def test_mixtral_budget_sweep_trace_exact():
    """configs[3]: one 64-token cold decode per budget S in {0, 32, 64, 128, 192, 256}."""
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden_big()["mixtral_sweep"]
    cfg, dec, w = big_traces("mixtral_sweep")
    store = ExpertStore(cfg, bits=(4, 2), seed=0)
    gd, chd = _dev(dec, cfg)
    for S, b in e["budgets"].items():
        want = b["decode_cold"]
        eng = OffloadEngine(cfg, b["plan"], store, w, StrategyKnobs(budget_n=want["n"]), max_tokens=64)
        res = eng.decode(gd, chd, want_logs=True)
        _steps_equal(res.logs, want["steps"])
        assert [eng.arc_state(l) for l in range(cfg.num_layers)] == want["arcs"], S
        assert res.stats["prefetch_issued"] == want["transfers"]["prefetch"], S
        assert res.stats["ondemand_issued"] == want["transfers"]["ondemand"], S
        eng.close()


@pytest.mark.parametrize("name", ["tiny", "qwen"])
def test_lod_decode_trace_exact(name):
    """LoD (pipeline.py:44-104): zero plan, no predictor, 16-bit on-demand loads."""
    from golden_util import config_traces
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import CachePlan
    from paper_2502_12224_b200.engine import OffloadEngine
    from paper_2502_12224_b200.experts import ExpertStore
    if name == "tiny":
        cfg, dec, _, w = config_traces("tiny")
        want = golden()["schedules"]["tiny"]["decode_lod"]
        caps = [0] * cfg.num_layers
    else:
        e = golden_big()["qwen_lod"]
        cfg, dec, w = big_traces("qwen_lod")
        want, caps = e["decode"], e["plan"]
    assert caps == [0] * cfg.num_layers
    store = ExpertStore(cfg, bits=(16,), seed=0)
    kn = P.knobs_for(P.Strategy.lod(), CachePlan(0, 0, tuple(caps), 16), want["n"])
    eng = OffloadEngine(cfg, caps, store, w, kn, max_tokens=64)
    gd, chd = _dev(dec, cfg)
    res = eng.decode(gd, chd, want_logs=True)
    _steps_equal(res.logs, want["steps"])
    _src_bits(res.logs, want["steps"], 16, 16)
    st = res.stats
    assert st["ondemand_issued"] == want["transfers"]["ondemand"] == cfg.num_layers * cfg.top_k * dec.num_tokens
    assert st["prefetch_issued"] == 0 and st["cache_hits"] == 0
    assert st["dequant_count"] == want["report"]["dequant_count"]
    eng.close()


def test_k2_reference_arc_sequences():
    """K2 (the device ARC, one warp per layer) replays the reference's 400 random
    access sequences: per-access hit flags and the final T1/T2/B1/B2/p."""
    from paper_2502_12224_b200.core import ModelConfig
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    from paper_2502_12224_b200.gatesim import GateWeights
    cases = golden()["arc"]
    L, E = 9, 16  # layer c has capacity c (0..8); ids < 16
    cfg = ModelConfig.from_shape(L, E, 2, 256, 256, 1)
    store = ExpertStore(cfg, bits=(4,), seed=0)
    w = GateWeights(matrices=tuple(np.zeros((E, 256)) for _ in range(L)), temperatures=(1.0,) * L)
    eng = OffloadEngine(cfg, list(range(L)), store, w, StrategyKnobs(use_predictor=False, budget_n=0), max_tokens=8)
    for i, case in enumerate(cases):
        eng.reset_cache()
        c = case["c"]
        assert eng.access(c, case["seq"]) == case["hits"], i
        got = eng.arc_state(c)
        f = case["final"]
        assert (got["t1"], got["t2"], got["b1"], got["b2"]) == (f["t1"], f["t2"], f["b1"], f["b2"]), i
        assert got["p"] == f["p"], i
        assert eng.resident(c) == set(f["t1"]) | set(f["t2"]), i
    eng.close()
