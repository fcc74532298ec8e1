"""Pin the oracle and the trace generator at the measured configurations
(tests/golden/make_golden_big.py ran the reference to produce these): the
bench's Qwen 256-token n = 0 decode, the DeepSeek 512-token prefill chained
into decode, the Mixtral budget sweep and LoD on the Qwen shape."""

import numpy as np
import pytest

from golden_util import big_traces, golden_big, trace_sha
from oracle import fate_oracle as O
from test_oracle_golden import _check_decode


def _arrays(trace, cfg):
    _, g, ch = trace.dense_arrays(cfg)
    return g, ch.tolist()


@pytest.mark.parametrize("name", ["qwen_bench", "qwen_lod", "dsk_prefill512", "mixtral_sweep"])
def test_gen_trace_matches_reference_bytes_big(name):
    e = golden_big()[name]
    tr = big_traces(name)
    if name == "dsk_prefill512":
        assert trace_sha(tr[1]) == e["pre_sha"]
        assert trace_sha(tr[2]) == e["dec_sha"]
    else:
        assert trace_sha(tr[1]) == e["dec_sha"]


def test_oracle_bench_config_decode():
    """configs[1] as bench.py runs it: 256 tokens x 24 layers, n = 0, cold."""
    e = golden_big()["qwen_bench"]
    cfg, dec, w = big_traces("qwen_bench")
    g, ch = _arrays(dec, cfg)
    got = O.decode_schedule(g, ch, np.stack(w.matrices), np.array(w.temperatures), e["plan"], cfg.top_k, 0,
                            O.StrategyKnobs(), 4)
    _check_decode(got, e["decode_cold"])


def test_oracle_qwen_lod():
    e = golden_big()["qwen_lod"]
    cfg, dec, w = big_traces("qwen_lod")
    g, ch = _arrays(dec, cfg)
    got = O.decode_schedule(g, ch, np.stack(w.matrices), np.array(w.temperatures), e["plan"], cfg.top_k,
                            e["decode"]["n"], O.StrategyKnobs(kind="lod", quant=False), 16)
    _check_decode(got, e["decode"])


def test_oracle_dsk_prefill512_chained():
    e = golden_big()["dsk_prefill512"]
    cfg, pre, dec, w = big_traces("dsk_prefill512")
    mats, taus = np.stack(w.matrices), np.array(w.temperatures)
    arcs = [O.Arc(c) for c in e["plan"]]
    want = e["prefill_cold"]
    started = {l: set(x["started"]) for l, x in enumerate(want["layers"])}
    gp, chp = _arrays(pre, cfg)
    got = O.prefill_schedule(gp, chp, mats, taus, e["plan"], cfg.top_k, O.StrategyKnobs(), 4, started=started,
                             arcs=arcs)
    for gl, wl in zip(got["layers"], want["layers"]):
        assert [list(x) for x in gl.get("prefetch", [])] == wl["prefetch_for_next"], gl["layer"]
        assert [[x, 2] for x in gl["ondemand"]] == wl["ondemand"], gl["layer"]
        assert gl["victims"] == wl["victims"], gl["layer"]
    assert got["arcs"] == want["arcs"]
    assert got["recall"] == pytest.approx(want["report"]["recall"], abs=1e-12)
    assert got["dequant_count"] == want["report"]["dequant_count"]
    gd, chd = _arrays(dec, cfg)
    wd = e["decode_warm"]
    got = O.decode_schedule(gd, chd, mats, taus, e["plan"], cfg.top_k, wd["n"], O.StrategyKnobs(), 4, arcs=arcs)
    _check_decode(got, wd)


def test_oracle_mixtral_budget_sweep():
    e = golden_big()["mixtral_sweep"]
    cfg, dec, w = big_traces("mixtral_sweep")
    g, ch = _arrays(dec, cfg)
    mats, taus = np.stack(w.matrices), np.array(w.temperatures)
    for S, b in e["budgets"].items():
        got = O.decode_schedule(g, ch, mats, taus, b["plan"], cfg.top_k, b["decode_cold"]["n"], O.StrategyKnobs(), 4)
        _check_decode(got, b["decode_cold"])
