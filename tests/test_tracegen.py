"""The package's synthetic workload generator reproduces the reference's traces byte for byte."""
import hashlib
import os

import pytest

from golden_util import config_traces, golden
from paper_2502_12224_b200 import core


def _sha(trace, tmp_path):
    p = os.path.join(tmp_path, "t.ndjson")
    core.write_trace(trace, p)
    return hashlib.sha256(open(p, "rb").read()).hexdigest()


@pytest.mark.parametrize("name", ["tiny", "qwen", "dsk", "mixtral"])
def test_gen_trace_matches_reference_bytes(name, tmp_path):
    e = golden()["schedules"][name]
    cfg, dec, pre, w = config_traces(name)
    assert _sha(dec, tmp_path) == e["dec_sha"]
    assert _sha(pre, tmp_path) == e["pre_sha"]
    assert list(w.temperatures) == e["taus"]


def test_trace_roundtrip(tmp_path):
    cfg, dec, pre, w = config_traces("tiny")
    p = os.path.join(tmp_path, "t.ndjson")
    core.write_trace(dec, p)
    back = core.read_trace(p)
    assert back.equals(dec)
    assert core.validate_trace_for(back, cfg) is back


def test_dense_arrays_layout():
    cfg, dec, pre, w = config_traces("tiny")
    toks, g, ch = dec.dense_arrays(cfg)
    assert g.shape == (64, 4, 256) and ch.shape == (64, 4, 2)
    by = dec.by_token()
    assert (g[3, 2] == by[3][2].probe_hidden["gate_in_cur"]).all()
    assert list(ch[3, 2]) == sorted(by[3][2].chosen)
