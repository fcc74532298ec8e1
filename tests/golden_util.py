"""Shared helpers for tests that read the committed golden vectors."""
import functools
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def golden() -> dict:
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=1)
def tiny_traces():
    return dict(np.load(os.path.join(GOLDEN_DIR, "tiny_traces.npz")))


PAPER_TIMING = dict(t_moe=13.0, t_attn=9.0, t_gate=2.0, t_expert_io={16: 6.0, 8: 3.0, 4: 1.6, 2: 0.85})


@functools.lru_cache(maxsize=8)
def config_traces(name: str):
    """(cfg, decode trace, prefill trace, gate weights) regenerated with the package's
    own generator; tests/test_tracegen.py pins them to the reference's bytes."""
    from paper_2502_12224_b200 import core, gatesim
    c = golden()["schedules"][name]["cfg"]
    cfg = core.ModelConfig.from_shape(c["L"], c["E"], c["k"], c["H"], c["I"], c["Lb"])
    dec, w = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=0, num_tokens=c["dec_tokens"], phase="decoding"))
    pre, _ = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=1, num_tokens=c["pre_tokens"], phase="prefill"), weights=w)
    return cfg, dec, pre, w


@functools.lru_cache(maxsize=1)
def golden_big() -> dict:
    """Reference schedules at the measured configurations (tests/golden/make_golden_big.py)."""
    import gzip
    with gzip.open(os.path.join(GOLDEN_DIR, "golden_big.json.gz"), "rt") as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=4)
def big_traces(name: str):
    """(cfg, traces..., gate weights) of a golden_big entry, regenerated with the
    package's generator (pinned to the reference bytes by the dec/pre sha256)."""
    from paper_2502_12224_b200 import core, gatesim
    e = golden_big()[name]
    s = e["shape"]
    cfg = core.ModelConfig.from_shape(s["L"], s["E"], s["k"], s["H"], s["I"], s["Lb"])
    if name == "qwen_bench":
        dec, w = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=0, num_tokens=e["tokens"], phase="decoding"))
        return cfg, dec, w
    if name == "qwen_lod":
        dec, w = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=0, num_tokens=e["tokens"], phase="decoding"))
        return cfg, dec, w
    if name == "dsk_prefill512":
        pre, w = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=0, num_tokens=e["pre_tokens"], phase="prefill"))
        dec, _ = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=1, num_tokens=e["dec_tokens"], phase="decoding"),
                                   weights=w)
        return cfg, pre, dec, w
    if name == "mixtral_sweep":
        dec, w = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=0, num_tokens=e["tokens"], phase="decoding"))
        return cfg, dec, w
    raise KeyError(name)


def trace_sha(trace) -> str:
    import hashlib
    import tempfile
    from paper_2502_12224_b200 import core
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.ndjson")
        core.write_trace(trace, p)
        return hashlib.sha256(open(p, "rb").read()).hexdigest()
