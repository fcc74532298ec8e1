"""Golden schedules at the configurations the bench measures, produced by running
the REFERENCE (`moesim`) in this container.

Run from the repo root:  python tests/golden/make_golden_big.py
Writes tests/golden/golden_big.json.gz (committed; the tests never read
/root/reference).  Same observation-only instrumentation as make_golden.py.

* ``qwen_bench``: BASELINE configs[1] exactly as bench.py runs it -- Qwen1.5-MoE
  shape, 360 INT4 slots, gen_trace(seed=0, 256 decode tokens), Strategy.fate(),
  a B200-like TimingModel whose transfer budget is n = 0 (bench.py measures
  t_expert_io[4] = 0.10 ms > t_moe + t_attn + t_gate), cold cache.
* ``dsk_prefill512``: BASELINE configs[2] as bench.py runs it -- DeepSeek-MoE
  shape, 448 INT4 slots, gen_trace(seed=0, 512 prefill tokens), cold cache,
  paper TimingModel; then 32 decode tokens (seed 1, same gate weights) on the
  warmed cache (compare_strategies chaining, pipeline.py:828-849).
* ``mixtral_sweep``: BASELINE configs[3] -- Mixtral-8x7B shape, 64 decode tokens,
  S in {0, 32, 64, 128, 192, 256} INT4 slots, cold cache each, paper timing.
* ``qwen_lod``: the LoD baseline on the Qwen shape (zero plan, 16-bit on-demand).
"""

from __future__ import annotations

import gzip
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as MG  # noqa: E402  (instrumented reference: LogCache / run_*_logged)

from moesim import cache as mcache  # noqa: E402
from moesim import core as mcore  # noqa: E402
from moesim import gatesim as mgate  # noqa: E402
from moesim import pipeline as mpipe  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
# B200-like timings: transfer_budget = floor((0.02+0.01+0.005)/0.1) = 0
B200_N0 = dict(t_moe=0.02, t_attn=0.01, t_gate=0.005, t_expert_io={16: 0.3, 8: 0.16, 4: 0.1, 2: 0.06}, dequant_ms=0.0)

SHAPES = {
    "qwen": dict(L=24, E=60, k=4, H=2048, I=1408, Lb=3),
    "dsk": dict(L=28, E=64, k=6, H=2048, I=1408, Lb=3),
    "mixtral": dict(L=32, E=8, k=2, H=4096, I=14336, Lb=1),
}


def cfg_of(name):
    c = SHAPES[name]
    return MG.model_cfg(c)


def plan_of(cfg, S):
    return mcache.plan_allocation(cfg, cfg.dense_bytes + S * cfg.expert_bytes[4], 4)


def main():
    out = {}
    # ------------------------------------------------------------ configs[1]
    cfg = cfg_of("qwen")
    dec, w = mgate.gen_trace(cfg, mgate.GenConfig(seed=0, num_tokens=256, phase="decoding"))
    plan = plan_of(cfg, 360)
    timing = mcore.TimingModel(**B200_N0)
    r = MG.run_decode_logged(dec, mpipe.Strategy.fate(), plan, timing, cfg, w, MG.LogCache(plan))
    assert r["n"] == 0
    out["qwen_bench"] = {"shape": SHAPES["qwen"], "S": 360, "tokens": 256, "seed": 0,
                         "plan": list(plan.per_layer_capacity), "dec_sha": MG.trace_sha(dec), "decode_cold": r}
    print("qwen_bench hit", r["report"]["hit_rate"], flush=True)
    # LoD on the same trace (zero plan, no predictor, 16-bit on-demand)
    lod_plan = mcache.zero_plan(cfg, cfg.dense_bytes + 360 * cfg.expert_bytes[4])
    paper = mcore.TimingModel(**MG.PAPER_TIMING)
    dec32, _ = mgate.gen_trace(cfg, mgate.GenConfig(seed=0, num_tokens=32, phase="decoding"))
    r = MG.run_decode_logged(dec32, mpipe.Strategy.lod(), lod_plan, paper, cfg, w, MG.LogCache(lod_plan))
    out["qwen_lod"] = {"shape": SHAPES["qwen"], "tokens": 32, "seed": 0, "plan": list(lod_plan.per_layer_capacity),
                       "dec_sha": MG.trace_sha(dec32), "decode": r}

    # ------------------------------------------------------------ configs[2]
    cfg = cfg_of("dsk")
    pre, w = mgate.gen_trace(cfg, mgate.GenConfig(seed=0, num_tokens=512, phase="prefill"))
    dec, _ = mgate.gen_trace(cfg, mgate.GenConfig(seed=1, num_tokens=32, phase="decoding"), weights=w)
    plan = plan_of(cfg, 448)
    cache = MG.LogCache(plan)
    rp = MG.run_prefill_logged(pre, mpipe.Strategy.fate(), plan, paper, cfg, w, cache)
    rd = MG.run_decode_logged(dec, mpipe.Strategy.fate(), plan, paper, cfg, w, cache)
    out["dsk_prefill512"] = {"shape": SHAPES["dsk"], "S": 448, "pre_tokens": 512, "dec_tokens": 32,
                             "plan": list(plan.per_layer_capacity), "pre_sha": MG.trace_sha(pre),
                             "dec_sha": MG.trace_sha(dec), "prefill_cold": rp, "decode_warm": rd}
    print("dsk prefill tok/s", rp["report"]["tokens_per_s"], flush=True)

    # ------------------------------------------------------------ configs[3]
    cfg = cfg_of("mixtral")
    dec, w = mgate.gen_trace(cfg, mgate.GenConfig(seed=0, num_tokens=64, phase="decoding"))
    sweep = {}
    for S in (0, 32, 64, 128, 192, 256):
        plan = plan_of(cfg, S)
        r = MG.run_decode_logged(dec, mpipe.Strategy.fate(), plan, paper, cfg, w, MG.LogCache(plan))
        sweep[str(S)] = {"plan": list(plan.per_layer_capacity), "decode_cold": r}
        print("mixtral S", S, "hit", r["report"]["hit_rate"], flush=True)
    out["mixtral_sweep"] = {"shape": SHAPES["mixtral"], "tokens": 64, "seed": 0, "dec_sha": MG.trace_sha(dec),
                            "budgets": sweep}

    with gzip.open(os.path.join(OUT, "golden_big.json.gz"), "wt") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote golden_big.json.gz")


if __name__ == "__main__":
    main()
