"""Engine robustness on the GPU (run with -m gpu).

* Launch serialisation: under CUDA_LAUNCH_BLOCKING=1 (and under profilers,
  which inject through CUDA_INJECTION64_PATH) a launch may block its thread
  until the kernel ran; the engine then enqueues expert compute only after the
  step's transfers landed and must still finish with the same decisions.
* The trace's ``chosen`` set drives every cache decision, as record.chosen does
  in the reference (pipeline.py:422, 620-631); the device router only feeds the
  mismatch counter, the routing weights and the predictor.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from golden_util import config_traces, golden
from oracle import fate_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"CUDA_LAUNCH_BLOCKING": "1"}, {"FATE_PROFILE_SERIAL": "1"}])
def test_smoke_under_launch_serialisation(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "smoke ok" in r.stdout


def test_trace_chosen_drives_decisions():
    import torch
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    e = golden()["schedules"]["tiny"]
    cfg, dec, pre, w = config_traces("tiny")
    store = ExpertStore(cfg, bits=(4, 2), seed=0)
    n = 15
    eng = OffloadEngine(cfg, e["plan"], store, w, StrategyKnobs(budget_n=n), max_tokens=64)
    _, g, ch = dec.dense_arrays(cfg)
    T = 16
    g, ch = g[:T], ch[:T].copy()
    # replace the chosen set of every 7th step by a different ascending set
    rng = np.random.default_rng(3)
    changed = 0
    for s in range(0, T * cfg.num_layers, 7):
        t, l = divmod(s, cfg.num_layers)
        while True:
            alt = np.sort(rng.choice(cfg.num_experts, cfg.top_k, replace=False)).astype(np.int32)
            if not np.array_equal(alt, ch[t, l]):
                break
        ch[t, l] = alt
        changed += 1
    res = eng.decode(torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda"), want_logs=True)
    ora = O.decode_schedule(g, ch.tolist(), np.stack(w.matrices), np.array(w.temperatures), e["plan"], cfg.top_k, n,
                            O.StrategyKnobs(), 4)
    for got, want in zip(res.logs, ora["steps"]):
        assert (got["chosen"], got.get("pred"), got.get("prefetch"), got["hits"], got["ondemand"],
                got["victims"]) == (want["chosen"], want.get("pred"), want.get("prefetch"), want["hits"],
                                    want["ondemand"], want["victims"])
    for l in range(cfg.num_layers):
        assert eng.arc_state(l) == ora["arcs"][l]
    assert res.stats["trace_mismatches"] == changed
    eng.close()


def test_strategy_without_prefetch_policy_issues_no_prefetch():
    """Strategy('fate', quant_policy=QuantPolicy()) built directly has no predictor
    (build_decode_predictor returns None, pipeline.py:330-331)."""
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import LayeredExpertCache, plan_allocation
    from paper_2502_12224_b200.core import TimingModel
    from paper_2502_12224_b200.quant import QuantPolicy
    from golden_util import PAPER_TIMING
    cfg, dec, pre, w = config_traces("tiny")
    plan = plan_allocation(cfg, cfg.dense_bytes + 12 * cfg.expert_bytes[4], 4)
    s = P.Strategy("fate", None, QuantPolicy())
    tl, rep, res = P.simulate_decoding(dec, s, plan, TimingModel(**PAPER_TIMING), cfg, weights=w,
                                       cache=LayeredExpertCache(plan), return_result="logs")
    assert res.stats["prefetch_issued"] == 0
    assert all("pred" not in lg for lg in res.logs)
    assert rep.recall == 0.0
