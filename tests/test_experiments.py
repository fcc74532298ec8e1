"""The reference's experiment harness on the engine (paper_2502_12224_b200.experiments):
spec parsing and report formats on the CPU; the full matrix and the ablation
on the GPU, with the timing-independent recall of every run equal to the
reference's own run_experiment on the same spec (tests/golden/make_golden_harness.py)."""
import json
import os

import pytest

from golden_util import GOLDEN_DIR


def _golden():
    with open(os.path.join(GOLDEN_DIR, "golden_harness.json")) as fh:
        return json.load(fh)


def test_spec_parsing_and_csv_format():
    from paper_2502_12224_b200 import experiments as X
    g = _golden()
    spec = X.ExperimentSpec.from_dict(g["spec"])
    assert [s.kind for s in spec.strategies] == ["fate", "eap", "lod"]
    assert spec.budgets == tuple(g["spec"]["budgets"]) and spec.seeds == (0, 1) and spec.prefill_tokens == 16
    assert list(X.CSV_HEADER) == g["csv_header"]
    rows = []
    for vals in g["csv_rows"]:
        rid, strat, phase, budget = vals[:4]
        num = [None if v == "" else float(v) for v in vals[4:]]
        rows.append(X.RunRow(rid, strat, phase, int(budget), int(rid.rsplit("_s", 1)[1]), *num))
    assert X.csv_text(rows) == g["csv_head"]
    assert X.ablation_strategy("+prefetch")[1] is False and X.ablation_strategy("+prefetch+cache")[1] is True
    with pytest.raises(Exception):
        X.strategy_from_spec("nope")
    with pytest.raises(Exception):
        X.sweep_budget(spec, budgets=[3, 2])


def test_traces_for_seed_match_reference_generation():
    # the per-seed traces come from SeedSequence([gen.seed, seed]).spawn(2) (experiments.py:158-190)
    import numpy as np
    from paper_2502_12224_b200 import experiments as X
    from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
    spec = X.ExperimentSpec.from_dict(_golden()["spec"])
    pre, dec, w = X.traces_for_seed(spec, 1)
    d_seed, p_seed = (int(s.generate_state(1)[0]) for s in np.random.SeedSequence([3, 1]).spawn(2))
    dec2, w2 = gen_trace(spec.model, GenConfig(seed=d_seed, num_tokens=24))
    assert dec.equals(dec2) and pre.num_tokens == 16 and dec.num_tokens == 24


@pytest.mark.gpu
def test_run_experiment_and_ablation_on_engine(tmp_path):
    from paper_2502_12224_b200 import experiments as X
    g = _golden()
    spec = X.ExperimentSpec.from_dict(g["spec"])
    res = X.run_experiment(spec)
    assert [(r.run_id, r.strategy, r.phase, r.budget_bytes, r.seed) for r in res.rows] == \
           [(r["run_id"], r["strategy"], r["phase"], r["budget_bytes"], r["seed"]) for r in g["rows"]]
    for got, want in zip(res.rows, g["rows"]):
        assert got.recall == pytest.approx(want["recall"], abs=1e-12), got.run_id
        assert got.tokens_per_s > 0
    assert sorted(res.summary["groups"][0]) == g["summary_keys"]
    paths = X.write_outputs(res, tmp_path)
    assert open(paths["csv"]).read().splitlines()[0] == ",".join(g["csv_header"])
    abl = X.ablate(spec)
    assert [s["stage"] for s in abl["stages"]] == g["ablation_stages"] and abl["budget_bytes"] == g["ablation_budget"]
    assert all(s["tokens_per_s_mean"] > 0 for s in abl["stages"])
