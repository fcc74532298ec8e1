"""CPU-side tests: the C-ABI library loads and exports every declared symbol,
the reference-API mirrors behave like the reference's (validation, errors,
plans, policies), and the product path refuses to run without a GPU."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from golden_util import golden
from paper_2502_12224_b200 import cache, core, errors, pipeline, predict, quant

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "fate_b200.h")).read()
    return sorted(set(re.findall(r"\b(fate_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2502_12224_b200 import _lib, build
    build.build()
    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), set(declared) ^ set(_lib.SIGNATURES)
    assert lib.fate_version() == 1


def test_struct_sizes_match_header():
    from paper_2502_12224_b200 import _lib
    src = os.path.join(ROOT, "include")
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "s.c")
        open(c, "w").write('#include <stdio.h>\n#include "fate_b200.h"\nint main(){printf("%zu %zu %zu %zu\\n",'
                           'sizeof(fate_step_log),sizeof(fate_prefill_log),sizeof(fate_run_stats),'
                           'sizeof(fate_engine_config));}\n')
        exe = os.path.join(d, "s")
        subprocess.run(["gcc", "-I", src, c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    assert [int(x) for x in out] == [C.sizeof(_lib.StepLog), C.sizeof(_lib.PrefillLog), C.sizeof(_lib.RunStats),
                                     C.sizeof(_lib.EngineConfig)]


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2502_12224_b200 import _lib, ops
    with pytest.raises(errors.DeviceError):
        _lib.lib()
    with pytest.raises(errors.DeviceError):
        ops.device()


def test_status_codes_map_to_reference_errors():
    with pytest.raises(errors.InvalidConfig):
        errors.raise_for(1, "x")
    with pytest.raises(errors.TraceMismatch):
        errors.raise_for(2, "x")
    with pytest.raises(errors.BudgetTooSmall):
        errors.raise_for(3, "x")
    with pytest.raises(errors.DeviceError):
        errors.raise_for(5, "x")
    assert errors.InvalidConfig("m").code == "INVALID_CONFIG"
    errors.raise_for(0, "ok")


def _cfg():
    return core.ModelConfig.from_shape(4, 8, 2, 256, 512, 1)


def test_model_config_and_validation():
    cfg = _cfg()
    assert cfg.intermediate_dim == 512
    assert cfg.expert_bytes == {16: 786432, 8: 442368, 4: 245760, 2: 147456}
    tm = core.TimingModel(13, 9, 2, {16: 6, 8: 3.0, 4: 1.6, 2: 0.85})
    core.validate_config(cfg, tm)
    with pytest.raises(errors.InvalidConfig):
        core.validate_config(core.ModelConfig(4, 4, 5, 8, 1, {16: 10}, 0), tm)
    with pytest.raises(errors.InvalidConfig):
        core.validate_config(cfg, core.TimingModel(13, 9, 2, {2: 7, 4: 6}))
    assert quant.lint_expert_bytes(cfg) == []


def test_plan_allocation_matches_spec_examples():
    k = golden()["kat"]
    cfg = core.ModelConfig(24, 60, 4, 8, 3, {16: 100, 4: 10}, 0)
    assert list(cache.plan_allocation(cfg, 3000, 4).per_layer_capacity) == k["plan_300"]
    assert list(cache.plan_allocation(cfg, 1000, 4).per_layer_capacity) == k["plan_100"]
    assert list(cache.plan_allocation(cfg, 15000, 4).per_layer_capacity) == k["plan_1500"]
    with pytest.raises(errors.BudgetTooSmall):
        cache.plan_allocation(core.ModelConfig(24, 60, 4, 8, 3, {16: 100, 4: 10}, 50), 10, 4)
    assert cache.zero_plan(cfg).per_layer_capacity == (0,) * 24
    assert sum(cache.uniform_plan(cfg, 3000, 4).per_layer_capacity) == 300


def test_policies_and_bits():
    with pytest.raises(errors.InvalidConfig):
        predict.PrefetchPolicy("nope")
    with pytest.raises(errors.InvalidConfig):
        predict.PrefetchPolicy("percentile", 0.9).validate_for(8, 2)
    prof = quant.PopularityProfile.from_counts(0, {i: 10 - i for i in range(8)})
    assert {str(e): b for e, b in quant.assign_bits(prof, quant.QuantPolicy(), "prefill").items()} == \
        golden()["kat"]["assign_bits_8"]
    assert quant.search_p(lambda p: 0.0 if p <= 0.25 + 1e-9 else 0.05) == pytest.approx(0.25)
    with pytest.raises(errors.NoFeasibleP):
        quant.search_p(lambda p: 0.02)
    lists = [predict.PrefetchList(1, (predict.PrefetchEntry(1, .5, None), predict.PrefetchEntry(2, .4, None)))] * 3
    assert predict.prefill_merge(lists).ordering == (1, 2)
    assert predict.prefetch_recall([5, 11, 21, 36], [5, 21, 31, 36]) == 0.75


def test_strategy_and_budget():
    s = pipeline.Strategy.fate()
    assert (s.prefetch_bits(), s.ondemand_bits(), s.cache_bits()) == (4, 2, 4)
    assert pipeline.Strategy.fate(quant_policy=None).quant_policy == quant.QuantPolicy()  # pipeline.py:78 quirk
    lod = pipeline.Strategy.lod()
    assert (lod.prefetch_bits(), lod.ondemand_bits()) == (16, 16)
    with pytest.raises(errors.InvalidConfig):
        pipeline.Strategy("lod", prefetch_policy=predict.PrefetchPolicy())
    tm = core.TimingModel(13, 9, 2, {4: 6, 16: 12})
    assert pipeline.transfer_budget(tm, 4) == 4
    knobs = pipeline.knobs_for(s, cache.plan_allocation(_cfg(), 12 * 245760, 4), 4)
    assert (knobs.use_predictor, knobs.policy, knobs.budget_n, knobs.prefill_ondemand_bits) == (True, "percentile", 4, 2)
    # EAP maps onto the engine's co-activation predictor (policy "eap"), 16-bit transfers, decode only
    ek = pipeline.knobs_for(pipeline.Strategy.eap(), cache.zero_plan(_cfg()), 3)
    assert (ek.use_predictor, ek.policy, ek.budget_n, ek.prefetch_bits, ek.ondemand_bits,
            ek.prefill_use_predictor) == (True, "eap", 3, 16, 16, True)


def test_unbound_cache_protocol():
    plan = cache.plan_allocation(_cfg(), 12 * 245760, 4)
    c = cache.LayeredExpertCache(plan)
    c.seed_resident(1, [3, 4, 5])
    assert c.layers[1].resident() == {3, 4}  # capacity 2
    assert c.contains(1, 3) and not c.contains(1, 5)
    with pytest.raises(errors.InvalidConfig):
        cache.update_after_layer(c, 0, [1])


def test_simulate_rejects_bad_inputs_before_touching_the_gpu():
    from golden_util import config_traces
    cfg, dec, pre, w = config_traces("tiny")
    plan = cache.plan_allocation(cfg, 12 * cfg.expert_bytes[4], 4)
    tm = core.TimingModel(13, 9, 2, {16: 6, 8: 3.0, 4: 1.6, 2: 0.85})
    with pytest.raises(errors.TraceMismatch):
        pipeline.simulate_decoding(pre, pipeline.Strategy.fate(), plan, tm, cfg, weights=w)
    with pytest.raises(errors.TraceMismatch):
        pipeline.simulate_prefill(dec, pipeline.Strategy.fate(), plan, tm, cfg, weights=w)
    with pytest.raises(errors.InvalidConfig):
        pipeline.simulate_decoding(dec, pipeline.Strategy.fate(), plan, tm, cfg, weights=None)
    with pytest.raises(errors.InvalidConfig):
        pipeline.simulate_decoding(dec, pipeline.Strategy.fate(), plan, tm, cfg, weights=w, predictor=object())
