"""The reference harness (experiments.run_experiment / sweep_budget / ablate) on
the B200 engine at the Qwen1.5-MoE shape: Fate, EAP and LoD over a memory-budget
sweep (paper Fig. 9) and the component ablation (Fig. 11), written in the
reference's report format under profiles/r02_experiments/.

The TimingModel is measured on this GPU by a short Fate decode (t_gate, t_moe
from the engine's CUDA events, t_expert_io from the copy events; attention is
not executed, t_attn = 0.01 ms as in bench.py), so the transfer budget n is the
one this hardware gives.  Usage: python tools/run_b200_experiments.py [tokens]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2502_12224_b200 import experiments as X  # noqa: E402
from paper_2502_12224_b200 import pipeline as P  # noqa: E402
from paper_2502_12224_b200.cache import plan_allocation  # noqa: E402
from paper_2502_12224_b200.core import ModelConfig, TimingModel  # noqa: E402
from paper_2502_12224_b200.experts import ExpertStore  # noqa: E402
from paper_2502_12224_b200.gatesim import GenConfig, gen_trace  # noqa: E402


def main():
    tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    out = os.path.join(ROOT, "profiles", "r02_experiments")
    cfg = ModelConfig.from_shape(24, 60, 4, 2048, 1408, 3, dense_bytes=24 * 3 * 2048 * 5632 * 2)
    store = ExpertStore(cfg, bits=(16, 4, 2), seed=0, shared_intermediate=5632)
    kw = dict(experts=store, shared_intermediate=5632)
    # measure the timing model with a short cold Fate decode at 25% of the expert slots
    probe, w = gen_trace(cfg, GenConfig(seed=99, num_tokens=16))
    plan = plan_allocation(cfg, cfg.dense_bytes + 360 * cfg.expert_bytes[4], 4)
    paper = TimingModel(t_moe=13.0, t_attn=9.0, t_gate=2.0, t_expert_io={16: 6.0, 8: 3.0, 4: 1.6, 2: 0.85})
    _, _, (res) = P.simulate_decoding(probe, P.Strategy.fate(), plan, paper, cfg, weights=w, return_result=True, **kw)
    tm = P.measure_timing_model(res.stats, cfg, res.stats["steps"], res.copies)
    io = dict(tm.t_expert_io)
    io.setdefault(4, io.get(2, 0.06) * 5.4 / 3.24)
    io.setdefault(16, io[4] * 17.3 / 5.4)
    io.setdefault(8, (io[16] + io[4]) / 2)
    io.setdefault(2, io[4] * 3.24 / 5.4)
    timing = TimingModel(t_moe=tm.t_moe, t_attn=tm.t_attn, t_gate=tm.t_gate, t_expert_io=io, dequant_ms=0.0)
    slots = cfg.num_layers * cfg.num_experts
    budgets = [cfg.dense_bytes + int(f * slots) * cfg.expert_bytes[4] for f in (0.1, 0.25, 0.5, 0.75)]
    spec = X.ExperimentSpec(model=cfg, timing=timing, strategies=(P.Strategy.fate(), P.Strategy.eap(),
                                                                  P.Strategy.lod()),
                            budgets=tuple(budgets), seeds=(0,), generation=GenConfig(seed=0, num_tokens=tokens),
                            prefill_tokens=tokens)
    t0 = time.time()
    res = X.sweep_budget(spec, **kw)
    paths = X.write_outputs(res, out)
    abl = X.ablate(X.ExperimentSpec(model=cfg, timing=timing, strategies=spec.strategies, budgets=(budgets[1],),
                                    seeds=(0,), generation=spec.generation, prefill_tokens=tokens), **kw)
    tok = {(r.strategy, r.phase, r.budget_bytes): r.tokens_per_s for r in res.rows}
    speedups = []
    for b in budgets:
        row = {"budget_bytes": b, "expert_slots": (b - cfg.dense_bytes) // cfg.expert_bytes[4]}
        for ph in ("decoding", "prefill"):
            row[f"fate_over_lod_{ph}"] = tok[("fate", ph, b)] / tok[("lod", ph, b)]
            row[f"fate_over_eap_{ph}"] = tok[("fate", ph, b)] / tok[("eap", ph, b)]
        speedups.append(row)
    summary = {"workload": f"Qwen1.5-MoE shape, {tokens} decode + {tokens} prefill tokens, seed 0, B200",
               "timing_model_ms": {"t_moe": timing.t_moe, "t_attn": timing.t_attn, "t_gate": timing.t_gate,
                                   "t_expert_io": {str(k): v for k, v in timing.t_expert_io.items()}},
               "transfer_budget_n": P.transfer_budget(timing, 4), "speedups": speedups, "ablation": abl,
               "wall_s": time.time() - t0, "files": paths}
    with open(os.path.join(out, "b200_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))
    P.release_pools()


if __name__ == "__main__":
    main()
