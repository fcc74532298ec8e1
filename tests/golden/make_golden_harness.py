"""Reference harness outputs (moesim.experiments) on a tiny spec, for the parity
test of paper_2502_12224_b200.experiments.  Run from the repo root in the build
container:  python tests/golden/make_golden_harness.py  (writes golden_harness.json)."""

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from moesim import experiments as mx  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
EB = {16: 786432, 8: 442368, 4: 245760, 2: 147456}  # tiny: n = 3 * 256 * 512
SPEC = {
    "model": {"num_layers": 4, "num_experts": 8, "top_k": 2, "hidden_dim": 256, "shallow_boundary_L": 1,
              "expert_bytes": {str(k): v for k, v in EB.items()}, "dense_bytes": 0},
    "timing": {"t_moe": 13.0, "t_attn": 9.0, "t_gate": 2.0, "t_expert_io": {"16": 6.0, "8": 3.0, "4": 1.6, "2": 0.85}},
    "strategies": ["fate", "eap", "lod"],
    "budgets": [8 * EB[4], 12 * EB[4]],
    "seeds": [0, 1],
    "generation": {"seed": 3, "num_tokens": 24},
    "prefill_tokens": 16,
}


def main():
    spec = mx.ExperimentSpec.from_dict(SPEC)
    res = mx.run_experiment(spec)
    rows = [{"run_id": r.run_id, "strategy": r.strategy, "phase": r.phase, "budget_bytes": r.budget_bytes,
             "seed": r.seed, "recall": r.recall} for r in res.rows]
    abl = mx.ablate(spec)
    out = {"spec": SPEC, "rows": rows, "csv_header": list(mx.CSV_HEADER), "csv_head": mx.csv_text(res.rows[:2]),
           "csv_rows": [list(r.csv_values()) for r in res.rows[:2]],
           "ablation_stages": [s["stage"] for s in abl["stages"]], "ablation_budget": abl["budget_bytes"],
           "summary_keys": sorted(res.summary["groups"][0].keys())}
    with open(os.path.join(OUT, "golden_harness.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote golden_harness.json", len(rows), "rows")


if __name__ == "__main__":
    main()
