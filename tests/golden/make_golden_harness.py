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
    # _Channel queue semantics (pipeline.py:163-264): random enqueue / promote /
    # drop_stale sequences and the pending order (seq ids) after every operation
    import numpy as np
    from moesim import pipeline as mp
    rng = np.random.default_rng(11)
    chans = []
    for _ in range(60):
        ch = mp._Channel()
        ops, states = [], []
        for _ in range(int(rng.integers(5, 40))):
            r = rng.random()
            if r < 0.6:
                op = ["enqueue", "prefetch" if rng.random() < 0.6 else "ondemand", int(rng.integers(0, 4)),
                      int(rng.integers(0, 4)), int(rng.integers(0, 8))]
                ch.enqueue(op[1], op[2], op[3], op[4], 4, 1.0, 0.0)
            elif r < 0.8:
                op = ["promote"]
                ch.promote_ondemand()
            else:
                op = ["drop_stale", int(rng.integers(0, 4)), int(rng.integers(0, 4))]
                ch.drop_stale((op[1], op[2]))
            ops.append(op)
            states.append([t.seq for t in ch.pending])
        chans.append({"ops": ops, "pending": states})
    out["channel"] = chans
    with open(os.path.join(OUT, "golden_harness.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote golden_harness.json", len(rows), "rows")


if __name__ == "__main__":
    main()
