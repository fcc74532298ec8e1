"""A/B of the decode step protocols on the bench workload (Qwen shape, 360 INT4
slots, cold cache): arrival-gated K3 (default) vs the stream wait, at n = 0 (the
bench's measured TimingModel) and n = 15 (the paper's), same trace, same
decisions.  Prints one JSON line per (n, protocol)."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_12224_b200 import pipeline as P  # noqa: E402
from paper_2502_12224_b200.cache import plan_allocation  # noqa: E402
from paper_2502_12224_b200.engine import OffloadEngine  # noqa: E402
from paper_2502_12224_b200.experts import ExpertStore  # noqa: E402


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    cfg = bench.qwen_cfg()
    trace, weights = bench.make_trace(cfg, T, seed=0)
    store = ExpertStore(cfg, bits=(4, 2), seed=0, shared_intermediate=bench.QWEN["shared"], shared_bits=16)
    plan = plan_allocation(cfg, cfg.dense_bytes + bench.QWEN["slots"] * cfg.expert_bytes[4], 4)
    strategy = P.Strategy.fate()
    _, g, ch = trace.dense_arrays(cfg)
    gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
    eng = OffloadEngine(cfg, plan.per_layer_capacity, store, weights, P.knobs_for(strategy, plan, 0),
                        max_tokens=max(T, 64))
    eng.decode(gd[:8], chd[:8])
    for n in (0, 15):
        eng.set_strategy(P.knobs_for(strategy, plan, n))
        for ov in (True, False, True):
            eng.set_overlap(ov)
            st = []
            for _ in range(runs):
                eng.reset_cache()
                st.append(eng.decode(gd, chd).stats)
            s = lambda k: sum(x[k] for x in st)  # noqa: E731
            print(json.dumps({
                "n": n, "overlap": ov, "tok_s": T * runs / (s("gpu_ms") / 1e3),
                "us_per_step": s("gpu_ms") * 1e3 / s("steps"),
                "k1_us": s("gate_ms") * 1e3 / s("steps"), "k3_us_incl_wait": s("ffn_ms") * 1e3 / s("steps"),
                "k3_wait_us": s("k3_wait_ms") * 1e3 / s("steps"),
                "hit_rate_combined": (s("cache_hits") + s("arrival_hits")) / s("accesses"),
                "arrival_hits": s("arrival_hits") // runs, "ondemand": s("ondemand_issued") // runs,
                "prefetch": s("prefetch_issued") // runs, "dropped": s("transfers_dropped") // runs,
                "h2d_gb": s("h2d_bytes") / runs / 1e9}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
