"""K1 event time per decode step vs the prediction budget n and residency (all
experts resident: no prefetches issued; 15 slots per layer: cold).  Args: n:r|c ..."""
import sys, os, json, torch
sys.path.insert(0, os.getcwd())
from paper_2502_12224_b200.core import ModelConfig
from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
from paper_2502_12224_b200.experts import ExpertStore
from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
cfg = ModelConfig.from_shape(24, 60, 4, 2048, 1408, 3)
tr, w = gen_trace(cfg, GenConfig(seed=0, num_tokens=64))
store = ExpertStore(cfg, bits=(4, 2), shared_intermediate=5632, shared_bits=16)
_, g, ch = tr.dense_arrays(cfg)
gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
cases = [(int(a.split(':')[0]), a.split(':')[1] == 'r') for a in sys.argv[1:]] or [(n, r) for n in (0, 15) for r in (True, False)]
for n, resident in cases:
    if True:
        eng = OffloadEngine(cfg, [60 if resident else 15] * 24, store, w, StrategyKnobs(budget_n=n), max_tokens=64)
        eng.set_copy_timing(1)
        if resident:
            for l in range(24): eng.seed_resident(l, range(60))
        eng.decode(gd[:4], chd[:4])
        if resident:
            for l in range(24): eng.seed_resident(l, range(60))
        else:
            eng.reset_cache()
        st = eng.decode(gd, chd).stats
        print(json.dumps({"n": n, "resident": resident, "k1_us": st["gate_ms"] * 1e3 / st["steps"],
                          "us_per_step": st["gpu_ms"] * 1e3 / st["steps"], "pf": st["prefetch_issued"]}), flush=True)
        eng.close()
