import sys, time, faulthandler
faulthandler.dump_traceback_later(150, exit=True)
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
t0 = time.time()
def log(*a):
    print(f"[{time.time()-t0:7.2f}s]", *a, flush=True)
import torch
from golden_util import config_traces, golden
from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
from paper_2502_12224_b200.experts import ExpertStore
name = sys.argv[1] if len(sys.argv) > 1 else "qwen"
cfg, dec, pre, w = config_traces(name); log("traces")
store = ExpertStore(cfg, bits=(4, 2)); log("store", store.host_bytes() / 1e9, "GB")
e = golden()["schedules"][name]
eng = OffloadEngine(cfg, e["plan"], store, w, StrategyKnobs(budget_n=15), max_tokens=64); log("engine")
toks, g, ch = dec.dense_arrays(cfg)
gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
res = eng.decode(gd, chd, want_logs=True); log("decode", {k: v for k, v in res.stats.items()})
res = eng.decode(gd, chd, want_logs=False); log("decode2", res.stats["gpu_ms"], res.stats["ffn_ms"], res.stats["gate_ms"])
