import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import torch
from golden_util import config_traces, golden
from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
from paper_2502_12224_b200.experts import ExpertStore
from paper_2502_12224_b200 import _lib
import numpy as np
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg, dec, pre, w = config_traces(name)
store = ExpertStore(cfg, bits=(4, 2))
e = golden()["schedules"][name]
eng = OffloadEngine(cfg, e["plan"], store, w, StrategyKnobs(budget_n=15), max_tokens=64)
_, g, ch = dec.dense_arrays(cfg)
try:
    res = eng.decode(torch.as_tensor(g[:T], device="cuda"), torch.as_tensor(ch[:T], device="cuda"))
    print("ok", res.stats["gpu_ms"])
except Exception as ex:
    print("ERR", ex)
k1 = np.zeros(8, dtype=np.uint64); _lib.load().fate_k1_profile(k1.ctypes.data); print("k1", k1)
prof = np.zeros((160, 8), dtype=np.uint64); _lib.load().fate_k3_profile(prof.ctypes.data); print("k3 cta0", prof[0], "cta1", prof[1])
