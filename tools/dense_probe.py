"""Per-kernel time of the dense part at the Qwen shape (run under ncu for the
launch list, or plain for CUDA-event totals)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_12224_b200 import ops  # noqa: E402
from paper_2502_12224_b200.core import ModelConfig  # noqa: E402
from paper_2502_12224_b200.dense import DenseConfig, DenseWeights  # noqa: E402

cfg = ModelConfig.from_shape(24, 60, 4, 2048, 1408, 3)
dc = DenseConfig.qwen_moe()
dw = DenseWeights(cfg, dc)
ly = dw.layers[0]
kv = torch.zeros(1024, 2, 2048, dtype=torch.bfloat16, device="cuda")
h = torch.randn(2048, device="cuda")
y = torch.randn(2048, device="cuda")
gi = torch.randn(2048, device="cuda", dtype=torch.float64) / math.sqrt(2048)
dims = {"H": 2048, "n_heads": 16, "n_kv_heads": 16, "head_dim": 128}
for _ in range(3):
    ops.dense_step(dims, ly, kv, h, y, gi, 600)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20):
    ops.dense_step(dims, ly, kv, h, y, gi, 600)
e1.record()
torch.cuda.synchronize()
print("dense step (incl. host sync per call) ms:", e0.elapsed_time(e1) / 20)
