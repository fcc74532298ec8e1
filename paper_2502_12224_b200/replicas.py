"""Multi-GPU plumbing: independent request streams, one process per GPU.

The path shards naturally: each rank owns an expert-slot pool,
ARC tables, copy stream and its own request stream (trace seed), with no
collective on the data path.  torch.distributed is used only for the
barrier and the end-of-run reduction of counters and times (max over ranks
for time, sum for tokens).  ``home_rank`` is the expert -> GPU map of the
expert-sharded peer-fetch mode, home(l, e) = (l*E + e) mod G.
"""

from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def replica_seed(rank: int, base: int = 0) -> int:
    """Each replica serves its own request stream."""
    return base + rank


def home_rank(layer: int, expert: int, num_experts: int, world_size: int) -> int:
    return (layer * num_experts + expert) % world_size


def shard_experts(num_layers: int, num_experts: int, rank: int, world_size: int) -> list:
    """(layer, expert) pairs homed on ``rank``."""
    return [(l, e) for l in range(num_layers) for e in range(num_experts)
            if home_rank(l, e, num_experts, world_size) == rank]


def aggregate(tokens: int, seconds: float, counters: dict | None = None, device=None) -> dict:
    """Whole-job throughput: sum of tokens over ranks / max of per-rank times;
    counters are summed.  Works on any initialised backend (nccl or gloo)."""
    import torch
    import torch.distributed as dist

    counters = dict(counters or {})
    keys = sorted(counters)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return {"tokens": tokens, "seconds": seconds, "tokens_per_s": tokens / seconds, **counters}
    dev = device or torch.device("cpu")
    t = torch.tensor([seconds], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = torch.tensor([float(tokens)] + [float(counters[k]) for k in keys], dtype=torch.float64, device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    out = {"tokens": int(s[0].item()), "seconds": float(t.item())}
    out["tokens_per_s"] = out["tokens"] / out["seconds"]
    for i, k in enumerate(keys):
        out[k] = float(s[1 + i].item())
    return out
