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


def shard_layout(num_layers: int, num_experts: int, world_size: int) -> tuple:
    """(homes, slot): homes[r] = rank r's (layer, expert) list in (l, e) order,
    slot[(l, e)] = its index in its home rank's pool."""
    homes = [shard_experts(num_layers, num_experts, r, world_size) for r in range(world_size)]
    slot = {le: i for r in range(world_size) for i, le in enumerate(homes[r])}
    return homes, slot


def source_table(num_layers: int, num_experts: int, world_size: int, bases: list, stride: int) -> list:
    """Per-(l, e) source address: home rank's pool base + slot * stride."""
    _, slot = shard_layout(num_layers, num_experts, world_size)
    return [bases[home_rank(l, e, num_experts, world_size)] + slot[(l, e)] * stride
            for l in range(num_layers) for e in range(num_experts)]


def ipc_export(dev_ptr: int) -> tuple:
    """(64-byte handle, offset) of the device allocation holding dev_ptr."""
    import ctypes as C

    from . import _lib
    h = (C.c_uint8 * 64)()
    off = C.c_int64(0)
    _lib.check(_lib.lib().fate_ipc_get_handle(C.c_void_p(dev_ptr), h, C.byref(off)), "fate_ipc_get_handle")
    return bytes(h), int(off.value)


def ipc_open(handle: bytes, offset: int) -> tuple:
    """Map a peer allocation; returns (base to close later, dev_ptr = base + offset)."""
    import ctypes as C

    from . import _lib
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p(0)
    _lib.check(_lib.lib().fate_ipc_open_handle(h, C.byref(p)), "fate_ipc_open_handle")
    return int(p.value), int(p.value) + offset


class ExpertShards:
    """Expert-sharded peer-fetch mode (north star "a cache miss is
    served by an NVLink peer read instead of a host fetch").

    Rank r keeps the packed copies (every width in ``bits``) of its home experts,
    home(l, e) = (l*E + e) mod G, resident in its own HBM (outside the expert
    cache budget: ``device_bytes`` says how much).  The home pools are exported
    with CUDA IPC, the handles all-gathered over torch.distributed, and every rank
    maps every peer's pool; ``attach(engine)`` points the engine's miss sources at
    them, so a miss of (l, e) is a device-to-device copy from the home GPU (NVLink
    for peers, HBM for local experts).  ARC, predictions and every trace decision
    are unchanged; only the source and the timing of the copies change.
    """

    def __init__(self, store, bits=(4, 2), rank: int = 0, world_size: int = 1, device=None):
        import torch
        import torch.distributed as dist

        self.cfg, self.bits, self.rank, self.world = store.cfg, tuple(bits), rank, world_size
        L, E = self.cfg.num_layers, self.cfg.num_experts
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        homes, self.slot = shard_layout(L, E, world_size)
        mine = homes[rank]
        idx = torch.tensor([l * E + e for (l, e) in mine], dtype=torch.long)
        self.pools, self.strides, local = {}, {}, {}
        for b in self.bits:
            src = store.host_pool(b)
            pool = torch.empty((len(mine), store.stride(b)), dtype=torch.uint8, device=self.device)
            for s0 in range(0, len(mine), 64):  # staged through pinned memory in chunks
                pool[s0:s0 + 64].copy_(src.index_select(0, idx[s0:s0 + 64]), non_blocking=False)
            self.pools[b], self.strides[b] = pool, store.stride(b)
            local[b] = ipc_export(pool.data_ptr()) if world_size > 1 else None
        self.device_bytes = sum(p.numel() for p in self.pools.values())
        self._opened = []
        self.bases = {b: [0] * world_size for b in self.bits}
        if world_size > 1:
            allh = [None] * world_size
            dist.all_gather_object(allh, local)
            for r in range(world_size):
                for b in self.bits:
                    if r == rank:
                        self.bases[b][r] = self.pools[b].data_ptr()
                    else:
                        base, ptr = ipc_open(*allh[r][b])
                        self._opened.append(base)
                        self.bases[b][r] = ptr
        else:
            for b in self.bits:
                self.bases[b][0] = self.pools[b].data_ptr()

    def sources(self, bits: int) -> list:
        """Source pointer of every (l, e) at this width: its home rank's pool slot."""
        return source_table(self.cfg.num_layers, self.cfg.num_experts, self.world, self.bases[bits],
                            self.strides[bits])

    def attach(self, engine) -> None:
        for b in self.bits:
            engine.set_expert_sources(b, self.sources(b))

    def detach(self, engine) -> None:
        for b in self.bits:
            engine.set_expert_sources(b, None)

    def close(self) -> None:
        import ctypes as C

        from . import _lib
        for base in self._opened:
            _lib.lib().fate_ipc_close(C.c_void_p(base))
        self._opened = []
        self.pools = {}


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
