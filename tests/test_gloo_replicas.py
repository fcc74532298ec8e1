"""World-size-2 gloo test of the replica plumbing (CPU, no GPU needed).

Each rank plays one GPU: its own request stream (seed = rank), its own cache
plan, the timing-independent decode schedule computed by the oracle, then the
end-of-run aggregation (sum tokens, max time, summed counters)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import fate_oracle as O
    from paper_2502_12224_b200 import core, gatesim, replicas
    r, ws, lr = replicas.world()
    cfg = core.ModelConfig.from_shape(4, 8, 2, 256, 512, 1)
    tr, w = gatesim.gen_trace(cfg, gatesim.GenConfig(seed=replicas.replica_seed(r), num_tokens=8))
    _, g, ch = tr.dense_arrays(cfg)
    caps = O.plan_capacities(4, 8, 1, 12)
    sched = O.decode_schedule(g, ch.tolist(), np.stack(w.matrices), np.array(w.temperatures), caps, 2, 0,
                              O.StrategyKnobs(), 4)
    agg = replicas.aggregate(tokens=8, seconds=1.0 + r, counters={"hits": sched["cache_hits"]})
    mine = [(l, e) for (l, e) in replicas.shard_experts(4, 8, r, ws)]
    q.put((r, agg, sched["cache_hits"], len(mine), int(ch[0, 0, 0])))
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, h0, n0, c0), (r1, a1, h1, n1, c1) = out
    assert a0 == a1                                   # every rank sees the same aggregate
    assert a0["tokens"] == 16 and a0["seconds"] == 2.0  # sum of tokens, max of times
    assert a0["tokens_per_s"] == 8.0
    assert a0["hits"] == h0 + h1
    assert n0 + n1 == 32 and n0 == 16                 # expert homes partition (l*E+e) mod G
    from paper_2502_12224_b200 import replicas
    assert replicas.home_rank(1, 3, 8, 2) == 1


@pytest.mark.parametrize("L,E,G", [(24, 60, 1), (24, 60, 2), (28, 64, 8), (4, 8, 3)])
def test_shard_layout_partitions_and_addresses(L, E, G):
    # expert-sharded peer-fetch mode: every expert has exactly one home slot,
    # homes are balanced, and source addresses never collide
    from paper_2502_12224_b200.replicas import home_rank, shard_layout, source_table
    homes, slot = shard_layout(L, E, G)
    assert sorted(le for h in homes for le in h) == [(l, e) for l in range(L) for e in range(E)]
    sizes = [len(h) for h in homes]
    assert max(sizes) - min(sizes) <= 1
    for r, h in enumerate(homes):
        assert all(home_rank(l, e, E, G) == r for (l, e) in h)
        assert [slot[le] for le in h] == list(range(len(h)))
    stride = 4096
    bases = [(r + 1) << 40 for r in range(G)]
    tab = source_table(L, E, G, bases, stride)
    assert len(tab) == L * E and len(set(tab)) == L * E
    for l in range(L):
        for e in range(E):
            r = home_rank(l, e, E, G)
            assert tab[l * E + e] == bases[r] + slot[(l, e)] * stride


def _shm_worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2502_12224_b200.experts import shared_host_pool
    n = 1 << 20
    if rank == 0:
        t = shared_host_pool(name, n, True)
        t[:] = torch.arange(n, dtype=torch.int64).remainder(251).to(torch.uint8)
    dist.barrier()
    if rank != 0:
        t = shared_host_pool(name, n, False)
    ok = bool(torch.equal(t, torch.arange(n, dtype=torch.int64).remainder(251).to(torch.uint8)))
    dist.barrier()
    if rank == 1:
        t[0] = 77  # a write by one rank is seen by the other (one physical copy)
    dist.barrier()
    seen = int(t[0])
    q.put((rank, ok, seen))
    dist.barrier()
    if rank == 0:
        os.remove(os.path.join("/dev/shm", name))
    dist.destroy_process_group()


def test_shared_host_pool_one_copy_across_ranks():
    """The node-wide expert pool: every rank maps the same /dev/shm
    segment, so the pinned host copy exists once per node instead of once per rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    name = f"fate_gloo_shm_{port}"
    ps = [ctx.Process(target=_shm_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert out == [(0, True, 77), (1, True, 77)]
