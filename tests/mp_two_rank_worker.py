"""Worker of tests/test_gpu_multirank.py (launched by torch.distributed.run with two
ranks on ONE GPU, gloo for the host-side exchange): both ranks map one shared
/dev/shm expert pool (filled by rank 0), decode the same trace, then run the
expert-sharded peer-fetch mode at world_size 2 over CUDA IPC.  Rank 0 writes the
verdict JSON to the path in argv[1]."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main(out_path):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    from golden_util import config_traces, golden
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    from paper_2502_12224_b200.replicas import ExpertShards
    e = golden()["schedules"]["tiny"]
    cfg, dec, pre, w = config_traces("tiny")
    shm = f"fate_mp_test_{os.environ['MASTER_PORT']}"
    store = ExpertStore(cfg, bits=(4, 2), seed=0, shm=shm, shm_owner=rank == 0, barrier=dist.barrier)
    ref = ExpertStore(cfg, bits=(4, 2), seed=0)  # private pinned pool, same weights
    same_bytes = all(torch.equal(store.host_pool(b), ref.host_pool(b)) for b in (4, 2))
    want = e["decode_cold"]
    eng = OffloadEngine(cfg, e["plan"], store, w, StrategyKnobs(budget_n=want["n"]), max_tokens=64)
    _, g, ch = dec.dense_arrays(cfg)
    gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
    host = eng.decode(gd, chd, want_logs=True)
    keys = ("chosen", "hits", "ondemand", "victims")
    sched_ok = all(tuple(a[k] for k in keys) == tuple(b[k] for k in keys) and a.get("pred") == b.get("pred")
                   for a, b in zip(host.logs, want["steps"]))
    # expert-sharded mode, world_size 2: half the experts homed on each rank, the
    # other half mapped from the peer process over CUDA IPC
    shards = ExpertShards(store, bits=(4, 2), rank=rank, world_size=world)
    eng.reset_cache()
    shards.attach(eng)
    peer = eng.decode(gd, chd, want_logs=True)
    peer_same = all(tuple(a[k] for k in keys) == tuple(b[k] for k in keys) for a, b in zip(peer.logs, host.logs))
    y_same = bool(torch.equal(peer.y, host.y))
    res = {"rank": rank, "shared_pool_bytes_equal": same_bytes, "schedule_equals_reference": sched_ok,
           "peer_decisions_equal": peer_same, "peer_y_equal": y_same, "h2d_bytes_peer": peer.stats["h2d_bytes"],
           "d2d_bytes_peer": peer.stats["d2d_bytes"], "y_checksum": float(host.y.double().sum().item())}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    shards.detach(eng)
    dist.barrier()  # no rank unmaps a peer pool while the other still copies from it
    shards.close()
    eng.close()
    store.close()
    dist.barrier()
    if rank == 0:
        store.remove_shared()
        with open(out_path, "w") as fh:
            json.dump(allres, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
