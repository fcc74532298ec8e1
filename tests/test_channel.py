"""The standalone transfer channel (fate_channel_*, SURVEY §8b prefetch_{enqueue,
promote, drop_stale, wait}): its queue semantics equal the reference's _Channel
(pipeline.py:163-264) on 60 random operation sequences (CPU, bookkeeping mode),
and on the GPU it moves real bytes in queue order, never copies a dropped
prefetch, and orders a consumer stream after a transfer."""
import json
import os

import pytest

from golden_util import GOLDEN_DIR


def test_channel_queue_matches_reference():
    from paper_2502_12224_b200.channel import Channel
    with open(os.path.join(GOLDEN_DIR, "golden_harness.json")) as fh:
        cases = json.load(fh)["channel"]
    for case in cases:
        ch = Channel(device=None)
        for op, want in zip(case["ops"], case["pending"]):
            if op[0] == "enqueue":
                ch.enqueue(op[1], op[2], op[3], op[4], 4)
            elif op[0] == "promote":
                ch.promote_ondemand()
            else:
                ch.drop_stale((op[1], op[2]))
            assert [t.id for t in ch.pending] == want, (case["ops"], op)
        ch.close()


@pytest.mark.gpu
def test_channel_copies_in_queue_order_on_device():
    import torch
    from paper_2502_12224_b200.channel import Channel
    n = 1 << 20
    src = [torch.full((n,), i + 1, dtype=torch.uint8).pin_memory() for i in range(5)]
    dst = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(5)]
    ch = Channel(device=torch.cuda.current_device(), max_inflight=2)
    ts = [ch.enqueue("prefetch" if i < 3 else "ondemand", 0, 1, i, 4, src[i].data_ptr(), dst[i].data_ptr(), n)
          for i in range(5)]
    ch.promote_ondemand()
    assert [t.expert for t in ch.pending] == [3, 4, 0, 1, 2]
    assert ch.drop_stale((0, 0)) == 0 and ch.drop_stale((0, 1)) == 3  # the three prefetches of step (0, 1)
    s = torch.cuda.Stream()
    ch.completion(ts[4], s)  # starts 3 then 4 in queue order; s waits for 4
    with torch.cuda.stream(s):
        out = dst[4].float().sum()
    torch.cuda.synchronize()
    assert float(out) == 5.0 * n and int(dst[3][0]) == 4
    assert all(int(dst[i].sum()) == 0 for i in range(3))  # dropped prefetches never copied
    assert ch.find(0, 1, 4)[0] == "done" and ch.find(0, 1, 0)[0] is None
    with pytest.raises(Exception):
        ch.completion(ts[0], s)  # vanished from the queue (pipeline.py:230)
    ch.close()
