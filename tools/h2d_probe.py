"""H2D copy patterns for the on-demand experts of a decode step (3.24 MB INT2
buffers): one stream sequential, two streams alternating whole copies, two
streams each copying half of every expert concurrently, four quarter copies."""
import json
import torch

n, k, reps = 3244032 + 256, 3, 50
src = torch.empty((k, n), dtype=torch.uint8).pin_memory()
dst = torch.empty((k, n), dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
out = {}


def run(pattern):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for _ in range(reps):
        if pattern == "1stream":
            with torch.cuda.stream(streams[0]):
                for i in range(k):
                    dst[i].copy_(src[i], non_blocking=True)
        elif pattern == "2stream_alternate":
            for i in range(k):
                with torch.cuda.stream(streams[i % 2]):
                    dst[i].copy_(src[i], non_blocking=True)
        else:
            parts = 2 if pattern == "2stream_halves" else 4
            step = (n + parts - 1) // parts
            for i in range(k):
                for p in range(parts):
                    with torch.cuda.stream(streams[p]):
                        dst[i, p * step:(p + 1) * step].copy_(src[i, p * step:(p + 1) * step], non_blocking=True)
    for s in streams:
        e1.wait(s) if False else None
    ev = []
    for s in streams:
        x = torch.cuda.Event()
        x.record(s)
        ev.append(x)
    for x in ev:
        torch.cuda.current_stream().wait_event(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return reps * k * n / (ms * 1e-3) / 1e9


for p in ("1stream", "2stream_alternate", "2stream_halves", "4stream_quarters"):
    run(p)
    out[p] = max(run(p) for _ in range(3))
print(json.dumps(out))
