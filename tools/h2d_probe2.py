"""H2D bandwidth of 3.24 MB expert copies: from a small pinned buffer vs random
experts of a 12 GB pinned pool (torch cudaHostAlloc) vs a 12 GB anonymous mapping
advised for transparent huge pages and page-locked with cudaHostRegister."""
import ctypes as C
import json
import mmap
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = 3244032 + 256
stride = (n + 4095) // 4096 * 4096
N = 12 * 1024 ** 3 // stride
dst = torch.empty((4, n), dtype=torch.uint8, device="cuda")
rng = np.random.default_rng(0)
out = {}


def bw(src_ptrs):
    # raw-pointer copies through the engine's standalone channel (fate_channel_*)
    from paper_2502_12224_b200.channel import Channel
    ch = Channel(device=torch.cuda.current_device(), max_inflight=4)
    s = torch.cuda.current_stream()
    ts = [ch.enqueue("ondemand", 0, 0, i, 2, p, dst[i % 4].data_ptr(), n) for i, p in enumerate(src_ptrs)]
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    ch.completion(ts[-1], s)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ch.close()
    return len(src_ptrs) * n / dt / 1e9


small = torch.empty((4, stride), dtype=torch.uint8).pin_memory()
out["small_pinned"] = max(bw([small[i % 4].data_ptr() for i in range(200)]) for _ in range(3))
big = torch.empty((N, stride), dtype=torch.uint8).pin_memory()
big[:, ::4096] = 1  # touch
idx = rng.integers(0, N, size=200)
out["pool12g_pinned_random"] = max(bw([big[int(i)].data_ptr() for i in idx]) for _ in range(3))
out["pool12g_pinned_seq"] = max(bw([big[i].data_ptr() for i in range(200)]) for _ in range(3))
del big
libc = C.CDLL("libc.so.6")
m = mmap.mmap(-1, N * stride, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
addr = C.addressof(C.c_char.from_buffer(m))
MADV_HUGEPAGE = 14
out["madvise_rc"] = libc.madvise(C.c_void_p(addr), C.c_size_t(N * stride), MADV_HUGEPAGE)
arr = np.frombuffer(m, dtype=np.uint8)
arr[::4096] = 1
from paper_2502_12224_b200 import _lib  # noqa: E402
L = _lib.lib()
out["register_rc"] = L.fate_host_register(C.c_void_p(addr), C.c_int64(N * stride))
out["pool12g_thp_random"] = max(bw([addr + int(i) * stride for i in idx]) for _ in range(3))
try:
    out["thp_kb"] = [l for l in open("/proc/meminfo") if "AnonHugePages" in l][0].strip()
    out["thp_enabled"] = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
except Exception as e:
    out["thp_err"] = str(e)
print(json.dumps(out))
