"""Two ranks on one GPU (torch.distributed.run, gloo for the host-side exchange):
the node-wide shared /dev/shm expert pool and the expert-sharded peer-fetch mode
at world_size 2 over CUDA IPC, checked for bit-identical decisions
and outputs against the single-process host-fetch run."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_shared_pool_and_ipc_peer_fetch(tmp_path):
    out = os.path.join(tmp_path, "mp.json")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mp_two_rank_worker.py"), out]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.load(open(out))
    assert len(res) == 2
    for x in res:
        assert x["shared_pool_bytes_equal"] and x["schedule_equals_reference"], x
        assert x["peer_decisions_equal"] and x["peer_y_equal"], x
        assert x["h2d_bytes_peer"] == 0 and x["d2d_bytes_peer"] > 0, x
    assert res[0]["y_checksum"] == res[1]["y_checksum"]
