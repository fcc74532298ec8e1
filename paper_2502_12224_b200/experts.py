"""Expert weights: synthetic random-init experts, quantized on the GPU (K5) into
pinned host pools that the engine streams from.

The reference has no expert weights at all ("no model weights
stored in traces"); Fate keeps an INT2 and an INT4 copy of every expert in
CPU memory (PAPER §4.5).  ``ExpertStore`` realises that: for
each requested bit width one pinned host tensor [L*E, stride] holding every
expert's packed buffer (256-byte header + the reference's group-64 affine
format, byte-identical codes to quant.quantize), plus the shared experts
resident in HBM (they are part of ``dense_bytes``).

Weights are N(0, 1) * init_scale fp32, drawn per (layer, expert) from a
seeded CUDA generator, so any expert can be regenerated bit-for-bit for the
parity tests.
"""

from __future__ import annotations

import os

import torch

from . import ops
from .core import ModelConfig
from .errors import InvalidConfig


def _align(x: int, a: int = 4096) -> int:
    return (x + a - 1) // a * a


def shared_host_pool(name: str, nbytes: int, create: bool) -> torch.Tensor:
    """A uint8 host tensor backed by the POSIX shared-memory segment
    /dev/shm/<name> (MAP_SHARED): every process of the node that maps the same
    name sees the same bytes, so one physical copy of the expert pools serves all
    ranks.  ``create`` sizes the segment; the others only map it."""
    path = os.path.join("/dev/shm", name)
    if create:
        with open(path, "wb") as fh:
            fh.truncate(nbytes)
    elif os.path.getsize(path) != nbytes:
        raise InvalidConfig(f"shared pool {path} has {os.path.getsize(path)} bytes, expected {nbytes}")
    return torch.from_file(path, shared=True, size=nbytes, dtype=torch.uint8)


def register_host(t: torch.Tensor) -> None:
    """Page-lock an existing host mapping for this process (cudaHostRegister,
    portable), so the copy engines DMA from it like from pinned memory."""
    from . import _lib
    import ctypes as C
    _lib.check(_lib.lib().fate_host_register(C.c_void_p(t.data_ptr()), C.c_int64(t.numel())), "fate_host_register")


def unregister_host(t: torch.Tensor) -> None:
    from . import _lib
    import ctypes as C
    _lib.lib().fate_host_unregister(C.c_void_p(t.data_ptr()))


class ExpertStore:
    """``shm``: name prefix of node-wide shared host pools (``shared_host_pool``):
    the rank with ``shm_owner`` True creates and fills them, the others map the
    same segments once ``barrier`` (e.g. torch.distributed.barrier) returns, and
    every rank page-locks its mapping.  Without ``shm`` each store pins a private
    pool."""

    def __init__(self, cfg: ModelConfig, bits=(4, 2), seed: int = 0, shared_intermediate: int = 0,
                 shared_bits: int = 16, init_scale: float = 0.02, device=None, chunk: int = 32,
                 shm: str | None = None, shm_owner: bool = True, barrier=None):
        self.cfg = cfg
        self.H, self.I = cfg.hidden_dim, cfg.intermediate_dim
        if self.I * 6 * self.H != cfg.expert_bytes[16]:
            raise InvalidConfig("expert_bytes[16] must equal 2 * 3 * hidden_dim * intermediate_dim")
        self.seed, self.scale = int(seed), float(init_scale)
        self.shared_intermediate, self.shared_bits = int(shared_intermediate), int(shared_bits)
        self.device = device or ops.device()
        self.bits = tuple(sorted(set(int(b) for b in bits), reverse=True))
        self._pool: dict[int, torch.Tensor] = {}
        self._stride: dict[int, int] = {}
        self._registered: list = []
        self.shm = shm
        L, E = cfg.num_layers, cfg.num_experts
        for b in self.bits:
            nb = ops.expert_buffer_bytes(self.H, self.I, b)
            if b in cfg.expert_bytes and nb - 256 != cfg.expert_bytes[b]:
                raise InvalidConfig(f"expert_bytes[{b}]={cfg.expert_bytes[b]} != packed payload {nb - 256}")
            self._stride[b] = _align(nb)
            if shm:
                if shm_owner:
                    flat = shared_host_pool(f"{shm}_{b}", L * E * self._stride[b], True)
                    register_host(flat)
                    self._registered.append(flat)
                    self._pool[b] = flat.view(L * E, self._stride[b])
            else:
                self._pool[b] = torch.empty((L * E, self._stride[b]), dtype=torch.uint8, pin_memory=True)
        if not shm or shm_owner:
            self._fill(chunk)
        if shm:
            torch.cuda.synchronize()
            if barrier is not None:
                barrier()  # the owner's pools are complete
            if not shm_owner:
                for b in self.bits:
                    flat = shared_host_pool(f"{shm}_{b}", L * E * self._stride[b], False)
                    register_host(flat)
                    self._registered.append(flat)
                    self._pool[b] = flat.view(L * E, self._stride[b])
        self._shared = []
        if self.shared_intermediate:
            for l in range(L):
                w1, w3, w2 = self.shared_weights(l)
                self._shared.append(ops.pack_expert(w1, w3, w2, self.shared_bits, l, -1))
        torch.cuda.synchronize()

    # -- weights ------------------------------------------------------------
    def _gen(self, key: int) -> torch.Generator:
        g = torch.Generator(device=self.device)
        g.manual_seed((self.seed * 1_000_003 + key) & 0x7FFFFFFFFFFFFFFF)
        return g

    def _draw(self, key: int, I: int):
        g = self._gen(key)
        H, s = self.H, self.scale
        w1 = torch.randn((I, H), generator=g, device=self.device, dtype=torch.float32) * s
        w3 = torch.randn((I, H), generator=g, device=self.device, dtype=torch.float32) * s
        w2 = torch.randn((H, I), generator=g, device=self.device, dtype=torch.float32) * s
        return w1, w3, w2

    def weights(self, layer: int, expert: int):
        """fp32 (w1 [I,H], w3 [I,H], w2 [H,I]) of a routed expert, on device."""
        return self._draw(layer * self.cfg.num_experts + expert, self.I)

    def shared_weights(self, layer: int):
        return self._draw(10_000_000 + layer, self.shared_intermediate)

    def _fill(self, chunk: int) -> None:
        L, E = self.cfg.num_layers, self.cfg.num_experts
        for b in self.bits:
            stage = torch.empty((chunk, self._stride[b]), dtype=torch.uint8, device=self.device)
            for start in range(0, L * E, chunk):
                n = min(chunk, L * E - start)
                for i in range(n):
                    le = start + i
                    w1, w3, w2 = self.weights(le // E, le % E)
                    ops.pack_expert(w1, w3, w2, b, le // E, le % E, out=stage[i])
                self._pool[b][start:start + n].copy_(stage[:n], non_blocking=False)

    # -- accessors ------------------------------------------------------------
    def host_pool(self, bits: int) -> torch.Tensor:
        if bits not in self._pool:
            raise InvalidConfig(f"expert store has no {bits}-bit copy (built: {self.bits})")
        return self._pool[bits]

    def stride(self, bits: int) -> int:
        return self._stride[bits]

    def shared_buffer(self, layer: int) -> torch.Tensor | None:
        return self._shared[layer] if self._shared else None

    def packed(self, layer: int, expert: int, bits: int) -> torch.Tensor:
        """The host copy of one expert's packed buffer (a view into the pinned pool)."""
        nb = ops.expert_buffer_bytes(self.H, self.I, bits)
        return self.host_pool(bits)[layer * self.cfg.num_experts + expert, :nb]

    def host_bytes(self) -> int:
        return sum(p.numel() for p in self._pool.values())

    def close(self) -> None:
        """Unregister shared pools (the segments stay until ``remove_shared``)."""
        for t in self._registered:
            unregister_host(t)
        self._registered = []

    def remove_shared(self) -> None:
        """Delete this store's /dev/shm segments (owner, after every rank closed)."""
        if self.shm:
            for b in self.bits:
                p = os.path.join("/dev/shm", f"{self.shm}_{b}")
                if os.path.exists(p):
                    os.remove(p)
