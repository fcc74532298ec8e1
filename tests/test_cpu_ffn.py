"""The CPU baseline's vectorised FFN (oracle/ffn_cpu.c, AVX2) against the fp64
oracle on buffers packed in numpy with the reference's quantization (CPU only)."""

import numpy as np
import pytest

from oracle import fate_oracle as O


@pytest.mark.parametrize("H,I,bits_list", [(256, 512, [4, 2]), (256, 384, [16, 8]), (512, 256, [2, 4, 16])])
def test_cpu_ffn_matches_oracle(H, I, bits_list):
    rng = np.random.default_rng(11)
    lib = O.cpu_lib()
    bufs, ws, refs = [], [], []
    for j, b in enumerate(bits_list):
        w1, w3 = (rng.standard_normal((I, H)) * 0.02 for _ in range(2))
        w2 = rng.standard_normal((H, I)) * 0.02
        buf = O.pack_buffer(w1, w3, w2, b)
        u = O.unpack_buffer(buf, H, I, b)
        if b != 16:  # the numpy packer and the unpacker agree with quantize on the original W2
            codes, _, _ = O.quantize(w2, b)
            np.testing.assert_array_equal(u["codes2"], codes)
        bufs.append(buf)
        ws.append(0.3 + 0.1 * j)
        refs.append(u)
    x = rng.standard_normal(H).astype(np.float32)
    scratch = np.empty(O.cpu_scratch_floats(H, [I] * len(bits_list)), np.float32)
    y = O.cpu_ffn(lib, x, bufs, [I] * len(bufs), bits_list, ws, scratch).astype(np.float64)
    xd = x.astype(np.float64)
    want = sum(np.float32(w) * O.ffn_swiglu(xd, r["w1"], r["w3"], r["w2"]) for w, r in zip(ws, refs))
    rel = np.linalg.norm(y - want) / np.linalg.norm(want)
    assert rel < 2e-5, rel
