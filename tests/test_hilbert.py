"""The tile path's point-sort key (csrc/pf_tile.cu, hilbert_key): a 24-state automaton of the 3-D
Hilbert curve of Skilling's transpose algorithm ("Programming the Hilbert curve", AIP Conf. Proc.
707, 2004). The automaton replaced a direct transcription of the transpose loops on the device (it
issues ~3x fewer instructions); the sort order, and with it every tile, must be unchanged.

CPU: the exported table (pf_hilbert_table) walked in numpy equals the transpose algorithm on every
cell of the 2^7 and 2^8 grids (the sort's two grid orders). GPU: pf_hilbert_keys (the sort's own
kernel) equals it on seeded points, including the cell clamping at the bbox faces.
"""

import ctypes as C

import numpy as np
import pytest

from paper_2511_03126_b200 import _lib


def skilling_keys(x, y, z, bits):
    """Skilling's AxestoTranspose + bit interleave, vectorised (uint32 cell coordinates)."""
    X = [np.asarray(a, np.uint32).copy() for a in (x, y, z)]
    Q = 1 << (bits - 1)
    while Q > 1:
        pm = np.uint32(Q - 1)
        for i in range(3):
            bit = (X[i] & np.uint32(Q)) != 0
            t = (X[0] ^ X[i]) & pm
            x0 = np.where(bit, X[0] ^ pm, X[0] ^ t)
            if i:
                X[i] = np.where(bit, X[i], X[i] ^ t)
            X[0] = x0
        Q >>= 1
    X[1] ^= X[0]
    X[2] ^= X[1]
    t = np.zeros_like(X[0])
    Q = 1 << (bits - 1)
    while Q > 1:
        t ^= np.where((X[2] & np.uint32(Q)) != 0, np.uint32(Q - 1), np.uint32(0))
        Q >>= 1
    X = [a ^ t for a in X]
    key = np.zeros_like(X[0])
    for b in range(bits - 1, -1, -1):
        for a in range(3):
            key = (key << np.uint32(1)) | ((X[a] >> np.uint32(b)) & np.uint32(1))
    return key


def table():
    buf = (C.c_uint8 * 192)()
    ns = _lib.load().pf_hilbert_table(C.cast(buf, C.c_void_p), 192)
    assert ns == 24
    return np.frombuffer(bytes(buf), np.uint8).astype(np.uint32)


def fsm_keys(tab, x, y, z, bits):
    s8 = np.zeros(np.shape(x), np.uint32)
    key = np.zeros(np.shape(x), np.uint32)
    for b in range(bits - 1, -1, -1):
        o = (((x >> b) & 1) << 2) | (((y >> b) & 1) << 1) | ((z >> b) & 1)
        e = tab[s8 | o]
        key = (key << np.uint32(3)) | (e & np.uint32(7))
        s8 = e & np.uint32(~7 & 0xFF)
    return key


@pytest.mark.parametrize("bits", [7, 8])
def test_table_is_the_transpose_curve_on_every_cell(bits):
    tab = table()
    g = np.arange(1 << bits, dtype=np.uint32)
    x, y, z = (a.ravel() for a in np.meshgrid(g, g, g, indexing="ij"))
    want = skilling_keys(x, y, z, bits)
    got = fsm_keys(tab, x, y, z, bits)
    assert np.array_equal(got, want)
    # a Hilbert curve: every key once, consecutive keys are face-adjacent cells
    order = np.argsort(want, kind="stable")
    assert np.array_equal(want[order], np.arange(1 << (3 * bits), dtype=np.uint32))
    step = np.abs(np.diff(x[order].astype(np.int64))) + np.abs(np.diff(y[order].astype(np.int64))) + \
        np.abs(np.diff(z[order].astype(np.int64)))
    assert np.all(step == 1)


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [7, 8])
def test_device_keys_match(cuda, bits):
    import torch

    rng = np.random.default_rng(5 + bits)
    pts = rng.normal(0.0, 0.3, (300_000, 3)).astype(np.float32)
    pts[:7] = [[-1, -1, -1], [1, 1, 1], [0, 0, 0], [-1, 1, -1], [1, -1, 1], [0.5, -1, 0.25], [1, 0, -1]]
    lo = pts.min(0).astype(np.float64)
    hi = pts.max(0).astype(np.float64)
    lo_hi = np.concatenate([lo, hi])
    dp = torch.from_numpy(pts).cuda()
    dlh = torch.from_numpy(lo_hi).cuda()
    keys = torch.empty(len(pts), dtype=torch.int32, device="cuda")
    _lib.call("pf_hilbert_keys", dp.data_ptr(), len(pts), dlh.data_ptr(), bits, keys.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = keys.cpu().numpy().view(np.uint32)
    # the kernel's cell mapping in fp32: c = clamp(int((p - lo) * (2^bits / ext)), 0, 2^bits - 1)
    cells = 1 << bits
    lo32 = lo.astype(np.float32)
    ext = np.float32(max(np.float32(hi[0] - lo[0]), np.float32(hi[1] - lo[1]), np.float32(hi[2] - lo[2])))
    inv = np.float32(cells) / ext
    c = np.clip(((pts - lo32).astype(np.float32) * inv).astype(np.float32).astype(np.int64), 0, cells - 1)
    want = skilling_keys(c[:, 0], c[:, 1], c[:, 2], bits)
    assert np.array_equal(got, want)
