"""Edit-stream codec, plain Python -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Written from the version-1 format in include/dmtz.h (which restates P:276-280: store the
integer count q per edited vertex; lossless entries keep their value bits), one
record at a time, with no blocking beyond what the format defines.  Shares no code with
the CUDA encoder (paper_2409_17346_b200/csrc/dmtz_codec.cuh)."""
from __future__ import annotations

import struct

import numpy as np

BLOCK = 4096


def _varint(x: int) -> bytes:
    out = bytearray()
    while True:
        b = x & 0x7F
        x >>= 7
        if x:
            out.append(b | 0x80)
        else:
            out.append(b)
            return bytes(out)


def _rel(fh: float, value: float) -> int:
    """version 2: zigzag of int64(fhat bits as int32) - int64(value bits as int32)"""
    d = int(np.float32(fh).view(np.int32)) - int(np.float32(value).view(np.int32))
    return (d << 1) if d >= 0 else ((-d) << 1) - 1


def encode(edits: np.ndarray, xi: float, q_max: int, fhat=None) -> bytes:
    """edits: structured array (v, q, lossless, value) sorted by v; fhat given -> version 2
    (lossless values relative to fhat), else version 1."""
    n = len(edits)
    nblocks = (n + BLOCK - 1) // BLOCK
    payload = bytearray()
    offsets = []
    prev = None
    for i in range(n):
        v, q, ll = int(edits["v"][i]), int(edits["q"][i]), int(edits["lossless"][i])
        if i % BLOCK == 0:
            offsets.append(len(payload))
            delta = v
        else:
            assert v > prev
            delta = v - prev - 1
        payload += _varint(delta) + _varint((q << 1) | ll)
        if ll:
            if fhat is None:
                payload += np.float32(edits["value"][i]).tobytes()
            else:
                payload += _varint(_rel(np.asarray(fhat).ravel()[v], edits["value"][i]))
        prev = v
    head = b"DMTE" + struct.pack("<IQIifI", 1 if fhat is None else 2, n, BLOCK, q_max, np.float32(xi), nblocks)
    return head + b"".join(struct.pack("<Q", o) for o in offsets) + bytes(payload)


def decode(data: bytes, fhat=None):
    """-> (edits structured array, xi, q_max); version 2 needs fhat."""
    from oracle import EDIT_DTYPE
    assert data[:4] == b"DMTE"
    ver, n, blk, q_max, xi, nblocks = struct.unpack("<IQIifI", data[4:32])
    assert ver in (1, 2) and blk == BLOCK and nblocks == (n + BLOCK - 1) // BLOCK
    assert ver == 1 or fhat is not None
    pos = 32 + 8 * nblocks
    out = np.zeros(n, EDIT_DTYPE)
    v = -1

    def get():
        nonlocal pos
        x, sh = 0, 0
        while True:
            b = data[pos]
            pos += 1
            x |= (b & 0x7F) << sh
            sh += 7
            if not b & 0x80:
                return x

    for i in range(n):
        d = get()
        v = d if i % BLOCK == 0 else v + d + 1
        code = get()
        out["v"][i], out["q"][i], out["lossless"][i] = v, code >> 1, code & 1
        if code & 1:
            if ver == 1:
                out["value"][i] = np.frombuffer(data[pos:pos + 4], "<f4")[0]
                pos += 4
            else:
                z = get()
                d = (z >> 1) if not z & 1 else -((z + 1) >> 1)
                fb = int(np.float32(np.asarray(fhat).ravel()[v]).view(np.int32))
                out["value"][i] = np.int32(fb - d).view(np.float32)
    assert pos == len(data)
    return out, float(xi), q_max


def apply(fhat: np.ndarray, edits: np.ndarray, xi: float, q_max: int) -> np.ndarray:
    """Decompression side (Fig. 2): g = fhat with each edit replayed by Eq. 2 from fhat
    in float32 with two roundings, lossless entries by their bits."""
    g = np.array(fhat, np.float32, copy=True).ravel()
    step = np.float32(np.ldexp(np.float32(xi), -q_max))
    fl = np.asarray(fhat, np.float32).ravel()
    for e in edits:
        v = int(e["v"])
        g[v] = np.float32(e["value"]) if e["lossless"] else np.float32(fl[v] - np.float32(np.float32(e["q"]) * step))
    return g.reshape(np.shape(fhat))
