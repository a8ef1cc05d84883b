"""Order-sensitive 64-bit checksums of result arrays (test infrastructure).

digest(X) = sum_i mix(X[i] ^ (i * 0x9E3779B97F4A7C15)) mod 2^64, mix = the
splitmix64 finalizer.  The full-size oracle goldens (tests/golden/oracle_full_*.json,
written by tools/oracle_goldens.py) hold digests because the C4 separatrix CSR
(~50 GB) does not fit in the build host's memory; ``oracle/dmtz_oracle.c``
computes the same sums while it traces (digest mode), and the GPU tests apply
these functions to the library's output arrays.  A checksum of outputs, not part
of the method; pinned against the oracle's digest mode in tests/test_digest.py.

Two implementations: numpy (uint64, wrap-around) and torch (int64 on any device,
logical shifts by masking; two's-complement wrap-around of * and sum).
"""
from __future__ import annotations

import numpy as np

GOLD = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1


def _s64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


# ---------------------------------------------------------------- numpy ----
def _mix_np(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(M1)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def digest_np(x: np.ndarray, start: int = 0, chunk: int = 1 << 24) -> int:
    """digest of a 1-D integer array (values zero-extended to 64 bits)."""
    x = np.ascontiguousarray(x).reshape(-1)
    if x.dtype.kind == "f":
        x = x.view(np.uint32 if x.dtype.itemsize == 4 else np.uint64)
    acc = 0
    with np.errstate(over="ignore"):
        for a in range(0, x.size, chunk):
            xs = x[a:a + chunk].astype(np.uint64)
            idx = np.arange(start + a, start + a + xs.size, dtype=np.uint64) * np.uint64(GOLD)
            acc = (acc + int(_mix_np(xs ^ idx).sum(dtype=np.uint64))) & MASK64
    return acc


# ---------------------------------------------------------------- torch ----
def _lsr(z, k: int):
    import torch
    return torch.bitwise_and(torch.bitwise_right_shift(z, k), (1 << (64 - k)) - 1)


def _mix_t(z):
    z = z ^ _lsr(z, 30)
    z = z * _s64(M1)
    z = z ^ _lsr(z, 27)
    z = z * _s64(M2)
    return z ^ _lsr(z, 31)


def digest_t(x, start: int = 0, chunk: int = 1 << 27) -> int:
    """digest of a 1-D torch tensor (any integer / float dtype, any device)."""
    import torch
    x = x.reshape(-1)
    if x.dtype == torch.float32:
        x = x.view(torch.int32)
    unsigned32 = x.dtype in (torch.int32, torch.float32)
    acc = 0
    for a in range(0, x.numel(), chunk):
        xs = x[a:a + chunk].to(torch.int64)
        if unsigned32:
            xs = torch.bitwise_and(xs, 0xFFFFFFFF)
        elif x.dtype in (torch.int16,):
            xs = torch.bitwise_and(xs, 0xFFFF)
        elif x.dtype in (torch.int8,):
            xs = torch.bitwise_and(xs, 0xFF)
        idx = torch.arange(start + a, start + a + xs.numel(), dtype=torch.int64, device=xs.device) * _s64(GOLD)
        acc = (acc + int(_mix_t(xs ^ idx).sum().item())) & MASK64
    return acc


def plane_digests_t(g, planes: int) -> list:
    """digest of each z-plane of a float32 field (global element indices)."""
    flat = g.reshape(-1)
    per = flat.numel() // planes
    return [digest_t(flat[z * per:(z + 1) * per], start=z * per) for z in range(planes)]


def csr_digest_np(t: dict) -> dict:
    """digests of an oracle.trace() result (numpy arrays)."""
    return {"offsets": digest_np(t["offsets"].astype(np.int64).view(np.uint64)),
            "cells": digest_np(t["cells"]), "origin": digest_np(t["origin"]),
            "terminal": digest_np(t["terminal"]), "kind": digest_np(t["kind"].astype(np.uint64))}
