"""The checksums of tests/digest.py agree across their implementations: numpy,
torch (CPU) and the oracle's digest mode (``oracle.trace_digest``) over the same
trace, so a full-size golden digest written by the oracle can be compared with a
digest the GPU tests compute from the library's arrays."""
import numpy as np
import torch

import dmtz_inputs as di
import oracle
from tests import digest as dg


def test_digest_numpy_equals_torch():
    rng = np.random.default_rng(0)
    x = rng.integers(0, 2 ** 63, 10007, dtype=np.int64).view(np.uint64) | np.uint64(1 << 63)
    assert dg.digest_np(x, start=5) == dg.digest_t(torch.from_numpy(x.view(np.int64)), start=5)
    f = rng.standard_normal(5000).astype(np.float32)
    assert dg.digest_np(f) == dg.digest_t(torch.from_numpy(f))
    assert dg.digest_np(f) == dg.digest_np(f, chunk=333)
    assert dg.digest_t(torch.from_numpy(f), chunk=77) == dg.digest_t(torch.from_numpy(f))
    k = rng.integers(0, 256, 999).astype(np.uint8)
    assert dg.digest_np(k.astype(np.uint64)) == dg.digest_t(torch.from_numpy(k))
    # order-sensitive: swapping two distinct entries changes the digest
    y = x.copy()
    y[[3, 4]] = y[[4, 3]]
    assert dg.digest_np(y) != dg.digest_np(x)


def test_digest_splitmix_known_value():
    # splitmix64 finalizer of 0x9E3779B97F4A7C15 (the first output of splitmix64 seeded with 0)
    assert dg.digest_np(np.array([0, 0x9E3779B97F4A7C15], np.uint64)[1:], start=0) == 0xE220A8397B1DCDAF


def test_oracle_digest_mode_equals_stored_trace():
    for shape, seed in (((9, 11, 10), 3), ((20, 23), 4)):
        f = di.field("noise", shape, seed)
        t = oracle.trace(f)
        nb, nc, d = oracle.trace_digest(f)
        assert nb == len(t["origin"]) and nc == len(t["cells"])
        assert d == dg.csr_digest_np(t)
