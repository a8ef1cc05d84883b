"""Full-size parity (``-m gpu``): the CUDA path at BASELINE.json's full sizes (C2 1800x3600,
C3 100x500x500, C4 512^3) against the CPU oracle, bit for bit, through digests.

The oracle's results at these sizes are tests/golden/oracle_full_<C>.json, written by
tools/oracle_goldens.py, which calls only ``dmtz_inputs`` and ``oracle`` (the 3D configs
in the oracle's frontier mode, itself checked equal to the literal loop in
tests/test_oracle_frontier.py).  They hold the input sha256, the C-loop's status and
statistics, order-sensitive digests (tests/digest.py) of g (whole and per z-plane)
and of the edit list, and digests of the separatrix CSR of the converged g (and of f
for C2) -- the C4 CSR (~50 GB) does not fit in the build host's memory, so the oracle
computes its digests while it traces.  Launch configuration = bench.py's."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import dmtz_inputs as di
from tests import digest as dg

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
STAT_KEYS = ("rounds", "n_edited", "n_quantized", "n_lossless", "n_false_round0", "false_by_kind_round0")


@pytest.fixture(scope="module")
def dmtz():
    import paper_2409_17346_b200 as d
    return d


def _gold(name):
    path = os.path.join(GOLDEN, f"oracle_full_{name}.json")
    if not os.path.exists(path):
        pytest.fail(f"missing golden {path} (tools/oracle_goldens.py {name})")
    return json.load(open(path))


def _csr_digests(tr):
    return {"offsets": dg.digest_t(tr["offsets"]), "cells": dg.digest_t(tr["cells"]),
            "origin": dg.digest_t(tr["origin"]), "terminal": dg.digest_t(tr["terminal"]),
            "kind": dg.digest_t(tr["kind"])}


def _trace_digest(ctx, codes, dev):
    sizes = ctx.trace_sizes(codes)
    bufs = ctx.trace_buffers(sizes["n_branches"], sizes["n_cells"], dev)
    tr = ctx.trace_separatrices(codes, out=bufs)
    out = {"n_branches": tr["origin"].shape[0], "n_cells": tr["cells"].shape[0], "digests": _csr_digests(tr)}
    del tr, bufs
    torch.cuda.empty_cache()
    return out


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
@pytest.mark.parametrize("full_sweeps", [False, True])
def test_full_size_correct_and_trace_vs_oracle(dmtz, name, full_sweeps):
    gold = _gold(name)
    f, fh, xi, cfg = di.config_inputs(name)
    assert hashlib.sha256(f.tobytes()).hexdigest() == gold["input_sha256"]["f"]
    assert hashlib.sha256(fh.tobytes()).hexdigest() == gold["input_sha256"]["fhat"]
    assert int(np.float32(xi).view(np.uint32)) == gold["xi_bits"]
    dev = torch.device("cuda", 0)
    ctx = dmtz.Context(f.shape, dev)
    ft, fht = torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev)
    r = ctx.correct(ft, fht, xi, q_max=gold["q_max"], q_cap=gold["q_cap"], tier=gold["tier"],
                    full_sweeps=full_sweeps)
    assert r.status == gold["status"], r.message
    for k in STAT_KEYS:
        assert r.stats[k] == gold["stats"][k], k
    assert r.n_edits == gold["n_edits"]
    gbits = r.g.reshape(-1).view(torch.int32)
    if dg.digest_t(gbits) != gold["g_digest"]:
        if "g_plane_digests" in gold:
            planes = dg.plane_digests_t(gbits, f.shape[0])
            bad = [z for z, (a, b) in enumerate(zip(planes, gold["g_plane_digests"])) if a != b]
            pytest.fail(f"g differs from the oracle on {len(bad)} z-planes, first {bad[:8]}")
        pytest.fail("g differs from the oracle")
    assert dg.digest_t(r.edits.reshape(-1, 16).contiguous().view(torch.int64).reshape(-1)) == gold["edits_digest"]
    if full_sweeps:
        return   # the trace of the same g is checked once, in the default mode
    codes = ctx.compute_gradient(r.g)
    got = _trace_digest(ctx, codes, dev)
    want = gold["trace_g"]
    assert got["n_branches"] == want["n_branches"] and got["n_cells"] == want["n_cells"]
    assert got["digests"] == want["digests"]
    if "trace_f" in gold:
        got = _trace_digest(ctx, ctx.compute_gradient(ft), dev)
        want = gold["trace_f"]
        assert got["n_branches"] == want["n_branches"] and got["n_cells"] == want["n_cells"]
        assert got["digests"] == want["digests"]
