"""Pins of the plain-Python edit-stream codec (oracle/edit_codec.py)."""
import json
import os

import numpy as np
import pytest

import dmtz_inputs as di
import oracle
from oracle import edit_codec as ec

GOLD = os.path.join(os.path.dirname(__file__), "golden", "edit_stream_small.json")


def _edits(rows):
    e = np.zeros(len(rows), oracle.EDIT_DTYPE)
    for i, (v, q, ll, val) in enumerate(rows):
        e[i] = (v, q, ll, 0, val)
    return e


def test_golden_bytes():
    g = json.load(open(GOLD))
    b = ec.encode(_edits(g["edits"]), g["xi"], g["q_max"])
    assert b.hex() == g["hex"].replace(" ", "")
    d, xi, qm = ec.decode(b)
    assert (xi, qm) == (g["xi"], g["q_max"]) and d.tolist() == _edits(g["edits"]).tolist()


@pytest.mark.parametrize("n,seed", [(0, 0), (1, 1), (4095, 2), (4097, 3), (9000, 4)])
def test_roundtrip(n, seed):
    rng = np.random.default_rng(seed)
    v = np.sort(rng.choice(10 ** 7, size=n, replace=False)) if n else np.zeros(0, np.int64)
    e = np.zeros(n, oracle.EDIT_DTYPE)
    e["v"] = v
    e["q"] = rng.integers(0, 65536, n)
    e["lossless"] = rng.integers(0, 2, n)
    e["value"] = np.where(e["lossless"] > 0, rng.standard_normal(n).astype(np.float32), 0)
    d, xi, qm = ec.decode(ec.encode(e, 0.125, 6))
    assert d.tobytes() == e.tobytes() and xi == 0.125 and qm == 6


def test_quantized_is_smaller():
    """10 quantized entries < 10 x 12 B key-value floats; the quantized
    stream of a C-loop result is no larger than the all-lossless stream of the same edits."""
    e = _edits([(1000 + 7 * i, 5, 0, 0.0) for i in range(10)])
    assert len(ec.encode(e, 0.1, 6)) - 32 - 8 < 10 * 12
    f, fh, xi, _ = di.config_inputs("C1")
    r = oracle.correct(f, fh, xi, q_cap=65535)
    q = ec.encode(r["edits"], xi, 6)
    ll = r["edits"].copy()
    ll["lossless"] = 1
    ll["value"] = r["g"].ravel()[ll["v"]]
    assert len(q) <= len(ec.encode(ll, xi, 6))


@pytest.mark.parametrize("q_cap", [6, 65535])
def test_apply_replays_the_cloop(q_cap):
    """Fig. 2: the decompression side rebuilds the editor's g bit for bit from fhat and the
    decoded edits."""
    f, fh, xi = di.random_case((9, 10, 11), 4, eps=0.05, family="lognormal")
    r = oracle.correct(f, fh, xi, q_cap=q_cap)
    d, x2, qm = ec.decode(ec.encode(r["edits"], xi, 6))
    g = ec.apply(fh, d, x2, qm)
    assert np.array_equal(g.view(np.uint32), r["g"].view(np.uint32))


GOLD2 = os.path.join(os.path.dirname(__file__), "golden", "edit_stream_small_v2.json")


def test_golden_bytes_v2():
    g = json.load(open(GOLD2))
    fhat = np.ones(301, np.float32)
    fhat[6] = np.uint32(int(g["fhat_bits_at_6"], 16)).view(np.float32)
    b = ec.encode(_edits(g["edits"]), g["xi"], g["q_max"], fhat=fhat)
    assert b.hex() == g["hex"].replace(" ", "")
    d, xi, qm = ec.decode(b, fhat=fhat)
    assert d.tolist() == _edits(g["edits"]).tolist()


@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_v2_roundtrip_and_size(sign):
    """relative lossless values round-trip exactly (both signs, crossing zero) and the
    C-loop's stream shrinks against version 1"""
    rng = np.random.default_rng(5)
    n = 5000
    fhat = (sign * rng.uniform(0.5, 2.0, 10 ** 5)).astype(np.float32)
    fhat[:10] = np.float32(1e-3) * sign
    e = np.zeros(n, oracle.EDIT_DTYPE)
    e["v"] = np.sort(rng.choice(10 ** 5, n, replace=False))
    e["lossless"] = 1
    e["value"] = (fhat[e["v"]] - np.float32(0.01)).astype(np.float32)
    d, _, _ = ec.decode(ec.encode(e, 0.01, 6, fhat=fhat), fhat=fhat)
    assert np.array_equal(d["value"].view(np.uint32), e["value"].view(np.uint32))
    f, fh, xi, _ = di.config_inputs("C1")
    r = oracle.correct(f, fh, xi)
    v1, v2 = ec.encode(r["edits"], xi, 6), ec.encode(r["edits"], xi, 6, fhat=fh)
    assert len(v2) < len(v1)
    d2, _, _ = ec.decode(v2, fhat=fh)
    assert np.array_equal(ec.apply(fh, d2, xi, 6).view(np.uint32), r["g"].view(np.uint32))


def test_base_size_model_entropy():
    """The SZ3 stand-in's size model (CR = original / compressed): an all-equal code
    array has zero entropy (only the code table), a uniform 4-symbol one 2 bits a value,
    and the Lorenzo codes of C1 are far below 32 bits a value."""
    f = np.full((16, 16), 1.5, np.float32)
    s = di.base_compressed_bytes(f, 1e-3)
    assert s["n_verbatim"] == 0 and s["bits_per_value"] < 0.05
    f, fh, xi, _ = di.config_inputs("C1")
    s = di.base_compressed_bytes(f, xi)
    _, codes = di.lorenzo_codes(f, xi)
    _, cnt = np.unique(codes, return_counts=True)
    p = cnt / cnt.sum()
    assert abs(s["bits_per_value"] - float(-(p * np.log2(p)).sum())) < 1e-9
    assert 4 * f.size / s["bytes"] > 4          # CR of the stand-in on a smooth field


def test_edit_stream_pack_roundtrip_and_ocr():
    """The stored edit artifact: the codec stream through the lossless stage and
    back; OCR = original bytes / (base bytes + packed edit bytes) is below CR."""
    import torch
    import paper_2409_17346_b200 as dmtz
    f, fh, xi, _ = di.config_inputs("C1")
    r = oracle.correct(f, fh, xi)
    stream = np.frombuffer(ec.encode(r["edits"], xi, 6), np.uint8)
    blob = dmtz.pack_edit_stream(torch.from_numpy(stream.copy()))
    back = dmtz.unpack_edit_stream(blob).numpy()
    assert back.tobytes() == stream.tobytes()
    base = di.base_compressed_bytes(f, xi)["bytes"]
    cr, ocr = 4 * f.size / base, 4 * f.size / (base + len(blob))
    assert ocr < cr and len(blob) <= len(stream) + 16
