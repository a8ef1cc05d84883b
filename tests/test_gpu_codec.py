"""GPU edit codec and decompression-side apply (``-m gpu``): the CUDA
encoder's bytes equal the plain-Python oracle encoder's, decode inverts it, and
dmtz_apply_edits rebuilds dmtz_correct's g bit for bit."""
import numpy as np
import pytest
import torch

import dmtz_inputs as di
import oracle
from oracle import edit_codec as ec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dmtz():
    import paper_2409_17346_b200 as d
    return d


def _same_edits(d, e):
    """decoded vs original: v, q, lossless; value bits of the lossless entries (quantized
    entries carry no value in the stream -- apply_edits recomputes it from fhat)."""
    a, b = d.cpu().numpy().view(oracle.EDIT_DTYPE).ravel(), e.cpu().numpy().view(oracle.EDIT_DTYPE).ravel()
    ll = b["lossless"] > 0
    return (len(a) == len(b) and all(np.array_equal(a[k], b[k]) for k in ("v", "q", "lossless")) and
            np.array_equal(a["value"][ll].view(np.uint32), b["value"][ll].view(np.uint32)))


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("name,shape,q_cap", [("C1", None, 6), ("C2", (180, 360), 65535), ("C3", (20, 50, 50), 6),
                                              ("C4", (48, 48, 48), 6)])
def test_encode_decode_apply(dmtz, name, shape, q_cap):
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    ft, fht = _cuda(f), _cuda(fh)
    ctx = dmtz.context(ft.shape, ft.device)
    r = ctx.correct(ft, fht, xi, q_cap=q_cap)
    assert r.status == 0
    s = ctx.encode_edits(r.edits, xi, 6)
    ref = ec.encode(r.edits_numpy(), xi, 6)
    assert s.cpu().numpy().tobytes() == ref
    d, x2, qm = ctx.decode_edits(s)
    assert (x2, qm) == (np.float32(xi), 6)
    assert _same_edits(d, r.edits)
    g = ctx.apply_edits(fht, x2, d, q_max=qm)
    assert torch.equal(g.view(torch.int32), r.g.view(torch.int32))
    assert s.numel() < 12 * max(r.n_edits, 1) + 64   # below the 12 B key-value float records
    # version 2: lossless values relative to fhat
    s2 = ctx.encode_edits(r.edits, xi, 6, fhat=fht)
    assert s2.cpu().numpy().tobytes() == ec.encode(r.edits_numpy(), xi, 6, fhat=fh)
    assert s2.numel() <= s.numel()
    d2, _, _ = ctx.decode_edits(s2, fhat=fht)
    assert _same_edits(d2, r.edits)
    assert torch.equal(ctx.apply_edits(fht, xi, d2).view(torch.int32), r.g.view(torch.int32))


def test_multi_block_and_errors(dmtz):
    f, fh, xi, _ = di.config_inputs("C4", shape=(64, 64, 64))
    ft, fht = _cuda(f), _cuda(fh)
    ctx = dmtz.context(ft.shape, ft.device)
    r = ctx.correct(ft, fht, xi)
    assert r.n_edits > 3 * 4096
    s = ctx.encode_edits(r.edits, xi, 6)
    assert s.cpu().numpy().tobytes() == ec.encode(r.edits_numpy(), xi, 6)
    d, _, _ = ctx.decode_edits(s)
    assert _same_edits(d, r.edits)
    bad = s.clone()
    bad[0] = ord("X")
    with pytest.raises(dmtz.DmtzError):
        ctx.decode_edits(bad)
    with pytest.raises(dmtz.DmtzError):
        ctx.decode_edits(s[:-3].clone())
    rev = torch.flip(r.edits[:10], dims=[0]).contiguous()
    with pytest.raises(dmtz.DmtzError):
        ctx.encode_edits(rev, xi, 6)
    far = r.edits[:1].clone()
    far[0, :8] = torch.tensor(list((f.size + 5).to_bytes(8, "little")), dtype=torch.uint8)
    with pytest.raises(dmtz.DmtzError):
        ctx.apply_edits(fht, xi, far)
    with pytest.raises(dmtz.DmtzError):   # a version-2 stream without fhat
        ctx.decode_edits(ctx.encode_edits(r.edits, xi, 6, fhat=fht))
    e0 = ctx.encode_edits(r.edits[:0], xi, 6)
    assert e0.numel() == 32 and ctx.decode_edits(e0)[0].shape[0] == 0


def _decode_env(ctx, s, fht, thread):
    """decode with the warp-per-block version-2 decoder (default) or the thread-per-block one."""
    import os
    if thread:
        os.environ["DMTZ_EC_DECODE_THREAD"] = "1"
    try:
        return ctx.decode_edits(s, fhat=fht)
    finally:
        os.environ.pop("DMTZ_EC_DECODE_THREAD", None)


def test_v2_warp_decoder_multi_block_and_fuzz(dmtz):
    """the warp decoder (records split across lanes, roles chained in lane order) returns
    the same records as the thread decoder on a multi-block version-2 stream, and takes
    the same accept / reject decision on corrupted copies (flipped continuation bits,
    changed bytes, truncations)."""
    f, fh, xi, _ = di.config_inputs("C4", shape=(64, 64, 64))
    ft, fht = _cuda(f), _cuda(fh)
    ctx = dmtz.context(ft.shape, ft.device)
    r = ctx.correct(ft, fht, xi)
    assert r.n_edits > 3 * 4096
    s = ctx.encode_edits(r.edits, xi, 6, fhat=fht)
    d, _, _ = _decode_env(ctx, s, fht, thread=False)
    assert _same_edits(d, r.edits)
    assert torch.equal(d, _decode_env(ctx, s, fht, thread=True)[0])
    rng = np.random.default_rng(7)
    nblk = (r.n_edits + 4095) // 4096
    pay0 = 32 + 8 * nblk
    verdicts = set()
    for trial in range(40):
        bad = s.clone()
        k = int(rng.integers(pay0, s.numel()))
        if trial % 4 == 0:
            bad[k] ^= 0x80                      # continuation bit: merges / splits varints
        elif trial % 4 == 1:
            bad[k] = int(rng.integers(0, 256))
        elif trial % 4 == 2:
            bad[k] ^= 0x01                      # a lossless flag or a low value bit
        else:
            bad = bad[:k].clone()               # truncated
        res = []
        for thread in (False, True):
            try:
                res.append(_decode_env(ctx, bad, fht, thread)[0].clone())
            except dmtz.DmtzError:
                res.append(None)
        assert (res[0] is None) == (res[1] is None), trial
        if res[0] is not None:
            a = res[0].cpu().numpy().view(oracle.EDIT_DTYPE).ravel()
            b = res[1].cpu().numpy().view(oracle.EDIT_DTYPE).ravel()
            assert all(np.array_equal(a[key], b[key]) for key in ("v", "q", "lossless")), trial
            ll = b["lossless"] > 0
            assert np.array_equal(a["value"][ll].view(np.uint32), b["value"][ll].view(np.uint32)), trial
        verdicts.add(res[0] is None)
    assert True in verdicts


@pytest.mark.parametrize("name,shape,full", [("C4", (40, 44, 48), False), ("C3", (20, 50, 50), True),
                                             ("C2", (180, 360), False)])
def test_correct_host_stream_is_the_oracle_stream(dmtz, name, shape, full):
    """dmtz_correct_host_stream (host f / fhat in, the encoded edit stream out): its bytes
    equal the oracle codec's version-2 stream of the oracle-equal edit list, and they
    decode and apply back to correct()'s g."""
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    ft, fht = _cuda(f), _cuda(fh)
    ctx = dmtz.Context(ft.shape, ft.device)
    r = ctx.correct(ft, fht, xi, full_sweeps=full)
    rh, sb = ctx.correct_host_stream(torch.from_numpy(f).pin_memory(), torch.from_numpy(fh).pin_memory(), xi,
                                     full_sweeps=full)
    assert rh.status == r.status == 0 and rh.n_edits == r.n_edits
    assert sb.numpy().tobytes() == ec.encode(r.edits_numpy(), xi, 6, fhat=fh)
    d, x2, qm = ctx.decode_edits(sb.cuda(), fhat=fht)
    g = ctx.apply_edits(fht, x2, d, q_max=qm)
    assert torch.equal(g.view(torch.int32), r.g.view(torch.int32))
