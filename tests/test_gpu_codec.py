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
