"""GPU §5.1 metrics (``-m gpu``): match counts of dmtz_critical_prf /
dmtz_separatrix_prf equal the plain-Python oracle's on decompressed and edited fields."""
import numpy as np
import pytest
import torch

import dmtz_inputs as di
import oracle
from oracle import metrics

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dmtz():
    import paper_2409_17346_b200 as d
    return d


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _np_trace(tr):
    out = {k: v.cpu().numpy() for k, v in tr.items()}
    for k in ("cells", "origin", "terminal"):
        out[k] = out[k].view(np.uint64)
    return out


@pytest.mark.parametrize("name,shape", [("C1", None), ("C2", (120, 240)), ("C3", (20, 50, 50)), ("C4", (24, 24, 24))])
def test_metrics_match_oracle(dmtz, name, shape):
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    ft, fht = _cuda(f), _cuda(fh)
    ctx = dmtz.context(ft.shape, ft.device)
    cf, ch = ctx.compute_gradient(ft), ctx.compute_gradient(fht)
    mf, mh = ctx.critical_prf(ctx.critical_mask(cf), ctx.critical_mask(ch)), None
    ref = metrics.critical_prf(oracle.gradient(f)[1], oracle.gradient(fh)[1])
    assert {k: mf[k] for k in ("n_orig", "n_rec", "n_match")} == {k: ref[k] for k in ("n_orig", "n_rec", "n_match")}
    tf, th = ctx.trace_separatrices(cf), ctx.trace_separatrices(ch)
    sg = ctx.separatrix_prf(tf, th)
    so = metrics.separatrix_prf(_np_trace(tf), _np_trace(th))
    assert {k: sg[k] for k in ("n_orig", "n_rec", "n_match")} == {k: so[k] for k in ("n_orig", "n_rec", "n_match")}
    assert sg["recall"] < 1.0 or mf["recall"] < 1.0 or name == "C1"
    r = ctx.preserve(ft, fht, xi, tier=4)
    cg = ctx.compute_gradient(r.g)
    assert ctx.critical_prf(ctx.critical_mask(cf), ctx.critical_mask(cg))["recall"] == 1.0
    s4 = ctx.separatrix_prf(tf, ctx.trace_separatrices(cg))
    assert s4["recall"] == s4["precision"] == 1.0
