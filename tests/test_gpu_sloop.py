"""GPU parity of the S-loop / alternating C-S workflow (``-m gpu``):
dmtz_preserve through the C-ABI against oracle.preserve on the same seeded inputs --
bit-exact edited field, edit list and round / troublemaker statistics -- and the tier
post-conditions checked with the GPU's own traces at sizes the oracle cannot reach."""
import numpy as np
import pytest
import torch

import dmtz_inputs as di
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dmtz():
    import paper_2409_17346_b200 as d
    return d


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _compare(dmtz, f, fh, xi, tier, q_cap=6, full_sweeps=False, ctx=None):
    ref = oracle.preserve(f, fh, xi, tier=tier, q_cap=q_cap)
    r = (ctx or dmtz).preserve(_cuda(f), _cuda(fh), xi, tier=tier, q_cap=q_cap, full_sweeps=full_sweeps)
    assert r.status == ref["status"], r.message
    assert np.array_equal(r.g.cpu().numpy().view(np.uint32), ref["g"].view(np.uint32))
    e = r.edits_numpy()
    for k in ("v", "q", "lossless"):
        assert np.array_equal(e[k], ref["edits"][k]), k
    assert np.array_equal(e["value"].view(np.uint32), ref["edits"]["value"].view(np.uint32))
    for k in ("c_rounds", "s_rounds", "troublemakers", "tm_round1", "sep_branches", "sep_cells"):
        assert r.stats[k] == ref["stats"][k], (k, r.stats[k], ref["stats"][k])
    assert r.stats["tm_by_kind"] == ref["stats"]["tm_by_kind"]
    assert r.stats["n_false_round0"] == ref["stats"]["n_false_round0"]
    assert r.stats["rounds"] == ref["stats"]["rounds"]
    return r, ref


CASES = [  # (family, shape, seed, eps, perturb, tier, q_cap)
    ("lognormal", (10, 10), 4, 0.05, "lorenzo", 3, 6),
    ("lognormal", (10, 10), 4, 0.05, "lorenzo", 4, 6),
    ("gauss2d", (12, 12), 1, 0.05, "noise", 4, 65535),
    ("multiscale", (5, 6, 6), 3, 0.05, "lorenzo", 3, 6),
    ("multiscale", (5, 6, 6), 3, 0.05, "noise", 4, 65535),
    ("multiscale", (6, 6, 6), 4, 0.2, "noise", 4, 6),
    ("lognormal", (6, 6, 6), 4, 0.2, "noise", 3, 6),
    ("noise", (33, 40, 37), 2, 0.05, "lorenzo", 4, 6),
    ("lognormal", (20, 31, 45), 3, 0.05, "lorenzo", 3, 6),
    ("noise", (97, 131), 5, 0.1, "noise", 4, 6),
    ("lognormal", (10, 10), 4, 0.05, "lorenzo", 5, 6),
    ("multiscale", (5, 6, 6), 3, 0.05, "lorenzo", 5, 65535),
    ("lognormal", (20, 31, 45), 3, 0.05, "lorenzo", 5, 6),
]


@pytest.mark.parametrize("family,shape,seed,eps,perturb,tier,q_cap", CASES)
def test_preserve_bit_exact(dmtz, family, shape, seed, eps, perturb, tier, q_cap):
    f, fh, xi = di.random_case(shape, seed, eps=eps, family=family, perturb=perturb)
    r, ref = _compare(dmtz, f, fh, xi, tier, q_cap)
    assert ref["stats"]["s_rounds"] > 0


@pytest.mark.parametrize("ordered,smem", [("0", "2"), ("0", "0"), ("1", "2"), ("1", "0")])
def test_tier3_connectors_at_every_level(dmtz, monkeypatch, ordered, smem):
    """Tier 3's candidate traces with the connector BFS forced through every escalation
    level (test knobs as in test_gpu_escalation.py), in the unordered fill (default) and
    the FIFO one, with the shared-memory and the global visited hash: bit-exact vs the
    oracle."""
    monkeypatch.setenv("DMTZ_TEST_CQ", "2")
    monkeypatch.setenv("DMTZ_TEST_WQ", "8")
    monkeypatch.setenv("DMTZ_TEST_BFS_GROW", "2")
    monkeypatch.setenv("DMTZ_BFS_SMEM", smem)
    monkeypatch.setenv("DMTZ_T3_ORDERED", ordered)   # read when the context is created
    f, fh, xi = di.random_case((20, 31, 45), 3, eps=0.05, family="lognormal", perturb="lorenzo")
    ctx = dmtz.Context(f.shape, torch.device("cuda", 0))
    r, ref = _compare(dmtz, f, fh, xi, 3, ctx=ctx)
    assert ref["stats"]["s_rounds"] > 0
    lv = dmtz.last_trace_levels()
    assert lv[2] > 0, lv   # the last candidate trace reached the block levels


@pytest.mark.parametrize("tier", [3, 4])
def test_preserve_full_sweeps(dmtz, tier):
    f, fh, xi = di.random_case((12, 14, 13), 7, eps=0.05, family="multiscale", perturb="noise")
    _compare(dmtz, f, fh, xi, tier, full_sweeps=True)


@pytest.mark.parametrize("name,shape,tier", [("C1", None, 4), ("C2", (120, 240), 4), ("C3", (20, 50, 50), 4),
                                             ("C4", (24, 24, 24), 4), ("C4", (20, 22, 24), 3),
                                             ("C5", (20, 24, 28), 4), ("C4", (24, 24, 24), 5)])
def test_preserve_config_crops(dmtz, name, shape, tier):
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    _compare(dmtz, f, fh, xi, tier)


@pytest.mark.parametrize("tier", [1, 2])
def test_preserve_low_tiers_equal_correct(dmtz, tier):
    f, fh, xi, _ = di.config_inputs("C4", shape=(24, 24, 24))
    a = dmtz.preserve(_cuda(f), _cuda(fh), xi, tier=tier)
    b = dmtz.correct(_cuda(f), _cuda(fh), xi, tier=tier)
    assert a.status == b.status == 0
    assert torch.equal(a.g, b.g) and a.stats["s_rounds"] == 0


def _ends(tr, nb):
    """per branch: terminal (DESC/ASC) or the sorted reached 1-saddles (CONN)."""
    off, cells, term, kind = (tr[k].cpu().numpy() for k in ("offsets", "cells", "terminal", "kind"))
    out = []
    for b in range(nb):
        if kind[b] == 4:
            seg = cells[off[b]:off[b + 1]].view(np.uint64)
            out.append(tuple(sorted(seg[(seg >> 56) == 1].tolist())))
        else:
            out.append(int(term[b]))
    return out


@pytest.mark.parametrize("name,shape,tier", [("C3", (50, 120, 120), 4), ("C4", (64, 64, 64), 4),
                                             ("C4", (48, 48, 48), 3)])
def test_preserve_postconditions_mid_size(dmtz, name, shape, tier):
    """P:141-143 on sizes beyond the oracle: critical cells equal (T2); tier 4: the
    separatrices of g equal those of f cell for cell; tier 3: every branch ends the same;
    |g - f| <= xi."""
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    ft, fht = _cuda(f), _cuda(fh)
    r = dmtz.preserve(ft, fht, xi, tier=tier)
    assert r.status == 0, r.message
    assert r.stats["s_rounds"] > 0
    g = r.g
    assert bool((g <= fht).all())
    assert bool(((g.double() - ft.double()).abs() <= xi).all())
    cf, cg = dmtz.compute_gradient(ft), dmtz.compute_gradient(g)
    assert torch.equal(dmtz.critical_mask(cf), dmtz.critical_mask(cg))
    tf, tg = dmtz.trace_separatrices(cf), dmtz.trace_separatrices(cg)
    if tier == 4:
        for k in tf:
            assert torch.equal(tf[k], tg[k]), k
    else:
        nb = tf["origin"].shape[0]
        assert tg["origin"].shape[0] == nb and torch.equal(tf["origin"], tg["origin"])
        assert _ends(tf, nb) == _ends(tg, nb)


@pytest.mark.parametrize("name,shape", [("C4", (48, 48, 48)), ("C2", (300, 600))])
def test_tier5_keeps_the_persistence_diagram(dmtz, name, shape):
    """P:143 / P:272: after tier 5 the 0-dim persistence pairs of g (oracle union-find)
    are those of f, and their vertices sit at their lower bounds (reading A18)."""
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    r = dmtz.preserve(_cuda(f), _cuda(fh), xi, tier=5)
    assert r.status == 0, r.message
    g = r.g.cpu().numpy()
    pf, pg = oracle.persistence0(f), oracle.persistence0(g)
    assert sorted(map(tuple, pf.tolist())) == sorted(map(tuple, pg.tolist()))
    e = r.edits_numpy()
    ends = np.unique(pf.ravel())
    clamped = e["v"][e["lossless"] > 0]
    assert np.isin(ends, clamped).all()


def test_preserve_capacity_and_errors(dmtz):
    f, fh, xi, _ = di.config_inputs("C4", shape=(24, 24, 24))
    ft, fht = _cuda(f), _cuda(fh)
    r = dmtz.preserve(ft, fht, xi, tier=4, sep_caps=(10, 10), raise_on_error=False)
    assert r.status == dmtz.E_CAPACITY
    ref = oracle.preserve(f, fh, xi, tier=4)["stats"]
    assert r.stats["sep_branches"] == ref["sep_branches"]
    with pytest.raises(dmtz.DmtzError):
        dmtz.preserve(ft, fht, xi, tier=6)
    bad = fh.copy()
    bad[3, 4, 5] = f[3, 4, 5] + np.float32(4 * xi)
    r = dmtz.preserve(ft, _cuda(bad), xi, tier=4, raise_on_error=False)
    assert r.status == dmtz.E_BOUND


@pytest.mark.parametrize("tier", [4, 5])
def test_full_size_C2_postconditions(dmtz, tier):
    """C2 at full size (1800x3600): the tier post-conditions with the GPU's own traces
     and, for tier 5, the 0-dim persistence pairs by the oracle's union-find."""
    f, fh, xi, _ = di.config_inputs("C2")
    ft, fht = _cuda(f), _cuda(fh)
    r = dmtz.preserve(ft, fht, xi, tier=tier)
    assert r.status == 0, r.message
    assert bool((r.g <= fht).all()) and bool(((r.g.double() - ft.double()).abs() <= xi).all())
    cf, cg = dmtz.compute_gradient(ft), dmtz.compute_gradient(r.g)
    assert torch.equal(dmtz.critical_mask(cf), dmtz.critical_mask(cg))
    tf, tg = dmtz.trace_separatrices(cf), dmtz.trace_separatrices(cg)
    for k in tf:
        assert torch.equal(tf[k], tg[k]), k
    if tier == 5:
        pf, pg = oracle.persistence0(f), oracle.persistence0(r.g.cpu().numpy())
        assert sorted(map(tuple, pf.tolist())) == sorted(map(tuple, pg.tolist()))
