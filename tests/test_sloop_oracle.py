"""Pins of the oracle's S-loop / alternating C-S driver (P:150,
P:226-259).  CPU only.

The independent brute force (tests/bruteforce.py: explicit Kuhn complex, set
operations, its own traces) reruns the whole workflow and must agree bit for bit;
the tier post-conditions are checked on the result with the brute
force's traces: tier 4 -- every separatrix of g is cell for cell the one of f;
tier 3 -- every separatrix ends where it ends in f."""
import numpy as np
import pytest

import dmtz_inputs as di
import oracle
from tests import bruteforce as bf


def _complex(shape):
    if len(shape) == 2:
        return bf.Complex(shape[1], shape[0], 1)
    return bf.Complex(shape[2], shape[1], shape[0])


CASES = [  # (family, shape, seed, eps, perturb, tier, q_cap)
    ("lognormal", (10, 10), 4, 0.05, "lorenzo", 3, 6),
    ("lognormal", (10, 10), 4, 0.05, "lorenzo", 4, 6),
    ("lognormal", (10, 10), 2, 0.2, "lorenzo", 4, 65535),
    ("gauss2d", (10, 10), 1, 0.05, "noise", 4, 6),
    ("multiscale", (12, 12), 4, 0.05, "lorenzo", 3, 65535),
    ("multiscale", (5, 6, 6), 3, 0.05, "lorenzo", 3, 6),
    ("multiscale", (5, 6, 6), 3, 0.05, "lorenzo", 4, 65535),
    ("lognormal", (5, 6, 6), 3, 0.2, "lorenzo", 4, 6),
    ("multiscale", (5, 6, 6), 5, 0.2, "lorenzo", 3, 6),
    ("noise", (5, 6, 6), 2, 0.2, "lorenzo", 4, 6),
]


@pytest.mark.parametrize("family,shape,seed,eps,perturb,tier,q_cap", CASES)
def test_preserve_matches_bruteforce(family, shape, seed, eps, perturb, tier, q_cap):
    f, fh, xi = di.random_case(shape, seed, eps=eps, family=family, perturb=perturb)
    r = oracle.preserve(f, fh, xi, tier=tier, q_cap=q_cap)
    st, g, q, ll, stats = bf.cs_loop(_complex(shape), f, fh, xi, 6, q_cap, tier)
    assert {"OK": 0, "STUCK": 7, "ITER_CAP": 6}[st] == r["status"]
    assert np.array_equal(r["g"].ravel().view(np.uint32), g.view(np.uint32))
    assert np.array_equal(r["state"].ravel() & 0xFFFF, q)
    assert np.array_equal((r["state"].ravel() >> 16).astype(bool), ll)
    for k in ("c_rounds", "s_rounds", "troublemakers"):
        assert r["stats"][k] == stats[k], k
    assert r["stats"]["s_rounds"] > 0


def _ends(sep):
    return [(k, o, sorted(map(sorted, t)) if k == "conn" else t) for k, o, _, t in sep]


@pytest.mark.parametrize("family,shape,seed,eps,perturb,tier,q_cap", CASES[::2])
def test_tier_postconditions(family, shape, seed, eps, perturb, tier, q_cap):
    """P:142 (T3: each saddle reaches the same extrema) and P:143 (T4: the separatrices
    follow the same paths), plus T2 and the error bound, on the brute force's
    own traces."""
    f, fh, xi = di.random_case(shape, seed, eps=eps, family=family, perturb=perturb)
    r = oracle.preserve(f, fh, xi, tier=tier, q_cap=q_cap)
    assert r["status"] == 0
    g = r["g"]
    assert np.all(g.astype(np.float64) <= fh) and np.all(np.abs(g.astype(np.float64) - f) <= xi)
    assert np.array_equal(oracle.gradient(f)[1], oracle.gradient(g)[1])
    C = _complex(shape)
    sf, sg = bf.trace(C, f), bf.trace(C, g)
    if tier == 4:
        assert sf == sg
    assert _ends(sf) == _ends(sg)


def test_tier4_is_stricter_than_tier3():
    """a state whose paths differ while every end agrees -> no fix under
    tier 3, at least one under tier 4.  (The C-loop alone leaves such a state here.)"""
    f, fh, xi = di.random_case((6, 7), 1, eps=5e-2)
    r3 = oracle.preserve(f, fh, xi, tier=3)
    r4 = oracle.preserve(f, fh, xi, tier=4)
    c = oracle.correct(f, fh, xi)
    assert r3["stats"]["s_rounds"] == 0 and np.array_equal(r3["g"], c["g"])
    assert r4["stats"]["s_rounds"] >= 1 and r4["n_edits"] > c["n_edits"]
    C = _complex(f.shape)
    sf, sc = bf.trace(C, f), bf.trace(C, c["g"])
    assert _ends(sf) == _ends(sc) and sf != sc


@pytest.mark.parametrize("tier", [1, 2])
def test_low_tiers_are_the_cloop(tier):
    f, fh, xi = di.random_case((7, 6, 5), 3, eps=0.05, family="lognormal")
    r = oracle.preserve(f, fh, xi, tier=tier)
    c = oracle.correct(f, fh, xi, tier=tier)
    assert r["status"] == c["status"] == 0
    assert np.array_equal(r["g"].view(np.uint32), c["g"].view(np.uint32))
    assert r["stats"]["rounds"] == c["stats"]["rounds"] and r["stats"]["s_rounds"] == 0


@pytest.mark.parametrize("tier", [3, 4])
def test_identity_needs_no_edit(tier):
    """fhat = f -> one pass, zero fixes."""
    f, _, xi = di.random_case((6, 5, 4), 2, eps=0.05)
    r = oracle.preserve(f, f.copy(), xi, tier=tier)
    assert r["status"] == 0 and r["n_edits"] == 0
    assert r["stats"]["c_rounds"] == r["stats"]["s_rounds"] == 0


def test_preserve_errors():
    f, fh, xi = di.random_case((5, 5), 1)
    assert oracle.preserve(f, fh, xi, tier=6)["status"] == oracle.E_ARG
    bad = fh.copy()
    bad[0, 0] = f[0, 0] + np.float32(3 * xi)
    assert oracle.preserve(f, bad, xi, tier=4)["status"] == oracle.E_BOUND


# ----------------------------------------------------------------------------- tier 5
def test_persistence0_double_well_golden():
    """a double well on a 5x2 strip -- minima at x=0 (f=0) and x=2 (f=1) merge at
    x=1 (f=4): exactly one finite pair, (vertex 2, vertex 1)."""
    f = np.array([[0, 4, 1, 5, 6], [0.5, 4.5, 1.5, 5.5, 6.5]], np.float32)
    assert oracle.persistence0(f).tolist() == [[2, 1]]
    assert bf.persistence0(_complex(f.shape), f) == [(2, 1)]


@pytest.mark.parametrize("shape,seed,ties", [((6, 7), 1, False), ((8, 8), 2, True), ((4, 4, 4), 3, False),
                                             ((3, 5, 4), 4, True)])
def test_persistence0_matches_bruteforce(shape, seed, ties):
    f, _, _ = di.random_case(shape, seed, ties=ties)
    po = sorted(map(tuple, oracle.persistence0(f).tolist()))
    assert po == bf.persistence0(_complex(shape), f)
    # one essential class: finite pairs = minima - 1 (every minimum but the global one dies)
    assert len(po) == int(np.count_nonzero(oracle.gradient(f)[1].ravel() & 1)) - 1


@pytest.mark.parametrize("family,shape,seed,eps,perturb", [("lognormal", (10, 10), 4, 0.05, "lorenzo"),
                                                           ("multiscale", (5, 6, 6), 3, 0.05, "lorenzo"),
                                                           ("gauss2d", (12, 12), 1, 0.05, "noise")])
def test_tier5_matches_bruteforce_and_keeps_the_diagram(family, shape, seed, eps, perturb):
    """P:272 / P:327: T5 pre-clamps every vertex of every critical cell of f to its lower
    bound, then runs the tier-4 workflow.  Post-conditions: the T4 ones, and the 0-dim
    persistence pairs of g are those of f with both ends at f - xi (reading A18)."""
    f, fh, xi = di.random_case(shape, seed, eps=eps, family=family, perturb=perturb)
    r = oracle.preserve(f, fh, xi, tier=5)
    st, g, q, ll, stats = bf.cs_loop(_complex(shape), f, fh, xi, 6, 6, 5)
    assert st == "OK" and r["status"] == 0
    assert np.array_equal(r["g"].ravel().view(np.uint32), g.view(np.uint32))
    assert np.array_equal((r["state"].ravel() >> 16).astype(bool), ll)
    C = _complex(shape)
    assert bf.trace(C, f) == bf.trace(C, r["g"])
    pf, pg = oracle.persistence0(f), oracle.persistence0(r["g"])
    assert sorted(map(tuple, pf.tolist())) == sorted(map(tuple, pg.tolist()))
    lb = np.array([bf.ru32(bf.Fraction(float(v)) - bf.Fraction(float(np.float32(xi)))) for v in f.ravel()],
                  np.float32)
    ends = np.unique(pf.ravel())
    assert np.array_equal(r["g"].ravel()[ends].view(np.uint32), lb[ends].view(np.uint32))
