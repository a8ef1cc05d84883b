"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against things
other than itself -- the paper's worked example (Fig. 3), closed-form cell counts,
the Euler/Morse relation, an independent explicit-complex brute force
(tests/bruteforce.py), exact rational arithmetic for the edit step, and the
convergence invariants of P:115 / P:249-259."""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import dmtz_inputs as di
import oracle
from tests import bruteforce as bf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _shape3(shape):
    return (1,) + tuple(shape) if len(shape) == 2 else tuple(shape)


# --------------------------------------------------------------------------- complex
@pytest.mark.parametrize("shape,counts", [((2, 2), [4, 5, 2, 0]), ((2, 2, 2), [8, 19, 18, 6]),
                                          ((3, 3), [9, 16, 8, 0])])
def test_cell_counts_closed_form(shape, counts):
    # (2,2,1) -> 4/5/2, (2,2,2) -> 8/19/18/6 (6-tet Kuhn cube); 3x3: 9 vertices,
    # 12 axis + 4 diagonal edges, 8 triangles.
    assert oracle.cell_counts(shape).tolist() == counts


@pytest.mark.parametrize("shape", [(2, 3), (5, 4), (7, 9), (2, 2, 3), (3, 4, 5), (4, 3, 2)])
def test_euler_characteristic_of_complex(shape):
    c = oracle.cell_counts(shape)
    assert c[0] - c[1] + c[2] - c[3] == 1          # simply connected grid domain
    C = bf.Complex(*reversed(_shape3(shape))) if len(shape) == 3 else bf.Complex(shape[1], shape[0])
    assert [len(C.by_dim.get(d, [])) for d in range(4)] == c.tolist()


@pytest.mark.parametrize("D", [2, 3])
def test_links_match_explicit_complex(D):
    """The oracle's per-type interior links (slot order) equal the links read off a
    padded explicit Kuhn complex built from axis permutations."""
    shape = (3, 3) if D == 2 else (3, 3, 3)
    info = oracle.complex_info(shape)
    C = bf.Complex(3, 3, 3 if D == 3 else 1, pad=2)
    centre = (1, 1, 1 if D == 3 else 0)
    for t in range(info["T"]):
        d = info["dim"][t]
        cell = frozenset(tuple(centre[a] + info["offsets"][t][k][a] for a in range(3)) for k in range(d + 1))
        assert cell in C.cells, (t, cell)
        link = sorted((next(iter(b - cell)) for b in C.cofacets[cell]),
                      key=lambda p: (p[2], p[1], p[0]))
        got = [tuple(centre[a] + info["links"][t][s][a] for a in range(3)) for s in range(info["nlink"][t])]
        assert got == link, t
    # type counts per anchor: 1/7/12/6 (3D), 1/3/2 (2D)
    per_dim = np.bincount(info["dim"], minlength=4)[:D + 1].tolist()
    assert per_dim == ([1, 3, 2] if D == 2 else [1, 7, 12, 6])


# --------------------------------------------------------------------------- gradient
def _decode_pairs(shape, codes, crit):
    """Oracle packed codes -> set of (cell, cofacet) pairs + critical set, using the
    oracle's own complex description (itself pinned by test_links_match_explicit_complex)."""
    info = oracle.complex_info(shape)
    s3 = _shape3(shape)
    D = 2 if len(shape) == 2 else 3
    codes = codes.ravel().astype(np.uint64)
    crit = crit.ravel()
    pairs, crits = set(), set()
    nz, ny, nx = s3
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                A = x + nx * (y + ny * z)
                c = int(codes[A])
                for t in range(info["T"]):
                    d = int(info["dim"][t])
                    verts = [(x + info["offsets"][t][k][0], y + info["offsets"][t][k][1],
                              z + info["offsets"][t][k][2]) for k in range(d + 1)]
                    cell = frozenset(verts)
                    if (crit[A] >> t) & 1:
                        crits.add(cell)
                    if d == D:
                        continue
                    k = t - int(np.searchsorted(info["dim"], d))
                    if D == 3:
                        s = (c & 15) if d == 0 else ((c >> (4 + 3 * k)) & 7) if d == 1 else ((c >> (25 + 2 * k)) & 3)
                        none = {0: 15, 1: 7, 2: 3}[d]
                    else:
                        s = (c & 7) if d == 0 else ((c >> (3 + 2 * k)) & 3)
                        none = {0: 7, 1: 3}[d]
                    if s != none:
                        w = tuple(p + info["links"][t][s][a] for a, p in enumerate((x, y, z)))
                        pairs.add((cell, cell | {w}))
    return pairs, crits


def _bf_pairs(shape, field):
    s3 = _shape3(shape)
    C = bf.Complex(s3[2], s3[1], s3[0] if len(shape) == 3 else 1)
    pair = bf.gradient(C, field)
    up = {(a, b) for a, b in pair.items() if len(b) > len(a)}
    return up, bf.critical(C, pair)


CASES = [((3, 3), 0, False), ((4, 5), 1, False), ((6, 6), 2, True), ((5, 4), 3, True),
         ((2, 2, 2), 4, False), ((3, 3, 3), 5, False), ((3, 4, 5), 6, False), ((3, 3, 4), 7, True),
         ((4, 4, 4), 8, True)]


@pytest.mark.parametrize("shape,seed,ties", CASES)
def test_gradient_matches_bruteforce(shape, seed, ties):
    f, _, _ = di.random_case(shape, seed, ties=ties)
    codes, crit = oracle.gradient(f)
    pairs, crits = _decode_pairs(shape, codes, crit)
    bpairs, bcrit = _bf_pairs(shape, f)
    assert pairs == bpairs
    assert crits == bcrit


def test_gradient_exhaustive_orders_2x2x2_sample():
    """Many value orders of the 2x2x2 cube (all 8! orders would take minutes in pure
    Python; a fixed-seed sample of 300 permutations, incl. ties)."""
    rng = np.random.default_rng(11)
    for it in range(300):
        vals = rng.permutation(8).astype(np.float32)
        if it % 3 == 0:
            vals = np.floor(vals / 3).astype(np.float32)
        f = vals.reshape(2, 2, 2)
        codes, crit = oracle.gradient(f)
        assert _decode_pairs((2, 2, 2), codes, crit) == _bf_pairs((2, 2, 2), f)


def test_gradient_all_orders_3x3_sample():
    rng = np.random.default_rng(12)
    for it in range(300):
        f = rng.permutation(9).astype(np.float32).reshape(3, 3)
        codes, crit = oracle.gradient(f)
        assert _decode_pairs((3, 3), codes, crit) == _bf_pairs((3, 3), f)


def test_fig3_triangle_bruteforce_golden():
    """The brute force itself reproduces the paper's worked example."""
    g = json.load(open(os.path.join(GOLDEN, "fig3_triangle.json")))
    # explicit one-triangle complex: i=(0,0,0), j=(1,0,0), k=(2,0,0) on a 3x1 "grid"
    # index order i<j<k (ties never occur here)
    pos = {"i": (0, 0, 0), "j": (1, 0, 0), "k": (2, 0, 0)}

    class Tri:
        D = 2
        n = (3, 1, 1)

        def __init__(self):
            verts = list(pos.values())
            self.cells = {frozenset(s) for r in (1, 2, 3) for s in itertools.combinations(verts, r)}
            self.by_dim = {d: sorted((c for c in self.cells if len(c) == d + 1), key=sorted) for d in range(3)}
            self.cofacets = {c: [b for b in self.cells if len(b) == len(c) + 1 and c < b] for c in self.cells}

        def vid(self, p):
            return p[0]

    T = Tri()
    name = {frozenset(pos[ch] for ch in s): s for s in ["i", "j", "k", "ij", "ik", "jk", "ijk"]}
    for field, crit_key in (("f", "critical_f"), ("fhat", "critical_fhat")):
        vals = np.array([g[field][c] for c in "ijk"], np.float32)
        pair = bf.gradient(T, vals)
        crit = sorted(name[c] for c in bf.critical(T, pair))
        assert crit == g[crit_key]
        if field == "f":
            got = sorted((name[a], name[b]) for a, b in pair.items() if len(b) > len(a))
            assert got == sorted(tuple(p) for p in g["pairs_f"])


@pytest.mark.parametrize("shape", [(5, 7), (4, 4, 4), (3, 5, 6)])
def test_constant_field_single_minimum(shape):
    # constant field -> SoS order = index order -> exactly one critical cell, vertex 0
    f = np.full(shape, 1.5, np.float32)
    _, crit = oracle.gradient(f)
    crit = crit.ravel()
    assert crit[0] == 1 and crit.sum() == 1 and np.count_nonzero(crit) == 1


@pytest.mark.parametrize("shape,seed", [((17, 23), 1), ((9, 8, 7), 2), ((6, 11, 5), 3)])
def test_morse_relation_and_order_invariance(shape, seed):
    f, _, _ = di.random_case(shape, seed)
    info = oracle.complex_info(shape)
    c1, m1 = oracle.gradient(f)
    counts = np.zeros(4, np.int64)
    for t in range(info["T"]):
        counts[info["dim"][t]] += int(((m1 >> t) & 1).sum())
    assert counts[0] - counts[1] + counts[2] - counts[3] == 1
    # order-only dependence: 2f is exact in binary floating point
    c2, m2 = oracle.gradient((2 * f).astype(np.float32))
    assert np.array_equal(c1, c2) and np.array_equal(m1, m2)


@pytest.mark.parametrize("shape", [(6, 7), (4, 5, 3)])
def test_reversed_index_order_single_minimum(shape):
    """f = -(vertex index): the SoS order is the reverse index order, a linear order on a
    collapsible complex -> exactly one critical cell, the minimum at the last vertex."""
    n = int(np.prod(shape))
    f = (-np.arange(n, dtype=np.float32)).reshape(shape)
    _, crit = oracle.gradient(f)
    crit = crit.ravel()
    assert np.count_nonzero(crit) == 1 and crit[n - 1] == 1


def test_table2_counts_satisfy_euler():
    # Heated Flow critical counts 98/703/606 and 158/1095/938 (2D): chi = 1, the
    # relation test_morse_relation_and_order_invariance enforces on the oracle.
    assert 98 - 703 + 606 == 1 and 158 - 1095 + 938 == 1


# --------------------------------------------------------------------------- C-loop
def test_b1_golden():
    g = json.load(open(os.path.join(GOLDEN, "b1_fig3_2x2.json")))
    f = np.array(g["f"], np.float32).reshape(g["shape"])
    fh = np.array(g["fhat"], np.float32).reshape(g["shape"])
    for case in g["cases"]:
        r = oracle.correct(f, fh, g["xi"], g["q_max"], case["q_cap"])
        assert r["status"] == case["status"]
        assert r["stats"]["rounds"] == case["rounds"]
        assert r["g"].ravel().tolist() == case["g"]
        assert [[int(e["v"]), int(e["q"]), int(e["lossless"]), float(e["value"])] for e in r["edits"]] == case["edits"]
        assert r["stats"]["false_by_kind_round0"] == case["false_round0"]


CLOOP_CASES = [  # (family, shape, seed, eps, perturb, q_cap, tier, ties)
    ("noise", (4, 4), 10, 5e-2, "lorenzo", 6, 2, False),
    ("noise", (5, 6), 11, 5e-2, "lorenzo", 6, 2, True),
    ("lognormal", (5, 6), 3, 5e-2, "noise", 1, 2, False),
    ("lognormal", (5, 6), 3, 5e-2, "noise", 6, 2, False),
    ("lognormal", (5, 6), 3, 5e-2, "noise", 65535, 2, False),
    ("gauss2d", (8, 8), 3, 0.2, "lorenzo", 1, 2, False),
    ("gauss2d", (8, 8), 3, 0.2, "noise", 6, 1, False),
    ("lognormal", (7, 7), 3, 0.2, "lorenzo", 6, 2, True),
    ("lognormal", (4, 4, 4), 3, 5e-2, "lorenzo", 6, 2, False),
    ("lognormal", (4, 4, 4), 3, 5e-2, "noise", 6, 2, False),
    ("lognormal", (3, 4, 5), 3, 0.2, "noise", 1, 2, False),
    ("lognormal", (3, 4, 5), 3, 0.2, "noise", 6, 1, False),
    ("multiscale", (4, 4, 4), 3, 0.2, "noise", 6, 2, False),
    ("multiscale", (4, 4, 4), 3, 0.05, "noise", 65535, 2, True),
]


@pytest.mark.parametrize("family,shape,seed,eps,perturb,q_cap,tier,ties", CLOOP_CASES)
def test_cloop_matches_bruteforce(family, shape, seed, eps, perturb, q_cap, tier, ties):
    f, fh, xi = di.random_case(shape, seed, eps=eps, ties=ties, perturb=perturb, family=family)
    r = oracle.correct(f, fh, xi, 6, q_cap, tier)
    s3 = _shape3(shape)
    C = bf.Complex(s3[2], s3[1], s3[0] if len(shape) == 3 else 1)
    st, g, q, ll, stats = bf.c_loop(C, f, fh, xi, 6, q_cap, tier)
    assert {"OK": 0, "STUCK": 7, "ITER_CAP": 6}[st] == r["status"]
    assert np.array_equal(r["g"].ravel().view(np.uint32), g.view(np.uint32))
    assert np.array_equal(r["state"].ravel() & 0xFFFF, q)
    assert np.array_equal((r["state"].ravel() >> 16).astype(bool), ll)
    assert r["stats"]["rounds"] == stats["rounds"]
    assert r["stats"]["n_false_round0"] == stats["n_false_round0"]
    assert r["stats"]["false_by_kind_round0"] == stats["kinds"]


@pytest.mark.parametrize("shape,seed", [((16, 16), 1), ((7, 9, 8), 2), ((10, 6, 7), 3)])
@pytest.mark.parametrize("q_cap", [6, 65535])
def test_cloop_invariants(shape, seed, q_cap):
    """P:115 monotone bounded edits; P:138 |g - f| <= xi; at exit the critical cells of g
    equal those of f (tier 2); the edit list reproduces g."""
    f, fh, xi = di.random_case(shape, seed, eps=2e-2)
    r = oracle.correct(f, fh, xi, 6, q_cap)
    assert r["status"] == 0
    g = r["g"]
    F, FH, G = (a.astype(np.float64) for a in (f, fh, g))
    assert np.all(G <= FH) and np.all(np.abs(G - F) <= xi)
    assert np.array_equal(oracle.gradient(f)[1], oracle.gradient(g)[1])
    step = np.float32(xi) * np.float32(2.0 ** -6)
    rec = fh.ravel().copy()
    for e in r["edits"]:
        if e["lossless"]:
            rec[e["v"]] = e["value"]
        else:
            rec[e["v"]] = np.float32(fh.ravel()[e["v"]] - np.float32(np.float32(e["q"]) * step))
    assert np.array_equal(rec.view(np.uint32), g.ravel().view(np.uint32))
    assert r["n_edits"] == r["stats"]["n_edited"] == np.count_nonzero(r["state"])


def test_lossless_values_are_exact_ru_lower_bound():
    """Clamped vertices hold RU(f - xi) exactly (Fraction arithmetic), P:162 / reading A9."""
    f, fh, xi, _ = di.config_inputs("C1")
    r = oracle.correct(f, fh, xi, 6, 1)           # q_cap = 1 forces many clamps
    assert r["stats"]["n_lossless"] > 0
    fr = f.ravel()
    for e in r["edits"]:
        if e["lossless"]:
            exact = Fraction(float(fr[e["v"]])) - Fraction(float(np.float32(xi)))
            want = bf.ru32(exact)
            assert np.float32(e["value"]).view(np.uint32) == want.view(np.uint32)


def test_edit_arithmetic_spec_example():
    """xi = 0.064, q_max = 6 -> step = xi / 64; q = 5 -> fhat - RN(5 step)."""
    f = np.array([[1.0, 1.2], [1.3, 1.25]], np.float32)
    fh = np.array([[1.06, 1.15], [1.3, 1.25]], np.float32)
    r = oracle.correct(f, fh, 0.064, 6, 6)
    step = np.float32(0.064) / np.float32(64)
    assert Fraction(float(step)) == Fraction(float(np.float32(0.064))) / 64
    for e in r["edits"]:
        if not e["lossless"]:
            v = int(e["v"])
            assert r["g"].ravel()[v] == np.float32(fh.ravel()[v] - np.float32(np.float32(e["q"]) * step))


def test_errors():
    f = np.ones((4, 4), np.float32)
    fh = f.copy()
    fh[1, 1] = np.nan
    assert oracle.correct(f, fh, 0.1)["status"] == oracle.E_NONFINITE
    fh = f.copy()
    fh[2, 2] = 1.2
    assert oracle.correct(f, fh, 0.1)["status"] == oracle.E_BOUND
    fh[2, 2] = np.float32(1.1)   # 1.1f - 1.0f > 0.1f exactly? decided by exact comparison
    exact_ok = Fraction(float(np.float32(1.1))) - 1 <= Fraction(float(np.float32(0.1)))
    assert (oracle.correct(f, fh, 0.1)["status"] == 0) == exact_ok
    assert oracle.correct(f, f, -1.0)["status"] == oracle.E_ARG
    assert oracle.correct(np.ones((1, 4), np.float32), np.ones((1, 4), np.float32), 0.1)["status"] == oracle.E_DIMS


def test_stuck_on_collapsing_lower_bounds():
    """Reading A10: near-zero fields with a large xi merge RU(f - xi) values and the
    loop can end STUCK; the oracle reports it instead of looping."""
    rng = np.random.default_rng(3)
    st = []
    for i in range(6):
        f = (rng.random((6, 6)) * 1e-7).astype(np.float32)
        fh = (f + (rng.random((6, 6)) - 0.5) * 0.5).astype(np.float32)
        st.append(oracle.correct(f, fh, 0.5)["status"])
    assert set(st) <= {0, oracle.E_STUCK} and oracle.E_STUCK in st


# --------------------------------------------------------------------------- trace
def _id_to_cell(cid, shape, info):
    cid = int(cid)
    d = cid >> 56
    rest = cid & ((1 << 56) - 1)
    types = [t for t in range(info["T"]) if info["dim"][t] == d]
    A, k = divmod(rest, len(types))
    t = types[k]
    s3 = _shape3(shape)
    nx, ny = s3[2], s3[1]
    x, y, z = A % nx, (A // nx) % ny, A // (nx * ny)
    return frozenset((x + info["offsets"][t][j][0], y + info["offsets"][t][j][1],
                      z + info["offsets"][t][j][2]) for j in range(d + 1))


@pytest.mark.parametrize("shape,seed", [((6, 7), 1), ((9, 9), 2), ((4, 4, 4), 3), ((3, 5, 4), 4),
                                        ((5, 5, 5), 5)])
def test_trace_matches_bruteforce(shape, seed):
    f, _, _ = di.random_case(shape, seed)
    tr = oracle.trace(f)
    info = oracle.complex_info(shape)
    s3 = _shape3(shape)
    C = bf.Complex(s3[2], s3[1], s3[0] if len(shape) == 3 else 1)
    ref = bf.trace(C, f)
    assert len(ref) == len(tr["origin"])
    kinds = {1: "desc", 2: "asc", 4: "conn"}
    for b, (kind, origin, cells, term) in enumerate(ref):
        assert kinds[int(tr["kind"][b])] == kind
        assert _id_to_cell(tr["origin"][b], shape, info) == origin
        got = [_id_to_cell(c, shape, info) for c in tr["cells"][tr["offsets"][b]:tr["offsets"][b + 1]]]
        if kind == "conn":
            d = len(origin)
            assert [c for c in got if len(c) == d] == cells
            assert [c for c in got if len(c) == d - 1] == term
        else:
            assert got == cells
            if term == "BOUNDARY":
                assert tr["terminal"][b] == oracle.BOUNDARY
            else:
                assert _id_to_cell(tr["terminal"][b], shape, info) == term


def test_trace_terminals_are_critical_or_boundary():
    f, _, _ = di.random_case((8, 9, 10), 9)
    tr = oracle.trace(f)
    _, crit = oracle.gradient(f)
    info = oracle.complex_info(f.shape)
    crit = crit.ravel()
    for b in range(len(tr["origin"])):
        t = int(tr["terminal"][b])
        if tr["kind"][b] == 4 or t == int(oracle.BOUNDARY):
            continue
        d = t >> 56
        types = [x for x in range(info["T"]) if info["dim"][x] == d]
        A, k = divmod(t & ((1 << 56) - 1), len(types))
        assert (crit[A] >> types[k]) & 1
