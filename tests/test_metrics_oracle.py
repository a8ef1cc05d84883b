"""Pins of the §5.1 metrics (oracle/metrics.py)
worked examples and a brute-force critical set."""
import numpy as np

import dmtz_inputs as di
import oracle
from oracle import metrics
from tests import bruteforce as bf


def test_critical_prf_examples():
    f, fh, _ = di.random_case((9, 9), 3)
    _, c = oracle.gradient(f)
    assert metrics.critical_prf(c, c)[ "recall"] == 1.0
    assert metrics.critical_prf(c, c)["precision"] == 1.0
    z = np.zeros_like(c)
    r = metrics.critical_prf(c, z)
    assert r["recall"] == 0.0 and r["precision"] == 1.0
    # |orig| = 9 minima, rec = orig + one spurious minimum -> recall 1, precision 9/10
    a = np.zeros(100, np.uint32)
    a[np.arange(9) * 11] = 1
    b = a.copy()
    b[99] = 1
    r = metrics.critical_prf(a, b)
    assert (r["recall"], r["precision"]) == (1.0, 0.9)


def test_critical_prf_against_bruteforce():
    """counts on a decompressed field agree with set arithmetic on the brute force's cells"""
    f, fh, _ = di.random_case((6, 7), 2, eps=0.1)
    C = bf.Complex(7, 6, 1)
    cf, cg = bf.critical(C, bf.gradient(C, f)), bf.critical(C, bf.gradient(C, fh))
    r = metrics.critical_prf(oracle.gradient(f)[1], oracle.gradient(fh)[1])
    assert (r["n_orig"], r["n_rec"], r["n_match"]) == (len(cf), len(cg), len(cf & cg))


def test_separatrix_prf_examples():
    f, _, _ = di.random_case((5, 5, 5), 1)
    tr = oracle.trace(f)
    r = metrics.separatrix_prf(tr, tr)
    assert r["recall"] == r["precision"] == 1.0 and r["n_orig"] == len(tr["origin"])
    # one diverged branch of 10 -> (0.9, 0.9)
    ten = {k: v[:10] for k, v in tr.items() if k != "offsets"}
    ten["offsets"] = tr["offsets"][:11]
    ten["cells"] = tr["cells"][:tr["offsets"][10]]
    bad = {k: v.copy() for k, v in ten.items()}
    bad["cells"][bad["offsets"][3]] ^= np.uint64(1)
    r = metrics.separatrix_prf(ten, bad)
    assert (r["recall"], r["precision"]) == (0.9, 0.9)
    # empty original: recall 1 by convention, precision 1 iff the reconstruction is empty too
    empty = {k: v[:0] for k, v in ten.items()}
    empty["offsets"] = ten["offsets"][:1]
    assert metrics.separatrix_prf(empty, empty)["precision"] == 1.0
    assert metrics.separatrix_prf(empty, ten)["recall"] == 1.0
    assert metrics.separatrix_prf(empty, ten)["precision"] == 0.0


def test_metrics_after_preserve_are_perfect():
    f, fh, xi = di.random_case((10, 10), 4, eps=0.05, family="lognormal")
    before = metrics.separatrix_prf(oracle.trace(f), oracle.trace(fh))
    r = oracle.preserve(f, fh, xi, tier=4)
    after = metrics.separatrix_prf(oracle.trace(f), oracle.trace(r["g"]))
    assert before["recall"] < 1.0 and after["recall"] == after["precision"] == 1.0
    c = metrics.critical_prf(oracle.gradient(f)[1], oracle.gradient(r["g"])[1])
    assert c["recall"] == c["precision"] == 1.0
