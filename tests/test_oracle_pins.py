"""More pins for the CPU oracle (``-m "not gpu"``), against things other than itself.

* The progress lemma (reading R3b): on fields normalised
  to [1, 2) -- where RU(f - xi) is strictly order-preserving (reading A10) -- every
  target a round selects still has g > lb, so every round moves, no run ends STUCK,
  and the loop terminates with F empty.  The test also shows that the paper-silent
  rule R3b is exercised (and R1 / R2 / R3a), counted by the oracle's diagnostics.
* The saddle-saddle connector's event log in its full interleaved order (critical
  edges and newly enqueued triangles as the breadth-first search meets them, S:212,
  P:228) against the explicit-complex brute force.
"""
import numpy as np
import pytest

import dmtz_inputs as di
import oracle
from tests import bruteforce as bf
from tests.test_oracle import _id_to_cell, _shape3


def _lemma_cases():
    shapes2 = [(9, 11), (14, 13), (17, 10), (12, 12)]
    shapes3 = [(5, 6, 7), (7, 7, 7), (6, 8, 5), (8, 6, 6)]
    cases = []
    for i in range(40):
        shape = (shapes2 + shapes3)[i % 8]
        fam = ("noise", "lognormal", "multiscale", "noise")[i % 4] if len(shape) == 3 else \
            ("noise", "gauss2d", "climate", "noise")[i % 4]
        cases.append((shape, 1000 + i, fam, i % 3 == 0, "lorenzo" if i % 2 else "noise"))
    return cases


@pytest.mark.parametrize("q_cap", [6, 65535])
def test_progress_lemma_and_rule_coverage(q_cap):
    """80 random 2D / 3D fields in [1, 2) (ties, four families, two perturbations) x
    q_cap in {6, 65535} = 160 runs: no target is ever at its lower bound, no run is
    STUCK, and every rule -- R3b included -- resolves false cells."""
    tot = dict(r1=0, r2=0, r3a=0, r3b=0, targets=0)
    n_runs = 0
    for shape, seed, fam, ties, pert in _lemma_cases() * 2:
        eps = 4e-2 if n_runs % 2 else 1.5e-2
        f, fh, xi = di.random_case(shape, seed + n_runs, eps=eps, ties=ties, perturb=pert, family=fam)
        assert f.min() >= 1.0 and f.max() < 2.0
        r = oracle.correct(f, fh, xi, q_cap=q_cap, diag=True)
        n_runs += 1
        assert r["status"] == oracle.OK, (shape, seed, r["status"])
        assert r["diag"]["targets_at_lb"] == 0, (shape, seed, r["diag"])
        for k in tot:
            tot[k] += r["diag"][k]
    assert n_runs == 80
    assert all(tot[k] > 0 for k in ("r1", "r2", "r3a", "r3b")), tot


def test_targets_at_lb_detected_on_merging_field():
    """The diagnostics are not vacuous: on a near-zero field where RU(f - xi) merges
    values (reading A10) targets at the lower bound do occur (and the run is STUCK)."""
    rng = np.random.default_rng(3)
    seen = 0
    for _ in range(6):
        f = (rng.random((6, 6)) * 1e-7).astype(np.float32)
        fh = (f + (rng.random((6, 6)) - 0.5) * 0.5).astype(np.float32)
        r = oracle.correct(f, fh, 0.5, diag=True)
        seen += r["diag"]["targets_at_lb"]
    assert seen > 0


@pytest.mark.parametrize("shape,seed,fam", [((4, 4, 4), 3, "noise"), ((5, 5, 5), 5, "noise"),
                                            ((3, 5, 4), 4, "noise"), ((6, 6, 6), 8, "lognormal"),
                                            ((5, 7, 6), 9, "hurricane")])
def test_connector_events_interleaved_vs_bruteforce(shape, seed, fam):
    f, fh, _ = di.random_case(shape, seed, family=fam)
    info = oracle.complex_info(shape)
    s3 = _shape3(shape)
    C = bf.Complex(s3[2], s3[1], s3[0])
    n_conn = 0
    for fld in (f, fh):
        tr = oracle.trace(fld, kinds=oracle.KIND_CONN)
        ref = bf.trace(C, fld, interleaved=True)
        ref = [r for r in ref if r[0] == "conn"]
        assert len(ref) == len(tr["origin"])
        for b, (_, origin, events, reached) in enumerate(ref):
            assert _id_to_cell(tr["origin"][b], shape, info) == origin
            got = [_id_to_cell(c, shape, info) for c in tr["cells"][tr["offsets"][b]:tr["offsets"][b + 1]]]
            assert got == events
            n_conn += len(events) > 2 and any(len(e) == 2 for e in events) and any(len(e) == 3 for e in events)
    if fam == "noise":
        assert n_conn > 0   # some logs really interleave edges and triangles
