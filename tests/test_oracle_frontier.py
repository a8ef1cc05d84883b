"""The oracle's frontier mode (``oracle.correct(frontier=True)``) equals its literal
full-recomputation loop bit for bit: g, per-vertex state, the edit list, the stats,
the status and the number of false cells in every round.  The frontier mode is what
makes the full-size C3/C4 goldens feasible ("frontier mode for
C4/C5, validated equal to full mode on C1-C3"); its reading -- only cells anchored
within [-2,1]^D of a target of the previous round can change or be false -- is
stated in ``oracle/dmtz_oracle.c`` (gradient_update, dmtz_oracle_correct_ex)."""
import numpy as np
import pytest

import dmtz_inputs as di
import oracle


def _same(a, b):
    assert a["status"] == b["status"]
    assert a["stats"] == b["stats"]
    assert np.array_equal(a["g"].view(np.uint32), b["g"].view(np.uint32))
    assert np.array_equal(a["state"], b["state"])
    assert a["n_edits"] == b["n_edits"]
    assert a["edits"].tobytes() == b["edits"].tobytes()
    assert a["false_per_round"] == b["false_per_round"]


def _both(f, fhat, xi, **kw):
    full = oracle.correct(f, fhat, xi, round_log=True, **kw)
    fr = oracle.correct(f, fhat, xi, round_log=True, frontier=True, **kw)
    _same(full, fr)
    return full


CASES = [((40, 40), 1, False, "lorenzo"), ((31, 45), 2, True, "lorenzo"), ((50, 37), 3, False, "noise"),
         ((12, 13, 11), 4, False, "lorenzo"), ((9, 14, 10), 5, True, "lorenzo"),
         ((10, 10, 10), 6, False, "noise"), ((3, 17, 16), 7, True, "noise")]


@pytest.mark.parametrize("shape,seed,ties,perturb", CASES)
@pytest.mark.parametrize("q_cap", [6, 65535])
def test_frontier_equals_full_random(shape, seed, ties, perturb, q_cap):
    f, fhat, xi = di.random_case(shape, seed, eps=2e-2, ties=ties, perturb=perturb)
    r = _both(f, fhat, xi, q_cap=q_cap)
    assert r["status"] == oracle.OK
    assert ties or r["stats"]["rounds"] > 1


@pytest.mark.parametrize("tier", [1, 2])
def test_frontier_equals_full_tiers(tier):
    f, fhat, xi = di.random_case((11, 12, 13), 21, eps=3e-2, perturb="noise")
    _both(f, fhat, xi, tier=tier)


@pytest.mark.parametrize("name,shape", [("C1", None), ("C2", (120, 240)), ("C3", (16, 40, 40)),
                                        ("C4", (24, 24, 24)), ("C5", (20, 20, 20))])
def test_frontier_equals_full_config_crops(name, shape):
    f, fhat, xi, _ = di.config_inputs(name, shape=shape)
    r = _both(f, fhat, xi)
    assert r["status"] == oracle.OK


def test_frontier_equals_full_iter_cap_and_stuck():
    f, fhat, xi = di.random_case((12, 12, 12), 8, eps=2e-2)
    _both(f, fhat, xi, max_rounds=3)
    # near-zero field with a coarse bound: RU(f - xi) merges values -> STUCK (reading A10)
    rng = np.random.default_rng(3)
    f = (rng.standard_normal((9, 10, 11)) * 1e-6).astype(np.float32)
    fhat = (f + rng.uniform(-0.5, 0.5, f.shape).astype(np.float32) * np.float32(0.9)).astype(np.float32)
    r = _both(f, fhat, 1.0)
    assert r["status"] in (oracle.OK, oracle.E_STUCK)
