"""GPU parity (``-m gpu``): the CUDA path, called through the C-ABI, against the CPU
oracle on the same seeded inputs -- bit-exact on gradient codes, critical masks,
edited-field bits, edit lists and statistics."""
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


def _codes_np(t):
    a = t.cpu().numpy()
    return a.view(np.uint64) if a.dtype == np.int64 else a.view(np.uint16)


GRAD_CASES = [((3, 3), 0, False), ((17, 23), 1, False), ((64, 64), 2, True), ((130, 257), 3, False),
              ((2, 2, 2), 4, False), ((3, 4, 5), 5, True), ((9, 8, 7), 6, False), ((33, 35, 131), 7, False),
              ((20, 40, 30), 8, True)]


@pytest.mark.parametrize("shape,seed,ties", GRAD_CASES)
def test_gradient_codes_and_crit_bit_exact(dmtz, shape, seed, ties):
    f, fh, _ = di.random_case(shape, seed, ties=ties)
    for fld in (f, fh):
        oc, om = oracle.gradient(fld)
        gc = dmtz.compute_gradient(_cuda(fld))
        gm = dmtz.critical_mask(gc)
        torch.cuda.synchronize()
        assert np.array_equal(_codes_np(gc), oc)
        assert np.array_equal(gm.cpu().numpy().view(np.uint32), om)


@pytest.mark.parametrize("name,shape", [("C1", None), ("C2", (180, 360)), ("C3", (20, 50, 50)),
                                        ("C4", (24, 24, 24)), ("C5", (20, 24, 28))])
def test_gradient_config_crops(dmtz, name, shape):
    f, fh, _, _ = di.config_inputs(name, shape=shape)
    for fld in (f, fh):
        oc, om = oracle.gradient(fld)
        gc = dmtz.compute_gradient(_cuda(fld))
        assert np.array_equal(_codes_np(gc), oc)
        assert np.array_equal(dmtz.critical_mask(gc).cpu().numpy().view(np.uint32), om)


def _compare_correct(dmtz, f, fh, xi, q_cap=6, tier=2, full_sweeps=False):
    ref = oracle.correct(f, fh, xi, 6, q_cap, tier)
    r = dmtz.correct(_cuda(f), _cuda(fh), xi, q_max=6, q_cap=q_cap, tier=tier, full_sweeps=full_sweeps)
    assert r.status == ref["status"], r.message
    assert np.array_equal(r.g.cpu().numpy().view(np.uint32), ref["g"].view(np.uint32))
    e = r.edits_numpy()
    assert r.n_edits == ref["n_edits"]
    assert np.array_equal(e["v"], ref["edits"]["v"])
    assert np.array_equal(e["q"], ref["edits"]["q"])
    assert np.array_equal(e["lossless"], ref["edits"]["lossless"])
    assert np.array_equal(e["value"].view(np.uint32), ref["edits"]["value"].view(np.uint32))
    for k in ("rounds", "n_edited", "n_quantized", "n_lossless", "n_false_round0", "false_by_kind_round0"):
        assert r.stats[k] == ref["stats"][k], k
    return r, ref


CLOOP_CASES = [  # (family, shape, seed, eps, perturb, q_cap, tier, ties)
    ("noise", (4, 4), 10, 5e-2, "lorenzo", 6, 2, False),
    ("lognormal", (5, 6), 3, 5e-2, "noise", 1, 2, False),
    ("lognormal", (5, 6), 3, 5e-2, "noise", 65535, 2, False),
    ("gauss2d", (40, 70), 3, 0.05, "noise", 6, 2, False),
    ("gauss2d", (40, 70), 3, 0.05, "noise", 6, 1, False),
    ("lognormal", (57, 61), 3, 0.02, "lorenzo", 6, 2, True),
    ("lognormal", (4, 4, 4), 3, 5e-2, "noise", 6, 2, False),
    ("lognormal", (13, 17, 19), 3, 0.01, "noise", 6, 2, False),
    ("lognormal", (13, 17, 19), 3, 0.01, "noise", 65535, 2, False),
    ("lognormal", (13, 17, 19), 3, 0.01, "noise", 6, 1, False),
    ("multiscale", (16, 16, 40), 3, 0.05, "noise", 6, 2, True),
    ("hurricane", (10, 33, 70), 4, 0.01, "lorenzo", 6, 2, False),
]


@pytest.mark.parametrize("family,shape,seed,eps,perturb,q_cap,tier,ties", CLOOP_CASES)
def test_cloop_bit_exact(dmtz, family, shape, seed, eps, perturb, q_cap, tier, ties):
    f, fh, xi = di.random_case(shape, seed, eps=eps, ties=ties, perturb=perturb, family=family)
    _compare_correct(dmtz, f, fh, xi, q_cap, tier)


@pytest.mark.parametrize("name,shape", [("C1", None), ("C2", (180, 360)), ("C3", (20, 50, 50)),
                                        ("C4", (32, 32, 32)), ("C5", (24, 24, 24))])
@pytest.mark.parametrize("full_sweeps", [False, True])
def test_cloop_config_crops(dmtz, name, shape, full_sweeps):
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    r, ref = _compare_correct(dmtz, f, fh, xi, full_sweeps=full_sweeps)
    assert ref["status"] == 0 and ref["stats"]["rounds"] > 0


def test_b1_golden_on_gpu(dmtz):
    f = np.array([[1, 2], [4, 3]], np.float32)
    fh = np.array([[2, 1], [4, 3]], np.float32)
    r, _ = _compare_correct(dmtz, f, fh, 1.0, q_cap=6)
    assert r.g.cpu().numpy().ravel().tolist() == [0.0, 1.0, 4.0, 3.0] and r.stats["rounds"] == 7
    r, _ = _compare_correct(dmtz, f, fh, 1.0, q_cap=65535)
    assert r.stats["rounds"] == 64


def test_errors_and_capacity(dmtz):
    f, fh, xi = di.random_case((20, 30), 3, eps=0.05, family="gauss2d", perturb="noise")
    bad = fh.copy()
    bad[3, 4] = np.nan
    r = dmtz.correct(_cuda(f), _cuda(bad), xi, raise_on_error=False)
    assert r.status == dmtz.E_NONFINITE and "vertex" in r.message
    bad = fh.copy()
    bad[5, 5] = f[5, 5] + 2 * xi
    r = dmtz.correct(_cuda(f), _cuda(bad), xi, raise_on_error=False)
    assert r.status == dmtz.E_BOUND
    ref = oracle.correct(f, fh, xi)
    assert ref["n_edits"] > 2
    r = dmtz.correct(_cuda(f), _cuda(fh), xi, edits_capacity=2)
    assert r.status == dmtz.E_CAPACITY and r.n_edits == ref["n_edits"]
    assert np.array_equal(r.edits_numpy()["v"], ref["edits"]["v"][:2])
    with pytest.raises(TypeError):
        dmtz.correct(torch.from_numpy(f), torch.from_numpy(fh), xi)


def test_stuck_matches_oracle(dmtz):
    rng = np.random.default_rng(3)
    seen = set()
    for i in range(6):
        f = (rng.random((6, 6)) * 1e-7).astype(np.float32)
        fh = (f + (rng.random((6, 6)) - 0.5) * 0.5).astype(np.float32)
        r, ref = _compare_correct(dmtz, f, fh, 0.5)
        seen.add(r.status)
    assert dmtz.E_STUCK in seen


def test_deterministic(dmtz):
    f, fh, xi, _ = di.config_inputs("C4", shape=(40, 40, 40))
    a = dmtz.correct(_cuda(f), _cuda(fh), xi)
    b = dmtz.correct(_cuda(f), _cuda(fh), xi)
    assert torch.equal(a.g.view(torch.int32), b.g.view(torch.int32)) and torch.equal(a.edits, b.edits)


TRACE_CASES = [("noise", (6, 7), 1), ("noise", (40, 33), 2), ("gauss2d", (64, 64), 3), ("noise", (4, 4, 4), 3),
               ("noise", (5, 6, 7), 4), ("lognormal", (12, 13, 14), 5), ("hurricane", (10, 30, 40), 6)]


def _compare_trace(dmtz, fld):
    ref = oracle.trace(fld)
    codes = dmtz.compute_gradient(_cuda(fld))
    tr = dmtz.trace_separatrices(codes)
    for k in ("offsets", "cells", "origin", "terminal"):
        got = tr[k].cpu().numpy()
        want = ref[k]
        if want.dtype == np.uint64:
            got = got.view(np.uint64)
        assert np.array_equal(got, want), k
    assert np.array_equal(tr["kind"].cpu().numpy(), ref["kind"])
    return ref


@pytest.mark.parametrize("family,shape,seed", TRACE_CASES)
def test_trace_bit_exact(dmtz, family, shape, seed):
    f, fh, xi = di.random_case(shape, seed, family=family)
    ref = _compare_trace(dmtz, f)
    assert len(ref["origin"]) > 0
    _compare_trace(dmtz, fh)


@pytest.mark.parametrize("name,shape", [("C1", None), ("C3", (20, 50, 50)), ("C4", (24, 24, 24))])
def test_trace_after_correct(dmtz, name, shape):
    """The separatrices of the converged field g (the S-loop's input)."""
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    r = dmtz.correct(_cuda(f), _cuda(fh), xi)
    _compare_trace(dmtz, r.g.cpu().numpy())


def test_trace_capacity(dmtz):
    f, _, _ = di.random_case((5, 6, 7), 4)
    ref = oracle.trace(f)
    codes = dmtz.compute_gradient(_cuda(f))
    with pytest.raises(dmtz.DmtzError) as ei:
        dmtz.trace_separatrices(codes, cap_branches=3, cap_cells=10)
    assert ei.value.status == dmtz.E_CAPACITY
    tr = dmtz.trace_separatrices(codes, kinds=dmtz.KIND_DESC)
    nd = int((ref["kind"] == 1).sum())
    assert tr["origin"].shape[0] == nd
    assert np.array_equal(tr["cells"].cpu().numpy().view(np.uint64), ref["cells"][:ref["offsets"][nd]])


# ----------------------------------------------------------------------------- full BASELINE sizes
def _crop_check(full_codes, full_crit, fld, rng, shape, edge, n=4):
    """Oracle gradient of random crops vs the GPU result on the full field, on the crop
    anchors whose codes (margin 1) and criticality (margin 1 below, 2 above) cannot see
    the crop boundary."""
    D = len(shape)
    for _ in range(n):
        lo = [int(rng.integers(0, s - edge + 1)) for s in shape]
        sl = tuple(slice(l, l + edge) for l in lo)
        oc, om = oracle.gradient(np.ascontiguousarray(fld[sl]))
        inner_c = tuple(slice(1, edge - 1) for _ in range(D))
        inner_m = tuple(slice(1, edge - 2) for _ in range(D))
        gc, gm = full_codes[sl], full_crit[sl]
        assert np.array_equal(gc[inner_c], oc[inner_c])
        assert np.array_equal(gm[inner_m], om[inner_m])


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_full_size_gradient_sampled(dmtz, name):
    f, fh, xi, cfg = di.config_inputs(name)
    rng = np.random.default_rng(7)
    edge = 96 if len(cfg.shape) == 2 else 20
    for fld in (f, fh):
        gc = dmtz.compute_gradient(_cuda(fld))
        gm = dmtz.critical_mask(gc).cpu().numpy().view(np.uint32)
        _crop_check(_codes_np(gc), gm, fld, rng, cfg.shape, edge)


def test_full_size_cloop_C2_bit_exact(dmtz):
    """BASELINE config C2 (2D 1800x3600) end to end against the full oracle run."""
    f, fh, xi, _ = di.config_inputs("C2")
    r, ref = _compare_correct(dmtz, f, fh, xi)
    assert ref["stats"]["rounds"] > 10


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_cloop_properties(dmtz, name):
    """Full-size C-loop (the launch configuration bench.py times): exact error bound,
    monotone edits, edit list replays g, and no false critical cell at exit -- checked
    by the oracle on sampled crops of f and g."""
    f, fh, xi, cfg = di.config_inputs(name)
    r = dmtz.correct(_cuda(f), _cuda(fh), xi)                    # default mode (what bench.py times)
    rf = dmtz.correct(_cuda(f), _cuda(fh), xi, full_sweeps=True)  # reference mode: every code, every round
    assert r.status == dmtz.OK and r.stats["rounds"] > 0
    assert r.stats["rounds"] == rf.stats["rounds"] and r.n_edits == rf.n_edits
    assert torch.equal(r.g.view(torch.int32), rf.g.view(torch.int32))
    assert torch.equal(r.edits, rf.edits)
    g = r.g.cpu().numpy()
    F, FH, G = f.astype(np.float64), fh.astype(np.float64), g.astype(np.float64)
    assert np.all(G <= FH) and np.all(np.abs(G - F) <= np.float64(np.float32(xi)))
    e = r.edits_numpy()
    assert np.all(np.diff(e["v"].astype(np.int64)) > 0)
    rec = fh.ravel().copy()
    step = np.float32(xi) * np.float32(2.0 ** -6)
    ql = e["lossless"] == 0
    rec[e["v"][ql]] = (fh.ravel()[e["v"][ql]] - (e["q"][ql].astype(np.float32) * step).astype(np.float32))
    rec[e["v"][~ql]] = e["value"][~ql]
    assert np.array_equal(rec.view(np.uint32), g.ravel().view(np.uint32))
    changed = np.nonzero(g.ravel() != fh.ravel())[0]
    assert np.isin(changed, e["v"]).all()
    # crit(g) == crit(f) everywhere on the GPU, and on oracle-sampled crops
    cf = dmtz.critical_mask(dmtz.compute_gradient(_cuda(f)))
    cg = dmtz.critical_mask(dmtz.compute_gradient(r.g))
    assert torch.equal(cf, cg)
    rng = np.random.default_rng(11)
    for _ in range(4):
        lo = [int(rng.integers(0, s - 20 + 1)) for s in cfg.shape]
        sl = tuple(slice(l, l + 20) for l in lo)
        _, mf = oracle.gradient(np.ascontiguousarray(f[sl]))
        _, mg = oracle.gradient(np.ascontiguousarray(g[sl]))
        inner = tuple(slice(1, 18) for _ in cfg.shape)
        assert np.array_equal(mf[inner], mg[inner])


@pytest.mark.parametrize("full_sweeps", [False, True])
def test_iter_cap_matches_oracle(dmtz, full_sweeps):
    """The device-side stop rule (CUDA-graph WHILE loop) on the round cap."""
    f, fh, xi, _ = di.config_inputs("C4", shape=(20, 21, 22))
    ref = oracle.correct(f, fh, xi, 6, 6, 2, max_rounds=3)
    assert ref["status"] == oracle.E_ITER_CAP
    r = dmtz.correct(_cuda(f), _cuda(fh), xi, max_rounds=3, full_sweeps=full_sweeps)
    assert r.status == dmtz.E_ITER_CAP and r.stats["rounds"] == 3 == ref["stats"]["rounds"]
    assert np.array_equal(r.g.cpu().numpy().view(np.uint32), ref["g"].view(np.uint32))
    assert np.array_equal(r.edits_numpy()["v"], ref["edits"]["v"])


def test_full_size_cloop_C5_one_gpu(dmtz):
    """BASELINE config C5 (3D 1024^3, nominally 8 GPUs) fits one B200: the default-mode
    C-loop to its fixed point, every property checked on the device -- exact error bound,
    edits only lower g, the edit list replays g bit for bit, and crit(g) == crit(f)
    everywhere."""
    f, fh, xi, cfg = di.config_inputs("C5")
    ft, fht = _cuda(f), _cuda(fh)
    del f, fh
    r = dmtz.correct(ft, fht, xi)
    assert r.status == dmtz.OK and r.stats["rounds"] > 0
    g = r.g
    x32 = torch.tensor(np.float32(xi), device=g.device)
    assert bool((g <= fht).all()) and bool(((g.double() - ft.double()).abs() <= x32.double()).all())
    e = r.edits.view(-1, 16)
    v = e[:, 0:8].contiguous().view(torch.int64).view(-1)
    q = e[:, 8:10].contiguous().view(torch.int16).view(-1).to(torch.int64) & 0xFFFF
    ll = e[:, 10] != 0
    val = e[:, 12:16].contiguous().view(torch.float32).view(-1)
    assert bool((v[1:] > v[:-1]).all())
    rec = fht.reshape(-1).clone()
    step = torch.tensor(np.float32(xi) * np.float32(2.0 ** -6), device=g.device)
    rec[v[~ll]] = fht.reshape(-1)[v[~ll]] - (q[~ll].to(torch.float32) * step)
    rec[v[ll]] = val[ll]
    assert torch.equal(rec.view(torch.int32), g.reshape(-1).view(torch.int32))
    codes_f, codes_g = dmtz.compute_gradient(ft), dmtz.compute_gradient(g)
    cf, cg = dmtz.critical_mask(codes_f), dmtz.critical_mask(codes_g)
    assert torch.equal(cf, cg)
    # sampled outputs the oracle computes one by one: on random 20^3 crops, the GPU's
    # full-grid codes (anchors whose stencil lies in the crop) and critical masks (anchors
    # whose 8 codes do) equal the oracle's literal gradient of the crop, for f and g
    rng = np.random.default_rng(5)
    for _ in range(6):
        lo = [int(rng.integers(0, s - 20 + 1)) for s in cfg.shape]
        sl = tuple(slice(l, l + 20) for l in lo)
        for fld, codes, crit in ((ft, codes_f, cf), (g, codes_g, cg)):
            oc, om = oracle.gradient(np.ascontiguousarray(fld[sl].cpu().numpy()))
            ic, im = tuple(slice(1, 19) for _ in range(3)), tuple(slice(1, 18) for _ in range(3))
            shp = tuple(cfg.shape)
            assert np.array_equal(_codes_np(codes.reshape(shp)[sl].contiguous())[ic], oc.reshape(20, 20, 20)[ic])
            assert np.array_equal(crit.reshape(shp)[sl].cpu().numpy().view(np.uint32)[im],
                                  om.reshape(20, 20, 20)[im])


@pytest.mark.parametrize("cap", ["0", "2048", "5000"])
def test_trace_connector_pool_fallback(dmtz, monkeypatch, cap):
    """The connector events kept by the count pass (a pool in the output buffer) and the
    BFS redone in the write pass give the same CSR: a pool too small for every connector
    (DMTZ_CONN_POOL_CAP entries) mixes both paths; DMTZ_CONN_POOL=0 disables the pool."""
    f, _, _ = di.random_case((20, 22, 24), 11, family="lognormal")
    monkeypatch.setenv("DMTZ_CONN_POOL_CAP", cap)
    _compare_trace(dmtz, f)
    monkeypatch.setenv("DMTZ_CONN_POOL", "0")
    _compare_trace(dmtz, f)


@pytest.mark.parametrize("name,shape", [("C2", (90, 180)), ("C4", (40, 40, 40))])
def test_correct_host_equals_device(dmtz, name, shape):
    """dmtz_correct_host (host buffers in and out, the copies inside the C call) returns
    the device call's g and edit list bit for bit; NULL host outputs are skipped."""
    import torch
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    ctx = dmtz.context(f.shape, torch.device("cuda", 0))
    r = ctx.correct(torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda(), xi)
    rh = ctx.correct_host(torch.from_numpy(f).pin_memory(), torch.from_numpy(fh).pin_memory(), xi)
    assert rh.status == r.status and rh.n_edits == r.n_edits > 0
    assert rh.g.device.type == "cpu" and rh.edits.device.type == "cpu"
    assert torch.equal(rh.g.view(torch.int32), r.g.cpu().view(torch.int32))
    assert torch.equal(rh.edits, r.edits.cpu())
    assert rh.stats["rounds"] == r.stats["rounds"]
    g2, e2, st2 = dmtz.correct_host(f, fh, xi)   # pageable numpy in, numpy out
    assert np.array_equal(g2.view(np.int32), r.g.cpu().numpy().view(np.int32))
    assert np.array_equal(e2, r.edits_numpy())


@pytest.mark.parametrize("family,shape", [("lognormal", (20, 22, 24)), ("multiscale", (16, 40, 36)),
                                          ("climate", (60, 90))])
def test_trace_static_walk_kernel(dmtz, monkeypatch, family, shape):
    """DMTZ_WALK_STATIC=1 (k_walk: one thread per branch) gives the oracle's CSR as the
    default k_walk_dyn (lanes refilled as their paths end) does."""
    f, _, _ = di.random_case(shape, 5, family=family)
    monkeypatch.setenv("DMTZ_WALK_STATIC", "1")
    _compare_trace(dmtz, f)
