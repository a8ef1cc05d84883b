"""Every escalation level of the connector BFS (saddle-saddle connectors; DESIGN.md
section 7) against the oracle, bit for bit.  Test knobs shrink the queues so that small
grids escalate: DMTZ_TEST_CQ (k_conn_small's per-thread queue), DMTZ_TEST_WQ
(k_conn_warp's per-warp queue), DMTZ_TEST_BFS_GROW (slot growth of k_walk_block's
levels), DMTZ_TEST_BFS_WORDS (its scratch); dmtz.last_trace_levels() reports how many
connectors each level handled.  Every DMTZ_BFS_THREADS block size is covered, and a
scratch too small for the largest connector ends in DMTZ_E_CAPACITY instead of a CSR
with missing connectors."""
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


def _compare_trace(dmtz, fld, kinds=oracle.KIND_DESC | oracle.KIND_ASC | oracle.KIND_CONN):
    ref = oracle.trace(fld, kinds=kinds)
    codes = dmtz.compute_gradient(torch.from_numpy(np.ascontiguousarray(fld)).cuda())
    tr = dmtz.trace_separatrices(codes, kinds=kinds)
    for k in ("offsets", "cells", "origin", "terminal"):
        got = tr[k].cpu().numpy()
        want = ref[k]
        if want.dtype == np.uint64:
            got = got.view(np.uint64)
        assert np.array_equal(got, want), k
    assert np.array_equal(tr["kind"].cpu().numpy(), ref["kind"])
    return ref


@pytest.fixture(scope="module")
def c3crop():
    f, fh, _, _ = di.config_inputs("C3", shape=(16, 60, 60))
    return f, fh


@pytest.mark.parametrize("bfs_threads,smem", [("64", "2"), ("64", "0"), ("128", "0"), ("256", "0"), ("512", "0"),
                                               ("1024", "0")])
def test_connector_escalation_every_level(dmtz, monkeypatch, c3crop, bfs_threads, smem):
    """smem = 2: levels with queues <= 8192 use the shared-memory hash (all levels here);
    0: the global-hash kernel at every block size."""
    monkeypatch.setenv("DMTZ_TEST_CQ", "2")
    monkeypatch.setenv("DMTZ_TEST_WQ", "8")
    monkeypatch.setenv("DMTZ_TEST_BFS_GROW", "2")
    monkeypatch.setenv("DMTZ_BFS_THREADS", bfs_threads)
    monkeypatch.setenv("DMTZ_BFS_SMEM", smem)
    for fld in c3crop:
        ref = _compare_trace(dmtz, fld)
        lv = dmtz.last_trace_levels()
        n_conn = int((ref["kind"] == oracle.KIND_CONN).sum())
        assert lv[0] == n_conn > 0
        # thread -> warp -> at least 3 block levels (slots 16, 32, 64, ...)
        assert lv[1] > 0 and lv[2] > 0 and lv[3] > 0 and lv[4] > 0, lv
        assert all(lv[i] >= lv[i + 1] for i in range(9)), lv


def test_connector_escalation_no_pool(dmtz, monkeypatch, c3crop):
    """The same levels with the count pass's event pool disabled (the write pass redoes
    every BFS at every level)."""
    monkeypatch.setenv("DMTZ_TEST_CQ", "3")
    monkeypatch.setenv("DMTZ_TEST_WQ", "16")
    monkeypatch.setenv("DMTZ_TEST_BFS_GROW", "4")
    monkeypatch.setenv("DMTZ_CONN_POOL", "0")
    _compare_trace(dmtz, c3crop[1])
    lv = dmtz.last_trace_levels()
    assert lv[1] > 0 and lv[2] > 0 and lv[3] > 0, lv


@pytest.mark.parametrize("smem", ["2", "0"])
def test_connector_escalation_scratch_pool(dmtz, monkeypatch, c3crop, smem):
    """Every level with the warp / block levels' event lists in the scratch pool (the
    upper part of the BFS scratch; forced on this small grid), copied by the write pass."""
    monkeypatch.setenv("DMTZ_TEST_CQ", "2")
    monkeypatch.setenv("DMTZ_TEST_WQ", "8")
    monkeypatch.setenv("DMTZ_TEST_BFS_GROW", "2")
    monkeypatch.setenv("DMTZ_BFS_SMEM", smem)
    monkeypatch.setenv("DMTZ_SCRATCH_POOL", "2")
    for fld in c3crop:
        _compare_trace(dmtz, fld)
        lv = dmtz.last_trace_levels()
        assert lv[1] > 0 and lv[2] > 0 and lv[3] > 0, lv


def test_connector_default_levels(dmtz, c3crop):
    """Without knobs the C3 crop's large connectors still reach the warp level."""
    _compare_trace(dmtz, c3crop[0])
    lv = dmtz.last_trace_levels()
    assert lv[0] > 0 and lv[1] > 0, lv


def test_connector_scratch_exhausted_is_capacity_error(dmtz, monkeypatch, c3crop):
    """A connector larger than all BFS scratch (1024 words here: slots of <= 204
    triangles; the crop has connectors of ~800) must not yield a CSR with missing
    connectors: the call fails with DMTZ_E_CAPACITY."""
    monkeypatch.setenv("DMTZ_TEST_BFS_WORDS", "1024")
    monkeypatch.setenv("DMTZ_TEST_BFS_GROW", "2")
    codes = dmtz.compute_gradient(torch.from_numpy(np.ascontiguousarray(c3crop[0])).cuda())
    with pytest.raises(dmtz.DmtzError) as ei:
        dmtz.trace_separatrices(codes)
    assert ei.value.status == dmtz.E_CAPACITY
    assert "scratch" in str(ei.value)
    # paths only (no connectors): unaffected by the scratch
    ref = oracle.trace(c3crop[0], kinds=oracle.KIND_DESC | oracle.KIND_ASC)
    tr = dmtz.trace_separatrices(codes, kinds=oracle.KIND_DESC | oracle.KIND_ASC)
    assert np.array_equal(tr["cells"].cpu().numpy().view(np.uint64), ref["cells"])
