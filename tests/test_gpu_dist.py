"""The library's multi-GPU C-loop (dmtz_correct on world > 1 contexts, csrc/dmtz_dist.cuh)
equals the one-GPU dmtz_correct bit for bit: the ranks' owned g planes concatenated and
their edit lists concatenated in rank order, the status and the (global) statistics.

Two / three processes share the one GPU of this pool over a host-staged gloo transport
(every exchange and reduction completes on the host between rounds, so no kernel of one
rank ever waits on another); the NCCL transport is exercised with a one-rank
communicator (the same driver, one slab)."""
import json
import os
import socket

import numpy as np
import pytest
import torch

from tests.dist_worker import make_case, worker

pytestmark = pytest.mark.gpu
STAT_KEYS = ("rounds", "n_edited", "n_quantized", "n_lossless", "n_false_round0", "false_by_kind_round0")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _single(case):
    import paper_2409_17346_b200 as dmtz
    f, fh, xi = make_case(case)
    r = dmtz.correct(torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda(), xi, q_cap=case.get("q_cap"),
                     max_rounds=case.get("max_rounds", 0), raise_on_error=False)
    return r


def _run(case, world, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(worker, args=(world, _port(), case, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(os.path.join(tmp_path, f"rank{k}.npz")) for k in range(world)]
    g = np.concatenate([p["g"] for p in parts], axis=0)
    edits = np.concatenate([p["edits"] for p in parts], axis=0)
    stats = [json.loads(str(p["stats"])) for p in parts]
    status = [int(p["status"]) for p in parts]
    return g, edits, stats, status, parts


CASES = [
    ({"kind": "config", "name": "C4", "shape": [40, 40, 40]}, 2),
    ({"kind": "config", "name": "C4", "shape": [36, 30, 34]}, 3),
    ({"kind": "config", "name": "C4", "shape": [30, 32, 28], "full": True}, 3),
    ({"kind": "config", "name": "C3", "shape": [20, 60, 60]}, 2),
    ({"kind": "random", "shape": [12, 17, 19], "seed": 4, "eps": 4e-2, "q_cap": 65535}, 2),
    ({"kind": "random", "shape": [14, 16, 15], "seed": 6, "eps": 4e-2, "max_rounds": 4}, 2),
    ({"kind": "stuck", "shape": [9, 10, 11]}, 2),
]


@pytest.mark.parametrize("sync", [1, 3, 8])
@pytest.mark.parametrize("case,world", CASES)
def test_dist_equals_single_gpu(case, world, sync, tmp_path):
    """sync = rounds per host check (dmtz_ctx_set_dist_sync): 1 = host-synchronous rounds
    with halo-transfer skipping, > 1 = the device stop flag (batches that overrun the
    stop by up to sync - 1 rounds, which must do nothing)."""
    case = dict(case, sync=sync)
    ref = _single(case)
    g, edits, stats, status, parts = _run(case, world, tmp_path)
    assert all(s == ref.status for s in status), (status, ref.status, ref.message)
    assert np.array_equal(g.view(np.uint32), ref.g.cpu().numpy().view(np.uint32))
    assert np.array_equal(edits, ref.edits.cpu().numpy())
    for st in stats:
        for k in STAT_KEYS:
            assert st[k] == ref.stats[k], k
    # every rank reports the same global statistics
    assert all(st["n_edited"] == stats[0]["n_edited"] for st in stats)
    sent = sum(st["halo_faces_sent"] for st in stats)
    skipped = sum(st["halo_faces_skipped"] for st in stats)
    # every round after the first decides each of the 2 (world - 1) faces once
    assert sent + skipped == 2 * (world - 1) * (stats[0]["sweeps"] - 1)
    if sync > 1:
        assert skipped == 0 and all(st["sweeps"] == stats[0]["sweeps"] for st in stats)


def test_dist_halo_faces_are_skipped(tmp_path):
    """A field whose edits stay away from the slab faces in late rounds: the faces no
    edit touched are not exchanged, and the result is still the one-GPU result."""
    case = {"kind": "config", "name": "C3", "shape": [24, 64, 64], "sync": 1}
    ref = _single(case)
    g, edits, stats, status, _ = _run(case, 2, tmp_path)
    assert np.array_equal(g.view(np.uint32), ref.g.cpu().numpy().view(np.uint32))
    assert np.array_equal(edits, ref.edits.cpu().numpy())
    assert sum(st["halo_faces_skipped"] for st in stats) > 0
    assert sum(st["halo_faces_sent"] for st in stats) > 0


def test_dist_one_rank_nccl():
    """The NCCL transport (libnccl.so.2 loaded by the library, its own communicator):
    world = 1 runs the distributed driver on one slab."""
    from paper_2409_17346_b200.dist import DistContext, nccl_unique_id
    case = {"kind": "config", "name": "C4", "shape": [32, 32, 32]}
    ref = _single(case)
    f, fh, xi = make_case(case)
    for sync, graph in ((1, False), (8, False), (8, True), (4, True)):
        ctx = DistContext(f.shape, 0, 1, device="cuda:0", nccl_id=nccl_unique_id(), rounds_per_sync=sync,
                          graph=graph)
        for full in (False, True):
            r = ctx.correct(torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda(), xi, full_sweeps=full)
            assert r.status == ref.status == 0
            assert torch.equal(r.g.view(torch.int32), ref.g.view(torch.int32))
            assert torch.equal(r.edits, ref.edits)
            for k in STAT_KEYS:
                assert r.stats[k] == ref.stats[k], k
            # graph: round 1 eagerly, then the captured batch replayed (NCCL all-reduce inside)
            assert ctx.graph_used() == graph
        ctx.close()
