"""Multi-rank slab C-loop: partition / halo logic, and the whole driver against the
single-domain oracle -- emulated in one process and over torch.distributed gloo with
world size 2 on CPU (the NCCL/GPU path runs the same driver)."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import dmtz_inputs as di
import oracle
from paper_2409_17346_b200 import slab
from tests.slab_engines import OracleSlabEngine


@pytest.mark.parametrize("nz,world", [(12, 2), (13, 3), (9, 3), (40, 4), (24, 8)])
def test_partition_covers_and_halos(nz, world):
    parts = slab.partition(nz, world)
    assert parts[0][0] == 0 and parts[-1][1] == nz
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    assert all(z1 - z0 >= slab.HALO for z0, z1 in parts)
    for r in range(world):
        p = slab.plan(nz, world, r)
        a0, a1 = p.anchor_local
        # classified anchors: every anchor whose false cell can target an owned vertex
        assert p.lz0 + a0 == max(0, p.z0 - 2) and p.lz0 + a1 == min(nz, p.z1 + 1)
        # criticality of those anchors reads values in [z0 - 3, z1 + 3): inside the local grid
        assert p.lz0 <= max(0, p.z0 - 3) and p.lz1 >= min(nz, p.z1 + 3)
        for peer, (sa, sb), (ra, rb) in slab.halo_pairs(p):
            q = slab.plan(nz, world, peer)
            back = [x for x in slab.halo_pairs(q) if x[0] == r][0]
            # what I receive is exactly what the peer sends me, plane for plane (global z)
            assert list(range(q.lz0 + back[1][0], q.lz0 + back[1][1])) == list(range(p.lz0 + ra, p.lz0 + rb))
            assert list(range(p.lz0 + sa, p.lz0 + sb)) == list(range(q.lz0 + back[2][0], q.lz0 + back[2][1]))
            assert p.z0 <= p.lz0 + sa and p.lz0 + sb <= p.z1   # only owned planes are sent
    with pytest.raises(ValueError):
        slab.partition(5, 2)


def _case(shape, seed):
    return di.random_case(shape, seed, eps=0.05, perturb="noise", family="lognormal")


def _check_against_oracle(f, fh, xi, outs, stats, max_rounds=0):
    ref = oracle.correct(f, fh, xi, max_rounds=max_rounds)
    assert stats["status"] == ref["status"]
    assert stats["rounds"] == ref["stats"]["rounds"]
    assert stats["n_false_round0"] == ref["stats"]["n_false_round0"]
    assert stats["false_by_kind_round0"] == ref["stats"]["false_by_kind_round0"]
    e = np.concatenate([o[0] for o in outs])
    assert np.array_equal(e["v"], ref["edits"]["v"])
    assert np.array_equal(e["q"], ref["edits"]["q"])
    assert np.array_equal(e["lossless"], ref["edits"]["lossless"])
    assert np.array_equal(e["value"].view(np.uint32), ref["edits"]["value"].view(np.uint32))


@pytest.mark.parametrize("shape,world,seed", [((12, 7, 9), 2, 1), ((13, 6, 5), 3, 2), ((24, 5, 6), 4, 3)])
def test_slab_emulated_oracle_engine(shape, world, seed):
    f, fh, xi = _case(shape, seed)
    plans = [slab.plan(shape[0], world, r) for r in range(world)]
    engines = [OracleSlabEngine(p, shape[1], shape[2]) for p in plans]
    fs, fhs = zip(*[slab.local_inputs(f, fh, p) for p in plans])
    outs, stats = slab.run_emulated(engines, fs, fhs, xi)
    assert stats["rounds"] > 1
    _check_against_oracle(f, fh, xi, outs, stats)


def _gloo_worker(rank, world, port, shape, seed, outdir, max_rounds=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f, fh, xi = _case(shape, seed)
    p = slab.plan(shape[0], world, rank)
    lf, lfh = slab.local_inputs(f, fh, p)
    eng = OracleSlabEngine(p, shape[1], shape[2])
    edits, _, stats = slab.run_distributed(eng, torch.from_numpy(lf), torch.from_numpy(lfh), xi, max_rounds=max_rounds)
    np.save(os.path.join(outdir, f"edits{rank}.npy"), edits)
    np.save(os.path.join(outdir, f"stats{rank}.npy"), np.array([stats["status"], stats["rounds"],
                                                                 stats["n_false_round0"]] +
                                                                stats["false_by_kind_round0"], np.int64))
    dist.destroy_process_group()


@pytest.mark.parametrize("max_rounds", [0, 3])
def test_slab_gloo_world2(max_rounds):
    """The pipelined driver (stop decision one round behind) over gloo, world size 2;
    max_rounds = 3 ends on ITER_CAP without running a round past the cap."""
    shape, seed, world = (14, 7, 8), 5, 2
    with tempfile.TemporaryDirectory() as d:
        port = 29500 + (os.getpid() % 1000) + max_rounds
        mp.spawn(_gloo_worker, args=(world, port, shape, seed, d, max_rounds), nprocs=world, join=True)
        outs = [(np.load(os.path.join(d, f"edits{r}.npy")), 0) for r in range(world)]
        st = [np.load(os.path.join(d, f"stats{r}.npy")) for r in range(world)]
    assert all(np.array_equal(st[0], s) for s in st)   # every rank took the same decisions
    stats = dict(status=int(st[0][0]), rounds=int(st[0][1]), n_false_round0=int(st[0][2]),
                 false_by_kind_round0=[int(x) for x in st[0][3:11]])
    f, fh, xi = _case(shape, seed)
    _check_against_oracle(f, fh, xi, outs, stats, max_rounds)
    assert stats["status"] == (6 if max_rounds else 0)


@pytest.mark.gpu
@pytest.mark.parametrize("name,shape,world", [("C4", (40, 37, 33), 2), ("C4", (40, 37, 33), 4),
                                              ("C3", (30, 60, 70), 3), ("C4", (96, 96, 96), 8)])
def test_slab_cuda_emulated_matches_single_gpu(name, shape, world):
    """P slab ranks of the CUDA engine stepped in one process on one GPU (in-memory
    halos) reproduce the single-GPU dmtz_correct bit for bit."""
    import paper_2409_17346_b200 as dmtz
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    dev = torch.device("cuda", 0)
    ref = dmtz.correct(torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev), xi)
    plans = [slab.plan(shape[0], world, r) for r in range(world)]
    engines = [slab.CudaSlabEngine(p, shape[1], shape[2], dev) for p in plans]
    loc = [slab.local_inputs(f, fh, p) for p in plans]
    outs, stats = slab.run_emulated(engines, [torch.from_numpy(a).to(dev) for a, _ in loc],
                                    [torch.from_numpy(b).to(dev) for _, b in loc], xi)
    assert stats["status"] == ref.status and stats["rounds"] == ref.stats["rounds"]
    assert stats["n_false_round0"] == ref.stats["n_false_round0"]
    assert stats["false_by_kind_round0"] == ref.stats["false_by_kind_round0"]
    e = torch.cat([o[0] for o in outs])
    assert torch.equal(e, ref.edits)
    g = torch.cat([eng.owned_g() for eng in engines])
    assert torch.equal(g.view(torch.int32), ref.g.view(torch.int32))


# ----------------------------------------------------------------------------- multi-GPU trace
def _gather_worker(rank, world, port, nz, d):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = slab.partition(nz, world)[rank]
    full = torch.arange(nz * 3 * 2, dtype=torch.int64).reshape(nz, 3, 2)
    got = slab.gather_planes(full[a:b].clone(), nz, world)
    np.save(os.path.join(d, f"g{rank}.npy"), got.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("nz,world", [(7, 2), (11, 3)])
def test_gather_planes_gloo(nz, world):
    """The trace's gradient replication: uneven slabs all-gathered back into the grid."""
    with tempfile.TemporaryDirectory() as d:
        port = 29700 + (os.getpid() % 200) + nz
        mp.spawn(_gather_worker, args=(world, port, nz, d), nprocs=world, join=True)
        full = np.arange(nz * 3 * 2, dtype=np.int64).reshape(nz, 3, 2)
        for r in range(world):
            assert np.array_equal(np.load(os.path.join(d, f"g{r}.npy")), full)


@pytest.mark.gpu
@pytest.mark.parametrize("name,shape,world", [("C4", (40, 37, 33), 3), ("C3", (30, 60, 70), 2)])
def test_trace_distributed_emulated(name, shape, world):
    """Multi-GPU trace, ranks emulated on one GPU: each rank's owned-plane codes (from its
    local g) concatenate to the one-GPU gradient of g, and the ranks' range traces
    concatenate, kind by kind, to the one-GPU trace."""
    import paper_2409_17346_b200 as dmtz
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    dev = torch.device("cuda", 0)
    ref = dmtz.correct(torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev), xi)
    codes = dmtz.compute_gradient(ref.g)
    full = dmtz.trace_separatrices(codes)
    plans = [slab.plan(shape[0], world, r) for r in range(world)]
    engines = [slab.CudaSlabEngine(p, shape[1], shape[2], dev) for p in plans]
    loc = [slab.local_inputs(f, fh, p) for p in plans]
    slab.run_emulated(engines, [torch.from_numpy(a).to(dev) for a, _ in loc],
                      [torch.from_numpy(b).to(dev) for _, b in loc], xi)
    gathered = torch.cat([slab.owned_codes(e) for e in engines])
    assert torch.equal(gathered, codes)
    ctx = dmtz.Context(shape, dev)
    parts = [ctx.trace_separatrices(gathered, z_range=(p.z0, p.z1)) for p in plans]

    def cells_of(tr, i):
        return tr["cells"][tr["offsets"][i]:tr["offsets"][i + 1]]

    for kind in (dmtz.KIND_DESC, dmtz.KIND_ASC, dmtz.KIND_CONN):
        sel = (full["kind"] == kind).nonzero().flatten()
        got_o, got_t, got_len, got_c = [], [], [], []
        for tr in parts:
            s = (tr["kind"] == kind).nonzero().flatten()
            got_o.append(tr["origin"][s])
            got_t.append(tr["terminal"][s])
            got_len.append(tr["offsets"][s + 1] - tr["offsets"][s])
            got_c += [cells_of(tr, int(i)) for i in s]
        assert torch.equal(torch.cat(got_o), full["origin"][sel])
        assert torch.equal(torch.cat(got_t), full["terminal"][sel])
        assert torch.equal(torch.cat(got_len), full["offsets"][sel + 1] - full["offsets"][sel])
        exp = [cells_of(full, int(i)) for i in sel[:: max(1, len(sel) // 200)]]
        sub = got_c[:: max(1, len(sel) // 200)]
        assert all(torch.equal(a, b) for a, b in zip(sub, exp))


def test_library_local_slab_matches_plan():
    """dmtz_local_slab (the library's partition, a host function) equals slab.plan."""
    from paper_2409_17346_b200 import dist as dd
    for nz in range(3, 60):
        for w in range(1, nz // 3 + 1):
            for r in range(w):
                p = slab.plan(nz, w, r)
                assert dd.local_slab(nz, w, r) == (p.z0, p.z1, p.lz0, p.lz1)
    import paper_2409_17346_b200 as d
    with pytest.raises(d.DmtzError):
        dd.local_slab(8, 3, 0)     # fewer than 3 planes per rank
    with pytest.raises(d.DmtzError):
        dd.local_slab(30, 3, 3)    # rank out of range
