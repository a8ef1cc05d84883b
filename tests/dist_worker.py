"""Worker of tests/test_gpu_dist.py: one rank of the library's multi-GPU C-loop
(DistContext over a host-staged gloo transport), all ranks sharing cuda:0.  Writes the
rank's owned g, edits and stats to <outdir>/rank<r>.npz."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def make_case(case):
    import dmtz_inputs as di
    if case["kind"] == "config":
        f, fh, xi, _ = di.config_inputs(case["name"], shape=tuple(case["shape"]))
        return f, fh, xi
    if case["kind"] == "stuck":   # reading A10: RU(f - xi) merges values -> STUCK
        rng = np.random.default_rng(case.get("seed", 3))
        f = (rng.standard_normal(tuple(case["shape"])) * 1e-6).astype(np.float32)
        fh = (f + rng.uniform(-0.45, 0.45, f.shape).astype(np.float32)).astype(np.float32)
        return f, fh, 0.5
    f, fh, xi = di.random_case(tuple(case["shape"]), case.get("seed", 1), eps=case.get("eps", 2e-2),
                               family=case.get("family", "noise"), perturb=case.get("perturb", "lorenzo"))
    return f, fh, xi


def worker(rank, world, port, case, outdir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2409_17346_b200.dist import DistContext, gloo_transport
    f, fh, xi = make_case(case)
    ctx = DistContext(f.shape, rank, world, device="cuda:0", rounds_per_sync=case.get("sync", 8))
    ctx.set_transport(*gloo_transport())
    ft = torch.from_numpy(np.ascontiguousarray(f[ctx.z0:ctx.z1])).cuda()
    fht = torch.from_numpy(np.ascontiguousarray(fh[ctx.z0:ctx.z1])).cuda()
    r = ctx.correct(ft, fht, xi, q_cap=case.get("q_cap"), max_rounds=case.get("max_rounds", 0),
                    full_sweeps=case.get("full", False), raise_on_error=False)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), g=r.g.cpu().numpy(), edits=r.edits.cpu().numpy(),
             stats=json.dumps(r.stats), status=r.status, z=np.array([ctx.z0, ctx.z1]))
    dist.barrier()
    dist.destroy_process_group()
