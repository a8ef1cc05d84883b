#!/usr/bin/env python3
"""Projected multi-GPU C-loop time from a one-GPU emulation of the z-slab ranks.

Runs the slab driver with every rank's engine on the one visible GPU, strictly
sequentially (no rank waits on another inside a kernel), timing each rank's round
and halo refresh with CUDA events.  The projection for N GPUs is
    sum over rounds of  max over ranks (halo + round time)  +  an all-reduce latency,
i.e. the step of N GPUs that run their ranks concurrently, with the halo transfer
itself (3 planes per face, ~3 MB at 512^2, ~3.5 us over NVLink) and the counter
all-reduce taken as a fixed latency.  It is a projection, not a measurement: this
run has one GPU.  usage: python tools/slab_projection.py C4 2 4 8
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402
from paper_2409_17346_b200 import slab  # noqa: E402

ALLREDUCE_US = 20.0   # per-round NCCL all-reduce of 12 int64 + halo send/recv latency (assumed)


def run(name, world):
    f, fh, xi, cfg = di.config_inputs(name)
    dev = torch.device("cuda", 0)
    plans = [slab.plan(f.shape[0], world, r) for r in range(world)]
    engines = [slab.CudaSlabEngine(p, f.shape[1], f.shape[2], dev) for p in plans]
    loc = [slab.local_inputs(f, fh, p) for p in plans]
    fs = [torch.from_numpy(a).to(dev) for a, _ in loc]
    fhs = [torch.from_numpy(b).to(dev) for _, b in loc]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for rep in range(2):  # warm-up + timed
        for e, a, b in zip(engines, fs, fhs):
            e.begin(a, b, xi)
        torch.cuda.synchronize()
        per_round, r, status = [], 0, None
        while status is None:
            r += 1
            tr = []
            tot = np.zeros(12, np.int64)
            if r > 1:  # every rank's halo first (from the neighbours' round r - 1 values), then the rounds
                for e in engines:
                    e0, e1 = ev(), ev()
                    e0.record()
                    for peer, (sa, sb), (ra, rb) in slab.halo_pairs(e.p):
                        src = engines[peer]
                        (_, (psa, psb), _) = [x for x in slab.halo_pairs(src.p) if x[0] == e.p.rank][0]
                        e.halo(r - 1, ra, rb, src.g[psa:psb].clone())
                    e1.record()
                    torch.cuda.synchronize()
                    tr.append(e0.elapsed_time(e1))
            else:
                tr = [0.0] * len(engines)
            for i, e in enumerate(engines):
                e0, e1 = ev(), ev()
                e0.record()
                c, k = e.round(r)
                e1.record()
                torch.cuda.synchronize()
                tr[i] += e0.elapsed_time(e1)
                tot += np.concatenate([c, k])
            per_round.append(tr)
            status = slab._stop(r, tot, 0)
        outs = [e.end() for e in engines]
    n_edits = sum(int(o[0].shape[0]) for o in outs)
    # traces: owned-plane codes (concatenated = the all-gather), each rank's range trace
    full = torch.cat([slab.owned_codes(e) for e in engines])
    del engines, fs, fhs, outs   # free the ranks' loop state before the traces (C5: ~80 GB)
    torch.cuda.empty_cache()
    tctx = dmtz.Context(tuple(full.shape), dev)
    t_ranks = []
    for p in plans:
        sz = tctx.trace_sizes(full, 7, z_range=(p.z0, p.z1))
        bufs = tctx.trace_buffers(sz["n_branches"], sz["n_cells"], dev)
        tctx.trace_separatrices(full, 7, out=bufs, z_range=(p.z0, p.z1))
        e0, e1 = ev(), ev()
        e0.record()
        tctx.trace_separatrices(full, 7, out=bufs, z_range=(p.z0, p.z1))
        e1.record()
        torch.cuda.synchronize()
        t_ranks.append(e0.elapsed_time(e1))
        del bufs
    gather_ms = full.numel() * 8 * (world - 1) / world / 400e9 * 1e3   # NVLink all-gather at ~400 GB/s per GPU
    del full, tctx
    proj_ms = sum(max(t) for t in per_round) + len(per_round) * ALLREDUCE_US * 1e-3
    sweeps = r + 1
    return {"config": name, "world": world, "rounds": r, "status": status, "n_edits": n_edits,
            "projected_ms": proj_ms, "sum_rank_ms": sum(sum(t) for t in per_round),
            "projected_value_mvox_s": f.size * sweeps / (proj_ms * 1e-3) / 1e6,
            "trace_rank_ms": t_ranks, "trace_projected_ms": max(t_ranks) + gather_ms,
            "note": "one-GPU emulation; per-round max over ranks + fixed all-reduce latency; trace: max over "
                    "ranks of the range trace + codes all-gather at 400 GB/s"}


if __name__ == "__main__":
    name = sys.argv[1]
    for w in [int(x) for x in sys.argv[2:]]:
        print(json.dumps(run(name, w)), flush=True)
