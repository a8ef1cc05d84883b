#!/usr/bin/env python3
"""Connector-trace time per block size of the block BFS (DMTZ_BFS_THREADS), same output
checked across sizes.  usage: python tools/bfs_sweep.py C3 [C5 --planes 160]
The connectors of a config are traced over the origin planes [z0, z0 + planes) (all of
them when --planes is 0), one kind per call (kinds=4), CUDA events on the stream."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--planes", type=int, default=0)
ap.add_argument("--sizes", default="256,512,1024")
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
for cname in a.configs:
    f, fh, xi, cfg = di.config_inputs(cname)
    ctx = dmtz.Context(f.shape)
    r = ctx.correct(torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda(), xi)
    del f, fh
    codes = ctx.compute_gradient(r.g)
    del r
    nz = codes.shape[0]
    z0 = (nz - a.planes) // 2 if a.planes else 0
    z1 = z0 + a.planes if a.planes else nz
    sz = ctx.trace_sizes(codes, z_range=(z0, z1))
    bufs = ctx.trace_buffers(sz["n_branches"], sz["n_cells"], codes.device)
    stream = torch.cuda.current_stream()
    ref = None
    for bt in a.sizes.split(","):
        os.environ["DMTZ_BFS_THREADS"] = bt
        best = None
        for _ in range(a.repeat):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tr = ctx.trace_separatrices(codes, kinds=4, out=bufs, z_range=(z0, z1))
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        sig = (tr["cells"].shape[0], int(tr["cells"].sum().item()), int(tr["offsets"].sum().item()))
        ref = ref or sig
        print(f"{cname} planes [{z0},{z1}) bfs_threads {bt}: conn {best:.1f} ms, cells {sig[0]}, sum {sig[1]}, "
              f"same_output {sig == ref}", flush=True)
