#!/usr/bin/env python3
"""One trace of the origin planes [z0, z1) of a converged config field (for launch lists).
usage: python tools/profile_trace_range.py C5 z0 z1"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402

name, z0, z1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
f, fh, xi, cfg = di.config_inputs(name)
ctx = dmtz.Context(f.shape)
r = ctx.correct(torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda(), xi)
codes = ctx.compute_gradient(r.g)
del r
sz = ctx.trace_sizes(codes, z_range=(z0, z1))
bufs = ctx.trace_buffers(sz["n_branches"], sz["n_cells"], codes.device)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = ctx.trace_separatrices(codes, out=bufs, z_range=(z0, z1))
    torch.cuda.synchronize()
    print(f"trace [{z0},{z1}) {time.perf_counter() - t0:.3f} s", sz, dmtz.last_trace_levels()[:6], flush=True)
