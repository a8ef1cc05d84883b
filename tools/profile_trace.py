#!/usr/bin/env python3
"""One timed trace of a converged config field (sizes first, outputs preallocated).
usage: python tools/profile_trace.py [C4] [--shape ...] [--repeat 1]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C4")
ap.add_argument("--shape", default=None)
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
shape = tuple(int(x) for x in a.shape.split(",")) if a.shape else None
f, fh, xi, cfg = di.config_inputs(a.config, shape=shape)
ctx = dmtz.Context(f.shape)
r = ctx.correct(torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda(), xi)
codes = ctx.compute_gradient(r.g)
sz = ctx.trace_sizes(codes)
bufs = ctx.trace_buffers(sz["n_branches"], sz["n_cells"], codes.device)
for _ in range(a.repeat):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = ctx.trace_separatrices(codes, out=bufs)
    torch.cuda.synchronize()
    print(f"trace {time.perf_counter() - t0:.3f} s", sz, flush=True)
