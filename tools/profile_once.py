#!/usr/bin/env python3
"""One dmtz_correct call on a config (for ncu launch lists / --set full captures).
usage: python tools/profile_once.py [C4] [--shape 512,512,512] [--full] [--trace]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C4")
ap.add_argument("--shape", default=None)
ap.add_argument("--full", action="store_true")
ap.add_argument("--trace", action="store_true")
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
shape = tuple(int(x) for x in a.shape.split(",")) if a.shape else None
f, fh, xi, cfg = di.config_inputs(a.config, shape=shape)
ft, fht = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
ctx = dmtz.Context(f.shape)
for _ in range(a.repeat):
    r = ctx.correct(ft, fht, xi, full_sweeps=a.full, profile=True)
    print(r.status, r.stats, flush=True)
    if a.trace:
        tr = ctx.trace_separatrices(ctx.compute_gradient(r.g))
        print("branches", tr["origin"].shape[0], "cells", tr["cells"].shape[0])
torch.cuda.synchronize()
