#!/usr/bin/env python3
"""Time dmtz_preserve (tiers 2/3/4) on a config: rounds, troublemakers, device times.
usage: python tools/sloop_probe.py C3 [tier ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import dmtz_inputs as di
import paper_2409_17346_b200 as dmtz

name = sys.argv[1]
tiers = [int(t) for t in sys.argv[2:]] or [4]
f, fh, xi, _ = di.config_inputs(name)
ft, fht = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
ctx = dmtz.context(ft.shape, ft.device)
for tier in tiers:
    for rep in range(int(os.environ.get("REPS", "2"))):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = ctx.preserve(ft, fht, xi, tier=tier)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    s = r.stats
    print(json.dumps(dict(config=name, tier=tier, status=r.status, wall_s=round(dt, 4), n_edits=r.n_edits,
                          **{k: s.get(k) for k in ("rounds", "c_rounds", "s_rounds", "troublemakers", "tm_by_kind",
                                                   "tm_round1", "sep_branches", "sep_cells", "trace_ms", "s_ms",
                                                   "sweeps", "cells_checked")})), flush=True)
