#!/usr/bin/env python3
"""Per-round counters and screen/decode device times of one dmtz_correct call
(host-driven rounds, DMTZ_VERBOSE=1 lines on stderr).  usage: DMTZ_VERBOSE=1 python tools/round_log.py C4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import dmtz_inputs as di
import paper_2409_17346_b200 as dmtz

f, fh, xi, _ = di.config_inputs(sys.argv[1] if len(sys.argv) > 1 else "C4")
ft, fht = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
ctx = dmtz.context(ft.shape, ft.device)
ctx.correct(ft, fht, xi)
r = ctx.correct(ft, fht, xi, profile=True)
print(r.stats, file=sys.stderr)
