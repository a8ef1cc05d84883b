#!/usr/bin/env python3
"""A/B timing of the round kernels on a config: one full-sweep step and one default
step with per-kernel CUDA events (profile=True).  Run twice, e.g. with DMTZ_NO_KEYS=1.
usage: python tools/screen_ab.py [C4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
f, fh, xi, cfg = di.config_inputs(name)
ft, fht = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
ctx = dmtz.Context(f.shape)
ctx.correct(ft, fht, xi, full_sweeps=True)
for full in (True, False):
    r = ctx.correct(ft, fht, xi, full_sweeps=full, profile=True)
    s = r.stats
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.correct(ft, fht, xi, full_sweeps=full)
    torch.cuda.synchronize()
    e0.record()
    r2 = ctx.correct(ft, fht, xi, full_sweeps=full)
    e1.record()
    torch.cuda.synchronize()
    print(f"{os.environ.get('TAG', '')} {name} full={full}: step {e0.elapsed_time(e1):.2f} ms  screen {s['screen_ms']:.2f} "
          f"decode {s['decode_ms']:.2f}  screen/full-launch "
          f"{s['screen_ms_full'] / max(s['n_screen_full'], 1):.3f} ms  rounds {s['rounds']} edits {r2.n_edits}",
          flush=True)
