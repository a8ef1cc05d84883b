#!/usr/bin/env python3
"""q_max sweep ("we evaluate different values of q_max and select
q_max = 6 based on a trade-off between storage and computational overhead"): for each
q_max (q_cap = q_max, reading A6) the C-loop's rounds, device time to the fixed point,
edits (quantized / lossless) and edit-stream bytes on one config.
usage: python tools/qmax_sweep.py C3 [tier]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import dmtz_inputs as di
import paper_2409_17346_b200 as dmtz

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
tier = int(sys.argv[2]) if len(sys.argv) > 2 else 2
f, fh, xi, cfg = di.config_inputs(name)
ft, fht = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
ctx = dmtz.context(ft.shape, ft.device)
stream = torch.cuda.current_stream()
for q_max in (2, 4, 6, 8, 10, 12):
    run = (lambda: ctx.preserve(ft, fht, xi, tier=tier, q_max=q_max)) if tier > 2 else \
          (lambda: ctx.correct(ft, fht, xi, q_max=q_max))
    run()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = run()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    s = ctx.encode_edits(r.edits[:r.n_edits], xi, q_max)
    st = r.stats
    print(json.dumps(dict(config=f"{cfg.name} {'x'.join(map(str, f.shape))}", tier=tier, q_max=q_max, status=r.status,
                          ms=float(np.median(ts)), rounds=st["rounds"], s_rounds=st.get("s_rounds", 0),
                          n_edited=r.n_edits, n_lossless=st["n_lossless"], n_quantized=st["n_quantized"],
                          edit_ratio=r.n_edits / f.size, stream_bytes=int(s.numel()),
                          bytes_per_edit=int(s.numel()) / max(r.n_edits, 1))), flush=True)
