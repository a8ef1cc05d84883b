#!/usr/bin/env python3
"""Edit-stream encode / decode / apply on a config (for ncu captures of the codec
kernels).  usage: python tools/codec_probe.py [C4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
f, fh, xi, _ = di.config_inputs(name)
ft, fht = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
ctx = dmtz.context(ft.shape, ft.device)
r = ctx.correct(ft, fht, xi)
ev = r.edits[:r.n_edits]
for _ in range(2):
    s = ctx.encode_edits(ev, xi, 6, fhat=fht)
    d, _, _ = ctx.decode_edits(s, fhat=fht)
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
d, _, _ = ctx.decode_edits(s, fhat=fht)
e1.record()
torch.cuda.synchronize()
print(name, "edits", r.n_edits, "stream", s.numel(), "decode_ms", e0.elapsed_time(e1),
      "same", bool(torch.equal(d[:, :12], ev[:, :12])))
