#!/usr/bin/env python3
"""Small end-to-end case for compute-sanitizer: C-loop (graph + host-driven), gradient,
traces (all connector levels), slab rounds with halos, on boundary-heavy shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402
from paper_2409_17346_b200 import slab  # noqa: E402

dev = torch.device("cuda", 0)
for name, shape in [("C4", (9, 10, 11)), ("C3", (12, 33, 40)), ("C1", (17, 19)), ("C2", (30, 61))]:
    f, fh, xi, _ = di.config_inputs(name, shape=shape)
    ft, fht = torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev)
    for full in (False, True):
        r = dmtz.correct(ft, fht, xi, full_sweeps=full)
        r2 = dmtz.correct(ft, fht, xi, full_sweeps=full, profile=True)
    codes = dmtz.compute_gradient(r.g)
    tr = dmtz.trace_separatrices(codes)
    # every connector escalation level (thread -> warp -> block BFS levels)
    os.environ.update(DMTZ_TEST_CQ="2", DMTZ_TEST_WQ="8", DMTZ_TEST_BFS_GROW="2")
    tr2 = dmtz.trace_separatrices(codes)
    lv = dmtz.last_trace_levels()
    for k in ("DMTZ_TEST_CQ", "DMTZ_TEST_WQ", "DMTZ_TEST_BFS_GROW"):
        del os.environ[k]
    assert torch.equal(tr2["cells"], tr["cells"])
    # the S-loop (tier 4) and the edit codec
    r4 = dmtz.preserve(ft, fht, xi, tier=4)
    ctx = dmtz.context(f.shape, dev)
    blob = ctx.encode_edits(r4.edits, xi, fhat=fht)
    ed, x2, qm = ctx.decode_edits(blob, fhat=fht)
    print(name, shape, r.status, r.stats["rounds"], tr["origin"].shape[0], "levels", lv[:5], "tier4", r4.status,
          flush=True)
    if len(shape) == 3:
        plans = [slab.plan(shape[0], 3, k) for k in range(3)]
        eng = [slab.CudaSlabEngine(p, shape[1], shape[2], dev) for p in plans]
        loc = [slab.local_inputs(f, fh, p) for p in plans]
        slab.run_emulated(eng, [torch.from_numpy(a).to(dev) for a, _ in loc],
                          [torch.from_numpy(b).to(dev) for _, b in loc], xi)
torch.cuda.synchronize()
print("done")
