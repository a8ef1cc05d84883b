"""Phase times of one separatrix trace of a config's converged g (DMTZ_TRACE_TIMES=1
prints them on stderr; the phases synchronise, so the sum exceeds the plain trace time).
usage: DMTZ_TRACE_TIMES=1 python tools/trace_phases.py C4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
f, fh, xi, cfg = di.config_inputs(name)
dev = torch.device("cuda", 0)
ctx = dmtz.Context(f.shape, dev)
r = ctx.correct(torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev), xi, q_max=cfg.q_max)
codes = ctx.compute_gradient(r.g)
sizes = ctx.trace_sizes(codes)
bufs = ctx.trace_buffers(sizes["n_branches"], sizes["n_cells"], dev)
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx.trace_separatrices(codes, out=bufs)
    torch.cuda.synchronize()
    print(f"{name} trace {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr, flush=True)
