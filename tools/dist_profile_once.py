"""One DistContext (one-rank NCCL) dmtz_correct on a config, for ncu launch lists of the
distributed driver.  usage: python tools/dist_profile_once.py C4 [--full] [--sync K]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmtz_inputs as di  # noqa: E402
from paper_2409_17346_b200.dist import DistContext, nccl_unique_id  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C4")
ap.add_argument("--full", action="store_true")
ap.add_argument("--sync", type=int, default=8)
ap.add_argument("--graph", action="store_true")
a = ap.parse_args()
f, fh, xi, cfg = di.config_inputs(a.config)
dev = torch.device("cuda", 0)
ctx = DistContext(f.shape, 0, 1, device=dev, nccl_id=nccl_unique_id(), rounds_per_sync=a.sync,
                  graph=a.graph)
ft, fht = torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev)
for _ in range(int(os.environ.get("REPS", "2"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = ctx.correct(ft, fht, xi, q_max=cfg.q_max, full_sweeps=a.full)
    e1.record()
    torch.cuda.synchronize()
    print(f"{a.config} dist full={a.full} sync={a.sync} graph={a.graph} (used {ctx.graph_used()}): "
          f"{e0.elapsed_time(e1):.1f} ms, rounds {r.stats['rounds']}", flush=True)
