"""Time the library's distributed C-loop driver on one GPU (a one-rank NCCL
communicator) in both synchronisation modes (dmtz_ctx_set_dist_sync), against the
one-GPU graph-driven loop, on a BASELINE config: the cost of the host hop per round."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dmtz_inputs as di  # noqa: E402
import paper_2409_17346_b200 as dmtz  # noqa: E402
from paper_2409_17346_b200.dist import DistContext, nccl_unique_id  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    f, fh, xi, cfg = di.config_inputs(a.config)
    dev = torch.device("cuda", 0)
    ft, fht = torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev)
    out = {"config": a.config}
    ctx = dmtz.Context(f.shape, dev)
    t, r = timed(lambda: ctx.correct(ft, fht, xi, q_max=cfg.q_max), a.reps)
    out["one_gpu_graph_ms"] = t
    out["rounds"] = r.stats["rounds"]
    ref_g = r.g.clone()
    del ctx
    for sync in (1, 8, 32):
        dc = DistContext(f.shape, 0, 1, device=dev, nccl_id=nccl_unique_id(), rounds_per_sync=sync)
        t, r = timed(lambda: dc.correct(ft, fht, xi, q_max=cfg.q_max), a.reps)
        assert torch.equal(r.g.view(torch.int32), ref_g.view(torch.int32))
        out[f"dist_sync{sync}_ms"] = t
        dc.close()
        del dc
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
