#!/usr/bin/env python3
"""Write the full-size oracle goldens tests/golden/oracle_full_<C>.json.

Calls only ``dmtz_inputs`` (seeded inputs) and ``oracle`` (the literal CPU oracle):
no value here comes from the CUDA path.  For a BASELINE config at its full size it
records the input sha256, the oracle C-loop's result (status, stats, false cells
per round, the digests of g -- whole and per z-plane -- and of the edit list) and
the oracle trace of the converged g (and, for the 2D config, of f) as branch /
cell counts plus digests (tests/digest.py; the oracle's digest mode, because the
C4 CSR does not fit in host memory).  The 3D configs use the oracle's frontier
mode (equal to the full loop, tests/test_oracle_frontier.py).

    python tools/oracle_goldens.py C2 C3 C4
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import dmtz_inputs as di  # noqa: E402
import oracle  # noqa: E402
from tests import digest as dg  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(names):
    for name in names:
        t0 = time.time()
        f, fhat, xi, cfg = di.config_inputs(name)
        out = {"config": name, "shape": list(cfg.shape), "eps": cfg.eps, "xi": xi,
               "xi_bits": int(np.float32(xi).view(np.uint32)), "q_max": cfg.q_max, "q_cap": cfg.q_max, "tier": 2,
               "input_sha256": {"f": sha(f), "fhat": sha(fhat)},
               "oracle_threads": oracle.num_threads(), "written_by": "tools/oracle_goldens.py (oracle/ only)"}
        print(f"[{name}] inputs {time.time() - t0:.1f}s", flush=True)
        frontier = len(cfg.shape) == 3
        t1 = time.time()
        r = oracle.correct(f, fhat, xi, q_max=cfg.q_max, frontier=frontier, round_log=True)
        out["correct_seconds"] = time.time() - t1
        out["mode"] = "frontier" if frontier else "full"
        out["status"] = r["status"]
        out["stats"] = r["stats"]
        out["false_per_round"] = r["false_per_round"]
        out["n_edits"] = r["n_edits"]
        g = r["g"]
        out["g_digest"] = dg.digest_np(g.view(np.uint32))
        if len(cfg.shape) == 3:
            per = g.shape[1] * g.shape[2]
            flat = g.reshape(-1).view(np.uint32)
            out["g_plane_digests"] = [dg.digest_np(flat[z * per:(z + 1) * per], start=z * per)
                                      for z in range(g.shape[0])]
        out["g_sha256"] = sha(g)
        out["edits_digest"] = dg.digest_np(r["edits"].view(np.uint64))
        out["state_digest"] = dg.digest_np(r["state"].reshape(-1))
        del r
        print(f"[{name}] correct {out['correct_seconds']:.1f}s status {out['status']} rounds "
              f"{out['stats']['rounds']} edits {out['n_edits']}", flush=True)
        fields = [("g", g)] + ([("f", f)] if len(cfg.shape) == 2 else [])
        for tag, fld in fields:
            t2 = time.time()
            nb, nc, d = oracle.trace_digest(fld)
            out[f"trace_{tag}"] = {"n_branches": nb, "n_cells": nc, "digests": d,
                                   "seconds": time.time() - t2}
            print(f"[{name}] trace of {tag}: {nb} branches {nc} cells {time.time() - t2:.1f}s", flush=True)
        path = os.path.join(ROOT, "tests", "golden", f"oracle_full_{name}.json")
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
        print(f"[{name}] wrote {path} ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C4"])
