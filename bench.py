#!/usr/bin/env python3
"""Benchmark of the DMTz hot path on B200 (contract: one JSON line on rank 0).

A STEP is one pass of the whole hot path over one synthetic input: the C-loop
to its fixed point (a1-a8 of SURVEY.md §8a: setup, reference gradient, every
round's gradient sweep + classification + edits, edit-list emission) with
full sweeps (every round evaluates every anchor), followed by the V-path
traces of the converged field (a9-a11) when the library provides them.

metric  "C-loop Mvoxels/s per iteration" = N * sweeps / step time (BASELINE.json)
e2e     the same metric through the public API from HOST arrays: pinned H2D of
        f and fhat, the C-loop, D2H of g and the edit list, every step
roofline the sweep of one round (gradient codes of g + classification), timed
        with CUDA events on the launching stream inside the library, against
        12 B/voxel algorithmic traffic (read g f32 + cand_f u64)
Workload: BASELINE config C4 (3D 512^3 lognormal "cosmology" field, rel. eps
1e-4, closed-loop Lorenzo quantizer), inputs 537 MB each > 126 MB L2.

--impl reference times the CPU oracle (this tier's reference arm) on a bounded
crop of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import dmtz_inputs as di  # noqa: E402


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index=0):
        self.rows, self._stop, self.idx = [], threading.Event(), gpu_index
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def oracle_sample(f, fh, xi, edge, budget_s=20.0):
    """Time the oracle (as it stands) on a bounded crop of the workload."""
    import oracle
    oracle.build()
    crop = tuple(slice(0, min(edge, s)) for s in f.shape)
    fc, fhc = np.ascontiguousarray(f[crop]), np.ascontiguousarray(fh[crop])
    t0 = time.perf_counter()
    r = oracle.correct(fc, fhc, xi)
    dt = time.perf_counter() - t0
    n = fc.size
    sweeps = r["stats"]["rounds"] + 1
    return dict(value=n * sweeps / dt / 1e6, seconds=dt, sweeps=sweeps, shape=list(fc.shape), rounds=r["stats"]["rounds"],
                threads=oracle.num_threads())


def run_reference(args, cfg, f, fh, xi):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_cores()))
    vals = []
    for i in range(args.warmup + args.steps):
        s = oracle_sample(f, fh, xi, args.ref_edge)
        if i >= args.warmup:
            vals.append(s)
    v = float(np.median([s["value"] for s in vals]))
    sample = (f"oracle C-loop to fixed point on the {vals[0]['shape']} crop of {cfg.name} "
              f"({vals[0]['sweeps']} sweeps, {vals[0]['seconds']:.1f} s each)")
    line = {"impl": "reference", "metric": "C-loop Mvoxels/s per iteration", "value": v, "unit": "Mvoxels/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.median([s["seconds"] for s in vals]) * 1e3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, cfg.shape))} eps {cfg.eps} (crop)",
                       "crop": vals[0]["shape"], "parallelism": "host cores"},
            "cpu_baseline": {"value": v, "unit": "Mvoxels/s", "cores": vals[0]["threads"], "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "Mvoxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dmtz", choices=["dmtz", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--shape", default=None, help="override config shape, e.g. 128,128,128")
    ap.add_argument("--ref-edge", type=int, default=64, help="oracle crop edge for the CPU baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "dmtz" else args.warmup

    shape = tuple(int(x) for x in args.shape.split(",")) if args.shape else None
    t0 = time.time()
    f, fh, xi, cfg = di.config_inputs(args.config, shape=shape)
    t_gen = time.time() - t0
    if args.impl == "reference":
        return run_reference(args, cfg, f, fh, xi)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2409_17346_b200 as dmtz

    dev = torch.device("cuda", local)
    ft = torch.from_numpy(f).to(dev)
    fht = torch.from_numpy(fh).to(dev)
    ctx = dmtz.Context(f.shape, dev)
    g = torch.empty_like(ft)
    edits = torch.empty((f.size, 16), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    has_trace = True

    def step(profile=False):
        nonlocal has_trace
        r = ctx.correct(ft, fht, xi, full_sweeps=True, g_out=g, edits=edits, profile=profile)
        ntr = 0
        if has_trace:
            try:
                codes = ctx.compute_gradient(g)
                tr = ctx.trace_separatrices(codes)
                ntr = int(tr["origin"].shape[0])
            except dmtz.DmtzError:
                has_trace = False
        return r, ntr

    for _ in range(args.warmup):
        r, _ = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times, sweeps, launches, prof = [], [], 0, []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r, ntr = step(profile=True)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            sweeps.append(r.stats["sweeps"])
            launches += r.stats.get("launches", 0)
            prof.append(r.stats)
    ms = float(np.median(times))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    N = f.size
    sw = int(np.median(sweeps))
    value = N * sw / (ms * 1e-3) / 1e6

    # roofline of the per-round sweep (codes of g + classification), live CUDA events
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs")
    sweep_ms = float(np.median([p["sweep_ms"] / max(p["sweeps"], 1) for p in prof]))
    bytes_alg = N * (12 if len(f.shape) == 3 else 6)
    achieved = bytes_alg / (sweep_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm if hbm else None, "traffic": None,
            "kernel": "round sweep (gradient of g + classification)", "kernel_ms": sweep_ms,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else "fallback 6650 GB/s"}
    if not hbm:
        roof["peak"] = 6650.0
        roof["frac"] = achieved / 6650.0

    # time-to-fixed-point in the default (frontier) mode: device-resident inputs -> g + edit list
    ttfp = []
    for i in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rf = ctx.correct(ft, fht, xi, full_sweeps=False, g_out=g, edits=edits)
        e1.record(stream)
        torch.cuda.synchronize()
        ttfp.append(e0.elapsed_time(e1))
    assert rf.stats["rounds"] == r.stats["rounds"] and rf.n_edits == r.n_edits
    frontier = {"time_to_fixed_point_ms": float(np.median(ttfp)), "rounds": rf.stats["rounds"],
                "anchors_swept": rf.stats["anchors_swept"], "sweeps": rf.stats["sweeps"],
                "full_sweep_equivalents": rf.stats["anchors_swept"] / N}

    e2e = None
    if not args.no_e2e:
        fp = torch.from_numpy(f).pin_memory()
        fhp = torch.from_numpy(fh).pin_memory()
        gh = torch.empty(f.shape, dtype=torch.float32).pin_memory()
        eh = torch.empty((f.size, 16), dtype=torch.uint8).pin_memory()
        et = []
        for i in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ft.copy_(fp, non_blocking=True)
            fht.copy_(fhp, non_blocking=True)
            r2, _ = step()
            gh.copy_(g, non_blocking=True)
            ne = r2.n_edits
            eh[:ne].copy_(edits[:ne], non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            et.append(e0.elapsed_time(e1))
        ems = float(np.median(et))
        e2e = {"value": N * r2.stats["sweeps"] / (ems * 1e-3) / 1e6, "unit": "Mvoxels/s",
               "h2d_bytes_per_step": 2 * 4 * N, "d2h_bytes_per_step": 4 * N + 16 * r2.n_edits,
               "ms_per_step": ems}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        s = oracle_sample(f, fh, xi, args.ref_edge)
        cpu = {"value": s["value"], "unit": "Mvoxels/s", "cores": s["threads"], "kind": "oracle",
               "sample": f"oracle C-loop to fixed point on the {s['shape']} crop of {cfg.name} "
                         f"({s['sweeps']} sweeps in {s['seconds']:.1f} s)"}

    st = r.stats
    line = {
        "metric": "C-loop Mvoxels/s per iteration", "value": value, "unit": "Mvoxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, f.shape))} rel eps {cfg.eps}",
                   "xi": xi, "q_max": 6, "q_cap": 6, "tier": 2, "sweeps_per_step": sw,
                   "rounds": st["rounds"], "full_sweeps": True, "l2": "inputs > L2 (537 MB each)",
                   "parallelism": f"slab{world}" if world > 1 else "1 GPU"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "frontier_mode": frontier,
        "gpu_launches": launches // max(args.steps, 1),
        "clocks": clk.summary(),
        "stats": {k: st[k] for k in ("rounds", "sweeps", "n_edited", "n_quantized", "n_lossless", "n_false_round0",
                                     "false_by_kind_round0")},
        "gen_seconds": t_gen,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
