#!/usr/bin/env python3
"""Benchmark of the DMTz hot path on B200 (contract: one JSON line on rank 0).

STEP    one pass of the C-loop to its fixed point on one synthetic input (rows
        a1-a8 of SURVEY.md §8a: setup + bound check, reference gradient, every
        round's gradient screening + classification + Eq. 2 edits, edit-list
        emission) in the library's default mode: each round works on the dirty
        frontier and recomputes only codes whose 3x3x3 box changed (exact; the
        output is bit-identical to recomputing everything); the rounds run on the
        device inside one CUDA-graph WHILE node.  value = N * rounds / time, i.e.
        the time to the fixed point expressed per C-loop iteration.
full_recompute  the same step with full_sweeps=1 (every code, every anchor, every
        round): the per-iteration cost of a complete gradient recomputation
value   "C-loop Mvoxels/s per iteration" = N * sweeps / step time (BASELINE.json)
time_to_fixed_point  the step time, the second half of BASELINE's metric
trace   rows a9-a11 (descending / ascending / connector V-paths) of the
        converged field, timed once after the steps
e2e     the same metric through the public API from pinned HOST arrays: H2D of
        f and fhat, the C-loop, the edit list encoded on the device and D2H of the
        encoded stream (the storable artifact), every step
        (dmtz_correct_host_stream); e2e_raw: D2H of g and the raw 16-byte edit
        records instead (dmtz_correct_host)
roofline the dominant kernel, k_screen (gradient codes of g), on the rounds it
        sweeps every anchor, timed with CUDA events on the launching stream
        inside the library during one extra (host-driven) step; algorithmic work per anchor: 105 SoS compare-selects
        (210 ALU ops) and 12 B (g f32 + the stored u64 code), DESIGN.md §7
Workload: BASELINE config C4 (3D 512^3 lognormal "cosmology" field, rel. eps
1e-4, closed-loop Lorenzo quantizer); inputs 537 MB each > 126 MB L2.

--impl reference times the CPU oracle (this tier's reference arm) on a bounded
crop of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import hashlib
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

METRIC = "C-loop Mvoxels/s per iteration"
ALU_OPS_PER_ANCHOR = {3: 210, 2: 30}      # k_screen: 2 x SoS compares per anchor (105 in 3D, 15 in 2D)
BYTES_PER_ANCHOR = {3: 12, 2: 6}          # g f32 + stored code (u64 3D / u16 2D)
# k_decode: per decoded anchor, crit(c) for every cell type = cand(c) == NONE (20 / 4 tests) and no
# facet pointing at c (74 / 12 tests), each a field extract + compare (2 ops); per false cell, one
# target rule R1 / R2 / R3 (three field tests + two selects, 6 ops)  -- DESIGN.md section 7
DECODE_OPS_PER_ANCHOR = {3: 2 * (20 + 74), 2: 2 * (4 + 12)}
RULE_OPS_PER_CELL = 6


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _ncu_traffic(kernel: str, workload: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        w = d.get(workload, {})
        e = w.get(kernel + "@step") or w.get(kernel)   # mean over the step's launches, else one capture
        return e["dram_bytes"] if e else None
    except Exception:
        return None


def _ncu_issue(kernel: str, workload: str):
    """issue-active and ALU-pipe % of `kernel` from the committed ncu --set full capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        e = d.get(workload, {}).get(kernel)
        return {"issue_active_pct": e["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                "alu_pipe_pct": e["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"],
                "warps_active_pct": e["sm__warps_active.avg.pct_of_peak_sustained_active"],
                "report": e.get("report")} if e else None
    except Exception:
        return None


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


def oracle_round(f, fh, xi, planes=None):
    """The oracle (as it stands) on one full C-loop round of the workload: the literal
    gradient of g = fhat, the classification of every cell and the Eq. 2 edits
    (max_rounds = 1), optionally on the first ``planes`` z-planes only.  The round is
    timed inside the oracle (omp_get_wtime around the round; the one-off setup -- lb and
    the gradient of f -- is not part of a round).  Returns dict(value Mvox/s, ...)."""
    import oracle
    oracle.build()
    if planes is not None and f.ndim == 3:
        f, fh = np.ascontiguousarray(f[:planes]), np.ascontiguousarray(fh[:planes])
    t0 = time.perf_counter()
    r = oracle.correct(f, fh, xi, max_rounds=1, round_log=True)
    total = time.perf_counter() - t0
    t = r["round_seconds"][0]
    return dict(value=f.size / t / 1e6, round_seconds=t, call_seconds=total, shape=list(f.shape),
                threads=oracle.num_threads(), n_false=r["false_per_round"][0])


def run_reference(args, cfg, f, fh, xi):
    """--impl reference: this tier's reference arm is the CPU oracle.  Each step = one full
    C-loop round of the oracle on a bounded sample of the workload (the first
    --ref-planes z-planes of the config's field), the same unit as the GPU arm's value."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    vals = []
    for i in range(args.warmup + args.steps):
        s = oracle_round(f, fh, xi, planes=args.ref_planes)
        if i >= args.warmup:
            vals.append(s)
    v = float(np.median([s["value"] for s in vals]))
    sample = (f"one oracle C-loop round (literal gradient of g, classification, Eq. 2 edits) on z-planes "
              f"[0, {vals[0]['shape'][0]}) of {cfg.name} {'x'.join(map(str, cfg.shape))} "
              f"({vals[0]['round_seconds']:.2f} s per round, setup untimed)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Mvoxels/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.median([s["round_seconds"] for s in vals]) * 1e3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, cfg.shape))} rel eps {cfg.eps}",
                       "sample_shape": vals[0]["shape"], "parallelism": "host cores (OpenMP)"},
            "cpu_baseline": {"value": v, "unit": "Mvoxels/s", "cores": vals[0]["threads"], "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "Mvoxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def sloop_line(name, tiers, dev, stream, with_cpu):
    """Tiers 3-5: the alternating C/S workflow to its fixed point on
    one config, device-resident inputs, CUDA events on the launching stream (1 warm-up,
    median of 2), and the oracle's workflow on a crop of the same config."""
    import torch
    import paper_2409_17346_b200 as dmtz
    f, fh, xi, cfg = di.config_inputs(name)
    ft, fht = torch.from_numpy(f).to(dev), torch.from_numpy(fh).to(dev)
    ctx = dmtz.Context(f.shape, dev)
    out = {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, f.shape))} rel eps {cfg.eps}"}
    for tier in tiers:
        ctx.preserve(ft, fht, xi, tier=tier)
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = ctx.preserve(ft, fht, xi, tier=tier)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        s = r.stats
        rounds = s["c_rounds"] + s["s_rounds"]
        out[f"tier{tier}"] = {
            "status": r.status, "time_to_fixed_point_ms": ms,
            "value": f.size * (rounds + 1) / (ms * 1e-3) / 1e6, "unit": "Mvoxels/s (voxels x rounds / time)",
            "c_rounds": s["c_rounds"], "s_rounds": s["s_rounds"], "troublemakers": s["troublemakers"],
            "tm_by_kind": s["tm_by_kind"], "n_edited": r.n_edits, "sep_branches": s["sep_branches"],
            "sep_cells": s["sep_cells"], "trace_of_f_ms": s["trace_ms"], "s_rounds_ms": s["s_ms"],
            "cells_rechecked": s["cells_checked"],
            "note": "includes sizing the separatrix CSR (a trace of f) in the binding" }
        del r
        torch.cuda.empty_cache()
    del ctx
    torch.cuda.empty_cache()
    if with_cpu:
        import oracle
        crop = tuple(min(n, 64) for n in f.shape) if len(f.shape) == 3 else tuple(min(n, 240) for n in f.shape)
        sl = tuple(slice(0, n) for n in crop)
        fc, fhc = np.ascontiguousarray(f[sl]), np.ascontiguousarray(fh[sl])
        t0 = time.perf_counter()
        ro = oracle.preserve(fc, fhc, xi, tier=max(tiers))
        dt = time.perf_counter() - t0
        so = ro["stats"]
        n = fc.size * (so["c_rounds"] + so["s_rounds"] + 1)
        out["cpu_baseline"] = {"value": n / dt / 1e6, "unit": "Mvoxels/s (voxels x rounds / time)",
                               "cores": oracle.num_threads(), "kind": "oracle",
                               "sample": f"oracle tier-{max(tiers)} workflow on the {list(crop)} crop of {cfg.name} "
                                         f"({so['c_rounds']} C- + {so['s_rounds']} S-rounds in {dt:.1f} s)"}
    return out


def chunked_trace(ctx, codes, dev, stream, budget, sizes):
    """Trace of a field whose CSR exceeds the free memory: the branches whose origin is
    anchored in a group of z-planes per call (dmtz_trace_separatrices_range), groups
    sized to ``budget`` bytes of outputs, one set of output buffers reused.  Times the
    sum of the calls; the outputs of each group are overwritten by the next."""
    import torch
    nz = codes.shape[0]
    step = max(1, nz // 32)
    parts = []
    for z0 in range(0, nz, step):
        z1 = min(nz, z0 + step)
        s = ctx.trace_sizes(codes, z_range=(z0, z1))
        parts.append([z0, z1, s["n_branches"], s["n_cells"], s["n_branches"] * 33 + s["n_cells"] * 8])
    groups = []
    for p in parts:
        if groups and groups[-1][4] + p[4] <= budget:
            g = groups[-1]
            groups[-1] = [g[0], p[1], g[2] + p[2], g[3] + p[3], g[4] + p[4]]
        else:
            groups.append(list(p))
    if max(g[4] for g in groups) > budget:
        return {"skipped": f"a {step}-plane group needs {max(g[4] for g in groups) / 1e9:.1f} GB", **sizes}
    bufs = ctx.trace_buffers(max(g[2] for g in groups), max(g[3] for g in groups), dev)
    nb = nc = 0
    ms = 0.0
    for g in groups:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tr = ctx.trace_separatrices(codes, out=bufs, z_range=(g[0], g[1]))
        e1.record(stream)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
        nb += tr["origin"].shape[0]
        nc += tr["cells"].shape[0]
        del tr
    per_kind = {}
    for kname, kb in (("desc_ms", 1), ("asc_ms", 2), ("conn_ms", 4)):   # one kind per call
        per_kind[kname] = 0.0
        for g in groups:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.trace_separatrices(codes, kinds=kb, out=bufs, z_range=(g[0], g[1]))
            e1.record(stream)
            torch.cuda.synchronize()
            per_kind[kname] += e0.elapsed_time(e1)
    del bufs
    return {"trace_ms": ms, **per_kind, "n_branches": nb, "n_cells": nc, "groups": len(groups),
            "mode": f"branches by origin plane in {len(groups)} groups of <= {budget / 1e9:.0f} GB of outputs "
                    "(outputs not kept); per-group sizing untimed",
            "full_csr_gb": (sizes["n_branches"] * 33 + sizes["n_cells"] * 8) / 1e9,
            "counts_match_full_sizing": nb == sizes["n_branches"] and nc == sizes["n_cells"]}


def dist_bench(args, f, fh, xi, cfg, world, rank, local):
    """bench.py --gpus N (torchrun, one rank per GPU): the library's multi-GPU C-loop
    (dmtz_correct on a world-N context with its own NCCL communicator; z-slabs, halo
    exchange with face skipping, counter reduction per round).  Same step and metric
    as N = 1: the C-loop to its fixed point with full-sweep rounds, value = global N x
    sweeps / step time; device time = max over ranks (barrier + sync on both sides)."""
    import torch
    import torch.distributed as dist
    from paper_2409_17346_b200.dist import DistContext, nccl_unique_id
    dev = torch.device("cuda", local)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = DistContext(f.shape, rank, world, device=dev, nccl_id=obj[0])
    own = (slice(ctx.z0, ctx.z1),)
    ft = torch.from_numpy(np.ascontiguousarray(f[own])).to(dev)
    fht = torch.from_numpy(np.ascontiguousarray(fh[own])).to(dev)

    def timed(fn, reps):
        ts, out = [], None
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t.item()))
        return out, ts

    for _ in range(args.warmup):
        ctx.correct(ft, fht, xi, full_sweeps=True)
    with Clocks(local) as clk:
        rfull, times = timed(lambda: ctx.correct(ft, fht, xi, full_sweeps=True), args.steps)
        r, tt = timed(lambda: ctx.correct(ft, fht, xi), max(3, args.steps))
    ms, ttfp = float(np.median(times)), float(np.median(tt))
    sweeps = rfull.stats["sweeps"]
    N = f.size
    value = N * sweeps / (ms * 1e-3) / 1e6
    peaks = _peaks()
    hbm = (peaks.get("hbm_gbs") or 6650.0) * world
    ach = BYTES_PER_ANCHOR[3] * N / (ms / sweeps * 1e-3) / 1e9
    # end to end: the rank's owned planes from pinned host memory, its g planes and edits back
    fp, fhp = torch.from_numpy(np.ascontiguousarray(f[own])).pin_memory(), \
        torch.from_numpy(np.ascontiguousarray(fh[own])).pin_memory()
    gh = torch.empty(tuple(ft.shape), dtype=torch.float32).pin_memory()
    eh = torch.empty((ft.numel(), 16), dtype=torch.uint8).pin_memory()

    def e2e_step():
        ft.copy_(fp, non_blocking=True)
        fht.copy_(fhp, non_blocking=True)
        rr = ctx.correct(ft, fht, xi, full_sweeps=True)
        gh.copy_(rr.g, non_blocking=True)
        eh[:rr.n_edits].copy_(rr.edits, non_blocking=True)
        torch.cuda.synchronize()
        return rr.n_edits
    ne, et = timed(e2e_step, 2)
    ems = float(np.median(et))
    nb = torch.tensor([ne * 16 + gh.numel() * 4, fp.numel() * 8], device=dev, dtype=torch.int64)
    dist.all_reduce(nb)
    st = r.stats
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Mvoxels/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, f.shape))} rel eps {cfg.eps}",
                           "step": "C-loop to its fixed point, every round a full sweep (full_sweeps=1)",
                           "parallelism": f"z-slabs x{world}: dmtz_correct on world-{world} contexts (NCCL)",
                           "sweeps_per_step": sweeps, "rounds": rfull.stats["rounds"],
                           "l2": "inputs larger than L2"},
                "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                             "traffic": None, "kernel": "full-sweep C-loop round over all GPUs (12 B/voxel)",
                             "peak_source": f"MEASURED_PEAKS.json hbm_gbs x {world}"},
                "cpu_baseline": None,
                "e2e": {"value": N * sweeps / (ems * 1e-3) / 1e6, "unit": "Mvoxels/s", "ms_per_step": ems,
                        "h2d_bytes_per_step": int(nb[1].item()), "d2h_bytes_per_step": int(nb[0].item())},
                "gpu_launches": rfull.stats["launches"], "clocks": clk.summary(),
                "time_to_fixed_point": {"time_to_fixed_point_ms": ttfp, "rounds": st["rounds"],
                                        "halo_faces_sent": st["halo_faces_sent"],
                                        "halo_faces_skipped": st["halo_faces_skipped"]},
                "stats": {k: st[k] for k in ("rounds", "n_edited", "n_quantized", "n_lossless", "n_false_round0")}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dmtz", choices=["dmtz", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--shape", default=None, help="override the config shape, e.g. 128,128,128")
    ap.add_argument("--ref-planes", type=int, default=48,
                    help="--impl reference: z-planes of the field per oracle round (a bounded sample)")
    ap.add_argument("--detail", default=None, help="also write the full result dict to this JSON file "
                    "(default gpurun_out/bench_detail.json when gpurun_out/ exists)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-golden-parity", dest="golden_parity", action="store_false",
                    help="skip the full-size parity check against tests/golden/oracle_full_<C>.json")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--slab", action="store_true", help="run the multi-GPU slab path even with one rank")
    ap.add_argument("--sloop-config", default="C4:4,5,3;C2:3,4,5",
                    help="configs:tiers of the tier-3/4/5 workflow lines, e.g. 'C4:4,5;C2:3,4,5' ('none' skips)")
    args = ap.parse_args()
    if args.impl == "dmtz":
        args.warmup = max(args.warmup, 3)

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
    if world > 1 or args.slab:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2409_17346_b200 as dmtz
    if world > 1 or args.slab:
        return dist_bench(args, f, fh, xi, cfg, world, rank, local)

    dev = torch.device("cuda", local)
    D = len(f.shape)
    N = f.size
    ft = torch.from_numpy(f).to(dev)
    fht = torch.from_numpy(fh).to(dev)
    ctx = dmtz.Context(f.shape, dev)
    g = torch.empty_like(ft)
    edits = torch.empty((N, 16), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(full=False, profile=False):
        return ctx.correct(ft, fht, xi, full_sweeps=full, g_out=g, edits=edits, profile=profile)

    def timed(fn, reps):
        ts, out = [], None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return out, ts

    # THE STEP: one pass of the C-loop to its fixed point with every round a full sweep
    # (full_sweeps=1: every code of g recomputed, every anchor classified in every round);
    # value = N x sweeps / step time = SURVEY.md §8(d-1)'s full-sweep round throughput.
    for _ in range(args.warmup):
        step(full=True)
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        rfull, times = timed(lambda: step(full=True), args.steps)
        # time to the fixed point in the library's default mode (dirty frontier + exact
        # change skipping, bit-identical output): the second half of BASELINE's metric
        r, ttfp_t = timed(step, max(3, args.steps))
        # per-kernel CUDA events (host-driven rounds, one extra step each) for the roofline
        rp = step(full=True, profile=True)
        rpd = step(profile=True)
    assert rfull.n_edits == r.n_edits and rfull.stats["rounds"] == r.stats["rounds"]
    ms = float(np.median(times))
    sweeps = rfull.stats["sweeps"]
    t_round = ms / sweeps
    value = N / (t_round * 1e-3) / 1e6
    ttfp = float(np.median(ttfp_t))

    peaks = _peaks()
    hbm = peaks.get("hbm_gbs") or 6650.0
    sm_mhz = peaks.get("sm_max_mhz") or 1965.0
    alu_peak = 148 * 64 * sm_mhz * 1e6 / 1e9          # Gop/s: 148 SMs x 4 SMSP x 16-lane ALU pipe
    workload = f"{cfg.name} {'x'.join(map(str, f.shape))}"
    ps = rp.stats
    # the full-sweep round's kernels (CUDA events on the launching stream, host-driven step)
    k_ms = {"screen": ps["screen_ms"], "decode": ps["decode_ms"], "edit": ps.get("edit_ms", 0.0)}
    round_dev_ms = sum(k_ms.values()) / sweeps
    alg_bytes = BYTES_PER_ANCHOR[D] * N           # per full-sweep round (g f32 + the f code)
    ach = alg_bytes / (t_round * 1e-3) / 1e9
    ncu_round = _ncu_traffic("round@full", workload)
    roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
            "traffic": ncu_round,
            "kernel": "full-sweep C-loop round (k_screen + k_decode + k_edit_rows), SURVEY §8(d-1)",
            "algorithmic_bytes_per_voxel": BYTES_PER_ANCHOR[D], "t_round_ms": t_round,
            "kernel_ms_per_round": {k: v / sweeps for k, v in k_ms.items()},
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
            "traffic_note": "ncu dram__bytes read+write of one full-sweep round's kernels (profiles/ncu_summary.json)"}
    t_launch = ps["screen_ms_full"] / max(ps["n_screen_full"], 1) * 1e-3
    nc = _ncu_issue("k_screen", workload)
    alu_frac = nc["alu_pipe_pct"] / 100.0 if nc else None
    roof_alu = {"bound": "alu", "kernel": "k_screen (gradient codes of g, one full-sweep launch)",
                "achieved": alu_frac * alu_peak if alu_frac is not None else None, "peak": alu_peak,
                "unit": "G ALU-pipe instr/s (lanes)", "frac": alu_frac, "launch_ms": t_launch * 1e3,
                "compares_per_anchor": ALU_OPS_PER_ANCHOR[D] // 2,
                "compares_per_s": ALU_OPS_PER_ANCHOR[D] // 2 * N / t_launch / 1e9, "ncu": nc,
                "source": "frac = ncu sm__inst_executed_pipe_alu of the committed capture (profiles/ncu_summary.json)",
                "peak_source": "ALU pipe: 148 SMs x 64 lanes/clk x sm_max_mhz (B300_MICROARCH: alu rt=2/SMSP)"}
    ds = rpd.stats
    frontier = {"time_to_fixed_point_ms": ttfp, "rounds": r.stats["rounds"], "sweeps": r.stats["sweeps"],
                "codes_recomputed_full_sweep_equivalents": r.stats["anchors_recomputed"] / N,
                "kernel_ms": {"screen": ds["screen_ms"], "decode": ds["decode_ms"], "edit": ds.get("edit_ms", 0.0)},
                "gpu_launches": r.stats["launches"]}

    # traces of the converged field (a9-a11), once; CSR digests for the parity check
    trace, csr_dig = None, None
    if not args.no_trace:
        codes = ctx.compute_gradient(g)
        try:
            sizes = ctx.trace_sizes(codes)
            need = sizes["n_branches"] * 33 + sizes["n_cells"] * 8
            free = torch.cuda.mem_get_info()[0]
            if need < 0.8 * free:
                bufs = ctx.trace_buffers(sizes["n_branches"], sizes["n_cells"], dev)
                tr, tt = timed(lambda: ctx.trace_separatrices(codes, out=bufs), 2)
                kinds = torch.bincount(tr["kind"].long(), minlength=5).tolist()
                tms = float(np.median(tt))
                # CSR write floor: 8 B per cell + 8 B offset + 8 B origin + 8 B terminal + 1 B kind per branch
                csr_bytes = 8 * sizes["n_cells"] + 25 * sizes["n_branches"]
                trace = {"trace_ms": tms, "n_branches": sizes["n_branches"], "n_cells": sizes["n_cells"],
                         "desc": kinds[1], "asc": kinds[2], "conn": kinds[4],
                         "roofline": {"bound": "hbm", "achieved": csr_bytes / (tms * 1e-3) / 1e9, "peak": hbm,
                                      "unit": "GB/s", "frac": csr_bytes / (tms * 1e-3) / 1e9 / hbm,
                                      "note": "CSR output bytes only (write floor); the walks are latency-bound"}}
                if args.golden_parity:
                    from tests import digest as dg
                    csr_dig = {"n_branches": tr["origin"].shape[0], "n_cells": tr["cells"].shape[0],
                               "digests": {k: dg.digest_t(tr[k]) for k in ("offsets", "cells", "origin",
                                                                            "terminal", "kind")}}
                del tr
                for kname, kb in (("desc_ms", 1), ("asc_ms", 2), ("conn_ms", 4)):   # one kind per call
                    _, tk = timed(lambda: ctx.trace_separatrices(codes, kinds=kb, out=bufs), 1)
                    trace[kname] = tk[0]
                del bufs
            else:   # the CSR does not fit: trace the branches in groups of origin planes
                trace = chunked_trace(ctx, codes, dev, stream, 0.4 * free, sizes)
        except Exception as e:  # noqa: BLE001
            trace = {"error": str(e)[:200]}
        torch.cuda.empty_cache()

    # parity with the CPU oracle at the full size: the committed oracle goldens
    # (tests/golden/oracle_full_<C>.json, written by tools/oracle_goldens.py from oracle/ only)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", f"oracle_full_{cfg.name}.json")
    if args.golden_parity and shape is None and os.path.exists(gpath):
        from tests import digest as dg
        gold = json.load(open(gpath))
        parity = {"crop": list(f.shape), "source": os.path.relpath(gpath, ROOT),
                  "inputs": gold["input_sha256"] == {"f": hashlib.sha256(f.tobytes()).hexdigest(),
                                                     "fhat": hashlib.sha256(fh.tobytes()).hexdigest()},
                  "status": r.status == gold["status"],
                  "stats": all(r.stats[k] == gold["stats"][k] for k in ("rounds", "n_edited", "n_quantized",
                                                                         "n_lossless", "n_false_round0",
                                                                         "false_by_kind_round0")),
                  "g_bits": dg.digest_t(g.reshape(-1).view(torch.int32)) == gold["g_digest"],
                  "edits": dg.digest_t(r.edits.reshape(-1, 16).contiguous().view(torch.int64).reshape(-1))
                  == gold["edits_digest"],
                  "full_sweeps_equal": rfull.n_edits == r.n_edits and rfull.stats["rounds"] == r.stats["rounds"]}
        if csr_dig is not None:
            parity["csr"] = csr_dig == {k: gold["trace_g"][k] for k in ("n_branches", "n_cells", "digests")}
        parity["all"] = all(v for k, v in parity.items() if isinstance(v, bool))

    e2e = None
    if not args.no_e2e:
        fp = torch.from_numpy(f).pin_memory()
        fhp = torch.from_numpy(fh).pin_memory()
        gh = torch.empty(f.shape, dtype=torch.float32).pin_memory()
        eh = torch.empty((N, 16), dtype=torch.uint8).pin_memory()
        hb = dict(f=ft, fhat=fht, g=g, edits=edits)
        # the same metric end to end: dmtz_correct_host (full sweeps), pinned host f / fhat
        # in, g and the edit list back into pinned host memory, every copy inside the call
        r2, et = timed(lambda: ctx.correct_host(fp, fhp, xi, full_sweeps=True, bufs=hb, g_host=gh,
                                                edits_host=eh), 2)
        ems = float(np.median(et))
        r3, et3 = timed(lambda: ctx.correct_host(fp, fhp, xi, bufs=hb, g_host=gh, edits_host=eh), 2)
        e2e_raw = {"value": N * r2.stats["sweeps"] / (ems * 1e-3) / 1e6, "unit": "Mvoxels/s",
                   "h2d_bytes_per_step": 2 * 4 * N, "d2h_bytes_per_step": 4 * N + 16 * r2.n_edits,
                   "ms_per_step": ems,
                   "api": "dmtz_correct_host (full sweeps): pinned host f, fhat in; g + edit list to pinned host",
                   "time_to_fixed_point_ms": float(np.median(et3))}
        # the artifact end to end: host f / fhat in, the encoded edit stream out
        hbs = dict(hb, stream=torch.empty(max(int(dmtz._lib.dmtz_edit_stream_bound(N)), 1), dtype=torch.uint8,
                                          device=dev))
        sh = torch.empty(hbs["stream"].numel(), dtype=torch.uint8).pin_memory()
        (r4, sb), et4 = timed(lambda: ctx.correct_host_stream(fp, fhp, xi, full_sweeps=True, bufs=hbs,
                                                              stream_host=sh), 2)
        (r5, sb5), et5 = timed(lambda: ctx.correct_host_stream(fp, fhp, xi, bufs=hbs, stream_host=sh), 2)
        # the artifact decodes back to the same g
        try:   # the host bytes, back on the device, decode and apply to the converged g
            sd = sb.to(dev)
            de, dxi, dqm = ctx.decode_edits(sd, fhat=fht)
            ga = ctx.apply_edits(fht, dxi, de, dqm)
            dec_ok = bool(torch.equal(ga.view(torch.int32), hbs["g"].view(torch.int32)))
            del sd, de, ga
        except Exception as ex:   # noqa: BLE001
            dec_ok = f"not checked: {str(ex)[:80]}"
        e4 = float(np.median(et4))
        e2e = {"value": N * r4.stats["sweeps"] / (e4 * 1e-3) / 1e6, "unit": "Mvoxels/s",
               "h2d_bytes_per_step": 2 * 4 * N, "d2h_bytes_per_step": int(sb.numel()), "ms_per_step": e4,
               "api": "dmtz_correct_host_stream (full sweeps): pinned host f, fhat in; the edit list encoded on "
                      "the device (version 2), the stream to pinned host",
               "stream_decodes_to_g": dec_ok,
               "time_to_fixed_point_ms": float(np.median(et5))}

    cpu = None
    if not args.no_cpu_baseline:
        s = oracle_round(f, fh, xi)
        cpu = {"value": s["value"], "unit": "Mvoxels/s", "cores": s["threads"], "kind": "oracle",
               "sample": f"one oracle C-loop round on the whole {'x'.join(map(str, s['shape']))} field of "
                         f"{cfg.name} ({s['round_seconds']:.1f} s; literal gradient of g, classification, Eq. 2 "
                         f"edits; {s['n_false']} false cells, equal to the GPU's round-1 count: "
                         f"{s['n_false'] == r.stats['n_false_round0']})"}

    # the edit list as an artifact (NEXT-2): encode / decode / apply on the device
    codec = None
    try:
        ev = r.edits[:r.n_edits]
        (sb1, _) = (ctx.encode_edits(ev, xi, 6), None)
        sb, tenc = timed(lambda: ctx.encode_edits(ev, xi, 6, fhat=fht), 2)
        (dec, _, _), tdec = timed(lambda: ctx.decode_edits(sb, fhat=fht), 2)
        ga, tapp = timed(lambda: ctx.apply_edits(fht, xi, dec), 2)
        nbytes = int(sb.numel())
        t0p = time.perf_counter()
        packed = dmtz.pack_edit_stream(sb)
        pack_s = time.perf_counter() - t0p
        base = di.base_compressed_bytes(f, xi)
        ocr = {"original_bytes": 4 * N, "base_bytes": base["bytes"], "base_model": base["model"],
               "cr": 4 * N / base["bytes"], "edit_stream_bytes": nbytes, "edits_packed_bytes": len(packed),
               "edits_coder": "zlib level 1 over the edit stream (host)", "pack_seconds": pack_s,
               "ocr": 4 * N / (base["bytes"] + len(packed)), "edit_ratio": r.n_edits / N,
               "definition": "CR = original / base; OCR = original / (base + packed edits) (P:291)"}
        codec = {"ocr": ocr, "format": "version 2 (lossless values relative to fhat)", "v1_stream_bytes": int(sb1.numel()),
                 "n_edits": r.n_edits, "stream_bytes": nbytes, "bytes_per_edit": nbytes / max(r.n_edits, 1),
                 "edit_ratio": r.n_edits / N, "stream_fraction_of_original": nbytes / (4 * N),
                 "encode_ms": tenc[-1], "decode_ms": tdec[-1], "apply_ms": tapp[-1],
                 "apply_matches_g": bool(torch.equal(ga.view(torch.int32), g.view(torch.int32)))}
        del sb, sb1, dec, ga
    except Exception as e:  # noqa: BLE001
        codec = {"error": str(e)[:200]}

    sloop = None
    if args.sloop_config != "none":
        del ctx
        torch.cuda.empty_cache()
        sloop = {}
        for item in args.sloop_config.split(";"):
            name, tl = item.split(":")
            try:  # a failed extra line (e.g. out of memory next to C5's buffers) must not lose the main line
                sloop[name] = sloop_line(name, [int(t) for t in tl.split(",")], dev, stream, not args.no_cpu_baseline)
            except Exception as e:  # noqa: BLE001
                sloop[name] = {"error": str(e)[:200]}
                torch.cuda.empty_cache()

    st = r.stats
    line = {
        "metric": METRIC, "value": value, "unit": "Mvoxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, f.shape))} rel eps {cfg.eps}",
                   "step": "C-loop to its fixed point, every round a full sweep (full_sweeps=1)",
                   "value": "N x sweeps / step time = full-sweep round throughput (SURVEY §8(d-1))",
                   "xi": xi, "q_max": 6, "q_cap": 6, "tier": 2, "sweeps_per_step": sweeps,
                   "rounds": rfull.stats["rounds"],
                   "l2": (f"inputs larger than L2 (2 x {4 * N / 1e6:.0f} MB)" if 8 * N > 126e6
                          else f"inputs fit in L2 (2 x {4 * N / 1e6:.1f} MB), not flushed between steps"),
                   "parallelism": "1 GPU"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_raw": e2e_raw if not args.no_e2e else None,
        "gpu_launches": rfull.stats["launches"],
        "clocks": clk.summary(),
        "parity_vs_oracle": parity,
        "full_sweep_mvox_s": value,
        "time_to_fixed_point": frontier,
        "roofline_alu": roof_alu,
        "trace": trace,
        "stats": {k: st[k] for k in ("rounds", "sweeps", "n_edited", "n_quantized", "n_lossless", "n_false_round0",
                                     "false_by_kind_round0")},
        "codec": codec,
        "gen_seconds": t_gen,
    }
    detail = dict(line, sloop=sloop,
                  input_sha256={"f": hashlib.sha256(f.tobytes()).hexdigest(),
                                "fhat": hashlib.sha256(fh.tobytes()).hexdigest()})
    dpath = args.detail or (os.path.join(ROOT, "gpurun_out", "bench_detail.json")
                            if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else None)
    if dpath and rank == 0:
        with open(dpath, "w") as fh_:
            json.dump(detail, fh_, indent=1)
    if sloop is not None:   # compact summary in the line; the full per-tier dicts in the detail file
        line["sloop_ms"] = {n: {t: v.get("time_to_fixed_point_ms") for t, v in d.items() if t.startswith("tier")}
                            for n, d in sloop.items() if isinstance(d, dict)}
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
