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
        f and fhat, the C-loop, D2H of g and the edit list, every step
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


def oracle_sample(f, fh, xi, edge):
    """Time the oracle (as it stands) on a bounded crop of the workload."""
    import oracle
    oracle.build()
    crop = tuple(slice(0, min(edge, s)) for s in f.shape)
    fc, fhc = np.ascontiguousarray(f[crop]), np.ascontiguousarray(fh[crop])
    t0 = time.perf_counter()
    r = oracle.correct(fc, fhc, xi)
    dt = time.perf_counter() - t0
    sweeps = r["stats"]["rounds"] + 1
    return dict(value=fc.size * sweeps / dt / 1e6, seconds=dt, sweeps=sweeps, shape=list(fc.shape),
                rounds=r["stats"]["rounds"], threads=oracle.num_threads(), ref=r, fc=fc, fhc=fhc)


def run_reference(args, cfg, f, fh, xi):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    vals = []
    for i in range(args.warmup + args.steps):
        s = oracle_sample(f, fh, xi, args.ref_edge)
        if i >= args.warmup:
            vals.append(s)
    v = float(np.median([s["value"] for s in vals]))
    sample = (f"oracle C-loop to its fixed point on the {vals[0]['shape']} crop of {cfg.name} "
              f"({vals[0]['sweeps']} sweeps, {vals[0]['seconds']:.1f} s each)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Mvoxels/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.median([s["seconds"] for s in vals]) * 1e3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, cfg.shape))} rel eps {cfg.eps}",
                       "crop": vals[0]["shape"], "parallelism": "host cores (OpenMP)"},
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dmtz", choices=["dmtz", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--shape", default=None, help="override the config shape, e.g. 128,128,128")
    ap.add_argument("--ref-edge", type=int, default=96, help="oracle crop edge for the CPU baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
        from paper_2409_17346_b200 import slab
        return slab.bench_main(args, f, fh, xi, cfg, world, rank, local, clocks_cls=Clocks)

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

    for _ in range(args.warmup):
        r = step()
    torch.cuda.synchronize()
    times, stats = [], []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            stats.append(r.stats)
        # the reference (full-recompute) mode: every code recomputed in every round
        fr_t = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rfull = step(full=True)
            e1.record(stream)
            torch.cuda.synchronize()
            fr_t.append(e0.elapsed_time(e1))
        # once more with per-kernel CUDA events (host-driven rounds) for the roofline
        rp = step(full=True, profile=True)
        rpd = step(profile=True)   # default mode, per-kernel events
    assert rfull.n_edits == r.n_edits and rfull.stats["rounds"] == r.stats["rounds"]
    ms = float(np.median(times))
    sweeps = int(np.median([s["sweeps"] for s in stats]))
    value = N * sweeps / (ms * 1e-3) / 1e6
    fr_ms = float(np.median(fr_t))
    full_recompute = {"value": N * rfull.stats["sweeps"] / (fr_ms * 1e-3) / 1e6, "unit": "Mvoxels/s",
                      "ms_per_step": fr_ms, "t_round_full_ms": fr_ms / rfull.stats["sweeps"],
                      "mode": "full_sweeps=1: every code recomputed, every anchor classified"}

    # roofline of the dominant kernel of the default step (live CUDA events on the launching stream,
    # one extra host-driven step): k_decode; k_screen's on the rounds that recompute every code
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs") or 6650.0
    sm_mhz = peaks.get("sm_max_mhz") or 1965.0
    alu_peak = 148 * 64 * sm_mhz * 1e6 / 1e9          # Gop/s: 148 SMs x 4 SMSP x 16-lane ALU pipe
    workload = f"{cfg.name} {'x'.join(map(str, f.shape))}"
    ds = rpd.stats
    dec_ops = DECODE_OPS_PER_ANCHOR[D] * ds["anchors_decoded"] + RULE_OPS_PER_CELL * ds["cells_evaluated"]
    dec_s = ds["decode_ms"] * 1e-3
    dec_ach = dec_ops / dec_s / 1e9
    roof = {"bound": "alu", "achieved": dec_ach, "peak": alu_peak, "unit": "Gop/s", "frac": dec_ach / alu_peak,
            "traffic": _ncu_traffic("k_decode", workload),
            "ncu_issue": _ncu_issue("k_decode", workload),
            "kernel": "k_decode (criticality of g, critical-cell diff, target rules; default step)",
            "decode_ms_per_step": ds["decode_ms"], "screen_ms_per_step": ds["screen_ms"],
            "share_of_step": ds["decode_ms"] / ms, "launches_per_step": ds["sweeps"],
            "anchors_decoded": ds["anchors_decoded"], "cells_evaluated": ds["cells_evaluated"],
            "anchors_replayed": ds["anchors_replayed"],
            "ops_per_decoded_anchor": DECODE_OPS_PER_ANCHOR[D], "ops_per_false_cell": RULE_OPS_PER_CELL,
            "peak_source": "ALU: 148 SMs x 64 lanes/clk x MEASURED_PEAKS sm_max_mhz (DESIGN.md section 7)",
            "traffic_note": "ncu dram bytes per launch, mean over one step's launches (profiles/ncu_summary.json)"}
    ps = rp.stats
    t_launch = ps["screen_ms_full"] / max(ps["n_screen_full"], 1) * 1e-3
    alu_achieved = ALU_OPS_PER_ANCHOR[D] * N / t_launch / 1e9
    gbs = BYTES_PER_ANCHOR[D] * N / t_launch / 1e9
    roof_screen = {"bound": "alu", "achieved": alu_achieved, "peak": alu_peak, "unit": "Gop/s",
                   "frac": alu_achieved / alu_peak, "traffic": _ncu_traffic("k_screen", workload),
                   "ncu_issue": _ncu_issue("k_screen", workload),
                   "kernel": "k_screen (gradient codes of g, a launch that recomputes every anchor)",
                   "launch_ms": t_launch * 1e3, "alu_ops_per_anchor": ALU_OPS_PER_ANCHOR[D],
                   "bytes_per_anchor": BYTES_PER_ANCHOR[D], "hbm_achieved_gbs": gbs, "hbm_peak_gbs": hbm,
                   "hbm_frac": gbs / hbm, "screen_ms_per_step": ds["screen_ms"],
                   "share_of_step": ds["screen_ms"] / ms}

    # the north star's per-iteration HBM fraction: 12 B/voxel (g + cand_f) per sweep over the whole step
    hbm_iter = {"algorithmic_bytes_per_voxel_sweep": BYTES_PER_ANCHOR[D],
                "achieved_gbs": BYTES_PER_ANCHOR[D] * N * sweeps / (ms * 1e-3) / 1e9, "peak_gbs": hbm,
                "frac": BYTES_PER_ANCHOR[D] * N * sweeps / (ms * 1e-3) / 1e9 / hbm,
                "full_sweep_round_frac": BYTES_PER_ANCHOR[D] * N / (fr_ms / rfull.stats["sweeps"] * 1e-3) / 1e9 / hbm,
                "note": "the path is ALU-bound (DESIGN.md section 7): 105 SoS compares per anchor per code"}
    # time-to-fixed-point (the second half of BASELINE's metric): the timed default step
    frontier = {"time_to_fixed_point_ms": ms, "rounds": r.stats["rounds"], "sweeps": r.stats["sweeps"],
                "anchors_classified": r.stats["anchors_swept"], "codes_recomputed": r.stats["anchors_recomputed"],
                "full_sweep_equivalents": r.stats["anchors_recomputed"] / N}

    # traces of the converged field (a9-a11), once
    trace = None
    if not args.no_trace:
        codes = ctx.compute_gradient(g)
        try:
            sizes = ctx.trace_sizes(codes)
            need = sizes["n_branches"] * 33 + sizes["n_cells"] * 8
            free = torch.cuda.mem_get_info()[0]
            if need < 0.8 * free:
                bufs = ctx.trace_buffers(sizes["n_branches"], sizes["n_cells"], dev)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                tr = ctx.trace_separatrices(codes, out=bufs)
                e1.record(stream)
                torch.cuda.synchronize()
                kinds = torch.bincount(tr["kind"].long(), minlength=5).tolist()
                trace = {"trace_ms": e0.elapsed_time(e1), "n_branches": sizes["n_branches"],
                         "n_cells": sizes["n_cells"], "desc": kinds[1], "asc": kinds[2], "conn": kinds[4]}
                del tr
                for kname, kb in (("desc_ms", 1), ("asc_ms", 2), ("conn_ms", 4)):   # one kind per call
                    torch.cuda.synchronize()
                    e0.record(stream)
                    ctx.trace_separatrices(codes, kinds=kb, out=bufs)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    trace[kname] = e0.elapsed_time(e1)
                del bufs
            else:   # the CSR does not fit: trace the branches in groups of origin planes
                trace = chunked_trace(ctx, codes, dev, stream, 0.4 * free, sizes)
        except Exception as e:  # noqa: BLE001
            trace = {"error": str(e)[:200]}
        torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        fp = torch.from_numpy(f).pin_memory()
        fhp = torch.from_numpy(fh).pin_memory()
        gh = torch.empty(f.shape, dtype=torch.float32).pin_memory()
        eh = torch.empty((N, 16), dtype=torch.uint8).pin_memory()
        hb = dict(f=ft, fhat=fht, g=g, edits=edits)
        et = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r2 = ctx.correct_host(fp, fhp, xi, bufs=hb, g_host=gh, edits_host=eh)   # copies inside the C call
            e1.record(stream)
            torch.cuda.synchronize()
            et.append(e0.elapsed_time(e1))
        ems = float(np.median(et))
        e2e = {"value": N * r2.stats["sweeps"] / (ems * 1e-3) / 1e6, "unit": "Mvoxels/s",
               "h2d_bytes_per_step": 2 * 4 * N, "d2h_bytes_per_step": 4 * N + 16 * r2.n_edits, "ms_per_step": ems,
               "api": "dmtz_correct_host: pinned host f, fhat in; g and the edit list back to pinned host"}
        # variant: the compressor-side artifact only -- the encoded edit stream comes back
        # (the decompressor rebuilds g from fhat + stream, dmtz_apply_edits)
        sh = torch.empty(int(dmtz.lib().dmtz_edit_stream_bound(N)), dtype=torch.uint8).pin_memory()
        et2 = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ft.copy_(fp, non_blocking=True)
            fht.copy_(fhp, non_blocking=True)
            r3 = step()
            sb = ctx.encode_edits(edits[:r3.n_edits], xi, 6, fhat=fht)
            sh[:sb.numel()].copy_(sb, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            et2.append(e0.elapsed_time(e1))
        ems2 = float(np.median(et2))
        e2e["stream_variant"] = {"value": N * r3.stats["sweeps"] / (ems2 * 1e-3) / 1e6, "unit": "Mvoxels/s",
                                 "h2d_bytes_per_step": 2 * 4 * N, "d2h_bytes_per_step": int(sb.numel()),
                                 "ms_per_step": ems2, "result": "encoded edit stream (dmtz_encode_edits)"}
        del sb

    cpu = None
    parity = None
    if not args.no_cpu_baseline:
        s = oracle_sample(f, fh, xi, args.ref_edge)
        cpu = {"value": s["value"], "unit": "Mvoxels/s", "cores": s["threads"], "kind": "oracle",
               "sample": f"oracle C-loop to its fixed point on the {s['shape']} crop of {cfg.name} "
                         f"({s['sweeps']} sweeps in {s['seconds']:.1f} s)"}
        # parity on the same crop: the CUDA path against the oracle, bit for bit
        import oracle
        ref, fc, fhc = s["ref"], s["fc"], s["fhc"]
        fct, fhct = torch.from_numpy(fc).to(dev), torch.from_numpy(fhc).to(dev)
        rc = dmtz.correct(fct, fhct, xi)
        oc, om = oracle.gradient(fc)
        gc = dmtz.compute_gradient(fct)
        e = rc.edits_numpy()
        tr_o = oracle.trace(ref["g"])
        tr_g = dmtz.trace_separatrices(dmtz.compute_gradient(rc.g))
        parity = {"crop": s["shape"],
                  "codes": bool(np.array_equal(gc.cpu().numpy().view(oc.dtype), oc)),
                  "crit": bool(np.array_equal(dmtz.critical_mask(gc).cpu().numpy().view(np.uint32), om)),
                  "g_bits": bool(np.array_equal(rc.g.cpu().numpy().view(np.uint32), ref["g"].view(np.uint32))),
                  "edits": bool(np.array_equal(e["v"], ref["edits"]["v"]) and np.array_equal(e["q"], ref["edits"]["q"])),
                  "rounds": rc.stats["rounds"] == ref["stats"]["rounds"],
                  "csr": all(bool(np.array_equal(tr_g[k].cpu().numpy().view(tr_o[k].dtype), tr_o[k])) for k in tr_o)}

    # the edit list as an artifact (NEXT-2): encode / decode / apply on the device
    codec = None
    try:
        ev = r.edits[:r.n_edits]
        def _t(fn):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return out, e0.elapsed_time(e1)
        sb1 = ctx.encode_edits(ev, xi, 6)
        sb, enc_ms = _t(lambda: ctx.encode_edits(ev, xi, 6, fhat=fht))
        (dec, _, _), dec_ms = _t(lambda: ctx.decode_edits(sb, fhat=fht))
        ga, app_ms = _t(lambda: ctx.apply_edits(fht, xi, dec))
        nbytes = int(sb.numel())
        codec = {"format": "version 2 (lossless values relative to fhat)", "v1_stream_bytes": int(sb1.numel()),
                 "n_edits": r.n_edits, "stream_bytes": nbytes, "bytes_per_edit": nbytes / max(r.n_edits, 1),
                 "keyvalue_float_bytes": 12 * r.n_edits, "edit_ratio": r.n_edits / N,
                 "stream_fraction_of_original": nbytes / (4 * N),
                 "encode_ms": enc_ms, "decode_ms": dec_ms, "apply_ms": app_ms,
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
                   "xi": xi, "q_max": 6, "q_cap": 6, "tier": 2, "sweeps_per_step": sweeps, "rounds": st["rounds"],
                   "mode": "default: dirty frontier + exact change skipping (bit-identical to full_sweeps=1)",
                   "l2": (f"inputs larger than L2 (2 x {4 * N / 1e6:.0f} MB)" if 8 * N > 126e6
                          else f"inputs fit in L2 (2 x {4 * N / 1e6:.1f} MB), not flushed between steps"), "parallelism": "1 GPU"},
        "roofline": roof, "roofline_screen": roof_screen, "hbm_per_iteration": hbm_iter, "cpu_baseline": cpu, "e2e": e2e, "time_to_fixed_point": frontier,
        "full_recompute": full_recompute, "trace": trace, "sloop": sloop, "codec": codec,
        "gpu_launches": st["launches"],
        "clocks": clk.summary(),
        "stats": {k: st[k] for k in ("rounds", "sweeps", "n_edited", "n_quantized", "n_lossless", "n_false_round0",
                                     "false_by_kind_round0")},
        "gen_seconds": t_gen,
        "parity_vs_oracle": parity,
        "input_sha256": {"f": hashlib.sha256(f.tobytes()).hexdigest(), "fhat": hashlib.sha256(fh.tobytes()).hexdigest()},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
