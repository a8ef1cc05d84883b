"""Multi-GPU C-loop: z-slab decomposition driven over torch.distributed.

Each rank owns a contiguous range of z-planes and every edit decision there.
Its LOCAL grid is the owned planes plus up to HALO = 3 planes below and above:
a target lies within [-1, 2]^3 of its false cell's anchor, so the cells whose
targets can be owned vertices are anchored in [z0 - 2, z1 + 1), and their
criticality reads values in [z0 - 3, z1 + 3).  Per round each rank

  1. refreshes its halo planes of g from the neighbours (send/recv of contiguous
     planes: NCCL over NVLink on GPUs, gloo on CPU),
  2. runs one round (dmtz_slab_round: screen, classify the anchored cells,
     edit the owned targets),
  3. all-reduces the round counters, so every rank takes the same stop decision.

The rounds are exactly those of dmtz_correct on the global grid (edits are
set-synchronous and read only round-start values), hence the concatenated
owned edit lists equal the single-GPU edit list bit for bit.

The driver is generic over an *engine* (the per-rank round kernels): the CUDA
engine below, or a test engine.  ``run_emulated`` steps several engines in one
process with in-memory halo copies (one GPU standing in for several, strictly
sequentially -- no rank ever waits on another inside a kernel).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

HALO = 3
OK, E_ITER_CAP, E_STUCK, E_INTERNAL = 0, 6, 7, 11


@dataclass(frozen=True)
class SlabPlan:
    rank: int
    world: int
    nz: int
    z0: int          # owned global planes [z0, z1)
    z1: int
    lz0: int         # global planes of the local grid [lz0, lz1)
    lz1: int

    @property
    def own_local(self):
        return self.z0 - self.lz0, self.z1 - self.lz0

    @property
    def anchor_local(self):
        a0 = max(0, self.z0 - 2)
        a1 = min(self.nz, self.z1 + 1)
        return a0 - self.lz0, a1 - self.lz0

    @property
    def halo_below(self):   # local planes received from rank - 1
        return 0, self.z0 - self.lz0

    @property
    def halo_above(self):   # local planes received from rank + 1
        return self.z1 - self.lz0, self.lz1 - self.lz0


def partition(nz: int, world: int):
    """Balanced contiguous z-ranges; every rank owns at least HALO planes."""
    if world * HALO > nz:
        raise ValueError(f"{world} ranks need nz >= {world * HALO} (got {nz})")
    base, extra = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((z, z + n))
        z += n
    return out


def plan(nz: int, world: int, rank: int) -> SlabPlan:
    z0, z1 = partition(nz, world)[rank]
    return SlabPlan(rank, world, nz, z0, z1, max(0, z0 - HALO), min(nz, z1 + HALO))


def halo_pairs(p: SlabPlan):
    """[(peer, send local planes (a, b), recv local planes (c, d))] of this rank."""
    out = []
    if p.rank > 0:
        lo = p.halo_below
        out.append((p.rank - 1, (p.z0 - p.lz0, p.z0 - p.lz0 + (lo[1] - lo[0])), lo))
    if p.rank < p.world - 1:
        hi = p.halo_above
        n = hi[1] - hi[0]
        out.append((p.rank + 1, (p.z1 - p.lz0 - n, p.z1 - p.lz0), hi))
    return out


class _Slab(ctypes.Structure):
    _fields_ = [("z_offset", ctypes.c_int64), ("own_z0", ctypes.c_int64), ("own_z1", ctypes.c_int64),
                ("anchor_z0", ctypes.c_int64), ("anchor_z1", ctypes.c_int64)]


class CudaSlabEngine:
    """The rank's round kernels: libdmtz slab entry points on its local grid."""

    def __init__(self, p: SlabPlan, ny: int, nx: int, device):
        from . import Context, _Opts, _check, _lib, _stream_ptr
        self._lib, self._check, self._Opts, self._stream_ptr = _lib, _check, _Opts, _stream_ptr
        self.p = p
        self.shape = (p.lz1 - p.lz0, ny, nx)
        self.ctx = Context(self.shape, device)
        o0, o1 = p.own_local
        a0, a1 = p.anchor_local
        self.slab = _Slab(p.lz0, o0, o1, a0, a1)
        self.device = torch.device(device)
        self.launches = 0   # kernels launched by the library calls below (fixed per call)

    def _P(self, t):
        return ctypes.c_void_p(t.data_ptr())

    def begin(self, f, fhat, xi, q_max=6, q_cap=None, tier=2):
        self.f, self.fhat = f.contiguous(), fhat.contiguous()
        self.g = torch.empty_like(self.f)
        self.opts = self._Opts(float(xi), int(q_max), int(q_max if q_cap is None else q_cap), int(tier), 0, 1, 0)
        self._check(self._lib.dmtz_slab_begin(self.ctx._h, self._P(self.f), self._P(self.fhat),
                                              ctypes.byref(self.opts), ctypes.byref(self.slab),
                                              self._P(self.ctx.workspace), self.ctx.ws_bytes, self._P(self.g),
                                              self._stream_ptr()))
        self.launches += 5   # k_setup, k_codes, k_critmask, k_lowpos, k_units_all

    def round(self, r: int):
        c = (ctypes.c_int64 * 4)()
        k = (ctypes.c_int64 * 8)()
        self._check(self._lib.dmtz_slab_round(self.ctx._h, self._P(self.f), self._P(self.fhat),
                                              ctypes.byref(self.opts), ctypes.byref(self.slab),
                                              self._P(self.ctx.workspace), self.ctx.ws_bytes, self._P(self.g), r,
                                              ctypes.cast(c, ctypes.c_void_p), ctypes.cast(k, ctypes.c_void_p),
                                              self._stream_ptr()))
        self.launches += 5 + (r > 1)  # set_round, [units_from_bits], screen, decode, edit_rows, loop_check
        return np.array(c[:], np.int64), np.array(k[:], np.int64)

    def round_async(self, r: int) -> torch.Tensor:
        """The round with its 12 counters left on the device (no host synchronisation)."""
        out = torch.empty(12, dtype=torch.int64, device=self.device)
        self._check(self._lib.dmtz_slab_round_async(self.ctx._h, self._P(self.f), self._P(self.fhat),
                                                    ctypes.byref(self.opts), ctypes.byref(self.slab),
                                                    self._P(self.ctx.workspace), self.ctx.ws_bytes, self._P(self.g),
                                                    r, self._P(out), self._stream_ptr()))
        self.launches += 6 + (r > 1)  # set_round, [units_from_bits], screen, decode, edit_rows, loop_check, counters
        return out

    def halo(self, r: int, a: int, b: int, planes):
        """Local planes [a, b) of g <- `planes` (the neighbour's values after round r);
        the library records the changed vertices for round r + 1's screen and frontier."""
        planes = planes.contiguous()
        self._check(self._lib.dmtz_slab_halo(self.ctx._h, ctypes.byref(self.slab), self._P(self.ctx.workspace),
                                             self.ctx.ws_bytes, self._P(self.g), self._P(planes), a, b, r,
                                             self._stream_ptr()))
        self.launches += 1 if b > a else 0

    def end(self):
        o0, o1 = self.p.own_local
        cap = (o1 - o0) * self.shape[1] * self.shape[2]
        edits = torch.empty((max(cap, 1), 16), dtype=torch.uint8, device=self.device)
        ne, nl = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.dmtz_slab_end(self.ctx._h, ctypes.byref(self.slab), self._P(self.ctx.workspace),
                                            self.ctx.ws_bytes, self._P(self.g), self._P(edits), cap,
                                            ctypes.byref(ne), ctypes.byref(nl), self._stream_ptr()))
        self.launches += 3   # edit count, scan, write
        return edits[:ne.value], nl.value

    def owned_g(self):
        o0, o1 = self.p.own_local
        return self.g[o0:o1]


def _stop(round_, tot, max_rounds):
    """Same stop rule as dmtz_correct on the summed counters."""
    if tot[3]:
        return E_INTERNAL
    if tot[0] == 0:
        return OK
    if tot[1] == 0:
        return E_STUCK
    if round_ == max_rounds:
        return E_ITER_CAP
    return None


def run_distributed(engine, f, fhat, xi, q_max=6, q_cap=None, tier=2, max_rounds=0, group=None):
    """One rank of the slab C-loop over torch.distributed (call on every rank).

    Pipelined by one round: round r's kernels, its halo exchange and its counter
    all-reduce are all enqueued on the device before the host looks at round r - 1's
    summed counters, so the host's stop decision never idles the GPU.  The one round
    run past the stop is a no-op: after the fixed point (F empty) or STUCK (no target
    can move) a round edits nothing, and no round is enqueued past max_rounds."""
    import torch.distributed as dist
    p = engine.p
    engine.begin(f, fhat, xi, q_max, q_cap, tier)
    pairs = halo_pairs(p)
    stats = dict(rounds=0, n_false_round0=0, false_by_kind_round0=[0] * 8)
    status = None
    pending = None   # (round, host counters, event) of the last enqueued round
    r = 0
    while status is None:
        if not (max_rounds and r >= max_rounds):
            r += 1
            if r > 1 and pairs:
                ops, bufs = [], []
                for peer, (sa, sb), (ra, rb) in pairs:
                    buf = torch.empty_like(engine.g[ra:rb])
                    bufs.append((ra, rb, buf))
                    ops.append(dist.P2POp(dist.isend, engine.g[sa:sb].contiguous(), peer, group))
                    ops.append(dist.P2POp(dist.irecv, buf, peer, group))
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
                for ra, rb, buf in bufs:   # apply + record the changed halo vertices
                    engine.halo(r - 1, ra, rb, buf)
            if hasattr(engine, "round_async"):
                tot = engine.round_async(r)
            else:
                c, k = engine.round(r)
                tot = torch.tensor(np.concatenate([c, k]), dtype=torch.int64, device=engine.g.device)
            dist.all_reduce(tot, group=group)
            if tot.is_cuda:
                host = torch.empty(12, dtype=torch.int64).pin_memory()
                host.copy_(tot, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
            else:
                host, ev = tot, None
            nxt = (r, host, ev)
        else:
            nxt = None          # max_rounds reached: only the decision on the last round is left
        if pending is not None:
            pr, host_p, ev_p = pending
            if ev_p is not None:
                ev_p.synchronize()
            t = host_p.numpy()
            if pr == 1:
                stats["n_false_round0"] = int(t[0])
                stats["false_by_kind_round0"] = [int(x) for x in t[4:12]]
            status = _stop(pr, t, max_rounds)
            if status != OK:     # rounds that found false cells
                stats["rounds"] = pr
        pending = nxt
        if pending is None and status is None:   # cannot happen: the cap round decides
            status = E_ITER_CAP
    if pending is not None and pending[2] is not None:
        pending[2].synchronize()
    edits, nl = engine.end()
    stats["status"] = status
    return edits, nl, stats


def run_emulated(engines, fs, fhats, xi, q_max=6, q_cap=None, tier=2, max_rounds=0):
    """All ranks in one process (one device or CPU): sequential rounds, in-memory halos."""
    for e, f, fh in zip(engines, fs, fhats):
        e.begin(f, fh, xi, q_max, q_cap, tier)
    stats = dict(rounds=0, n_false_round0=0, false_by_kind_round0=[0] * 8)
    status = None
    r = 0
    while status is None:
        r += 1
        if r > 1:
            for e in engines:
                for peer, (sa, sb), (ra, rb) in halo_pairs(e.p):
                    src = engines[peer]
                    # the peer's planes that this rank keeps as halo = peer's send range towards us
                    (_, (psa, psb), _) = [x for x in halo_pairs(src.p) if x[0] == e.p.rank][0]
                    e.halo(r - 1, ra, rb, src.g[psa:psb].clone())
        tot = np.zeros(12, np.int64)
        for e in engines:
            c, k = e.round(r)
            tot += np.concatenate([c, k])
        if r == 1:
            stats["n_false_round0"] = int(tot[0])
            stats["false_by_kind_round0"] = [int(x) for x in tot[4:12]]
        status = _stop(r, tot, max_rounds)
        if status != OK:
            stats["rounds"] = r
    outs = [e.end() for e in engines]
    stats["status"] = status
    return outs, stats


# ----------------------------------------------------------------------------- traces
# The traces do not shard along z without exchanging path segments (a V-path or a
# connector BFS can cross any number of slabs).  Instead the gradient is replicated:
# every rank computes the codes of its owned planes (its local grid holds the 1-plane
# stencil halo they need), the codes are all-gathered (C4: 1.07 GB, C5: 8.6 GB -- a
# small fraction of 180 GB of HBM), and each rank traces the branches whose origin
# cell is anchored in its owned planes (dmtz_trace_separatrices_range).  Per kind,
# the ranks' branches in rank order are exactly the one-GPU output.

def gather_planes(owned: torch.Tensor, nz: int, world: int, group=None) -> torch.Tensor:
    """All-gather the ranks' owned planes (partition(nz, world)) into the full array
    (uneven slabs: padded to the largest, then trimmed)."""
    import torch.distributed as dist
    parts = partition(nz, world)
    mx = max(b - a for a, b in parts)
    plane = tuple(owned.shape[1:])
    pad = torch.zeros((mx,) + plane, dtype=owned.dtype, device=owned.device)
    pad[:owned.shape[0]] = owned
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[r][:b - a] for r, (a, b) in enumerate(parts)], dim=0)


def owned_codes(engine) -> torch.Tensor:
    """Gradient codes of the rank's owned planes, from its local g (owned + halos)."""
    codes = engine.ctx.compute_gradient(engine.g)
    o0, o1 = engine.p.own_local
    return codes[o0:o1]


def trace_distributed(engine, kinds=7, group=None, ctx=None):
    """One rank of the multi-GPU trace after run_distributed: returns (its CSR dict,
    the global Context used).  Kinds are DESC | ASC | CONN bits."""
    from . import Context
    p = engine.p
    full = gather_planes(owned_codes(engine), p.nz, p.world, group)
    ctx = ctx or Context(tuple(full.shape), engine.device)
    return ctx.trace_separatrices(full, kinds, z_range=(p.z0, p.z1)), ctx


def local_inputs(f: np.ndarray, fhat: np.ndarray, p: SlabPlan):
    """The rank's local arrays (owned planes + halos) of global inputs."""
    return (np.ascontiguousarray(f[p.lz0:p.lz1]), np.ascontiguousarray(fhat[p.lz0:p.lz1]))


def bench_main(args, f, fh, xi, cfg, world, rank, local, clocks_cls=None):
    """bench.py --gpus N (torchrun): strong scaling of the slab C-loop on the config.
    Device time of a step = max over ranks (CUDA events, barrier + sync on both sides)."""
    import json

    import torch.distributed as dist
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    p = plan(f.shape[0], world, rank)
    lf, lfh = local_inputs(f, fh, p)
    eng = CudaSlabEngine(p, f.shape[1], f.shape[2], dev)
    ft, fht = torch.from_numpy(lf).to(dev), torch.from_numpy(lfh).to(dev)
    for _ in range(args.warmup):
        run_distributed(eng, ft, fht, xi)
    torch.cuda.synchronize()
    dist.barrier()

    def timed(fn):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    times = []
    clk = clocks_cls(local) if clocks_cls else None
    if clk:
        clk.__enter__()
    l0 = eng.launches
    for _ in range(args.steps):
        t, (edits, nl, st) = timed(lambda: run_distributed(eng, ft, fht, xi))
        times.append(t)
    launches = (eng.launches - l0) // max(args.steps, 1)
    if clk:
        clk.__exit__()
    ms = float(np.median(times))
    sweeps = st["rounds"] + 1
    value = f.size * sweeps / (ms * 1e-3) / 1e6
    # end to end: this rank's inputs from pinned host memory, its owned g and edit list back
    fp, fhp = torch.from_numpy(lf).pin_memory(), torch.from_numpy(lfh).pin_memory()
    o0, o1 = p.own_local
    gh = torch.empty((o1 - o0,) + tuple(f.shape[1:]), dtype=torch.float32).pin_memory()
    eh = torch.empty((max(gh.numel(), 1), 16), dtype=torch.uint8).pin_memory()

    def e2e_step():
        ft.copy_(fp, non_blocking=True)
        fht.copy_(fhp, non_blocking=True)
        e, n, s = run_distributed(eng, ft, fht, xi)
        gh.copy_(eng.owned_g(), non_blocking=True)
        eh[:e.shape[0]].copy_(e, non_blocking=True)
        torch.cuda.synchronize()
        return e.numel()
    ems, ebytes = timed(e2e_step)
    # traces of the converged field: codes all-gathered, branches split by origin plane
    trace = None
    if not getattr(args, "no_trace", False):
        try:
            from . import Context
            full = gather_planes(owned_codes(eng), p.nz, world)
            tctx = Context(tuple(full.shape), dev)
            zr = (p.z0, p.z1)
            sz = tctx.trace_sizes(full, 7, z_range=zr)
            bufs = tctx.trace_buffers(sz["n_branches"], sz["n_cells"], dev)
            del full

            def tr_step():   # gradient of the owned planes, all-gather, this rank's branches
                fc = gather_planes(owned_codes(eng), p.nz, world)
                return tctx.trace_separatrices(fc, 7, out=bufs, z_range=zr)
            tr_step()
            tms, tr = timed(tr_step)
            nbr = torch.tensor([tr["origin"].shape[0], tr["cells"].shape[0]], device=dev, dtype=torch.int64)
            dist.all_reduce(nbr)
            trace = {"trace_ms": tms, "n_branches": int(nbr[0].item()), "n_cells": int(nbr[1].item()),
                     "mode": "owned-plane codes all-gathered, branches split by origin plane (max over ranks)"}
            del tr, bufs
        except Exception as ex:  # noqa: BLE001
            trace = {"error": str(ex)[:200]}
    d2h = torch.tensor([gh.numel() * 4 + ebytes], device=dev, dtype=torch.int64)
    h2d = torch.tensor([lf.nbytes + lfh.nbytes], device=dev, dtype=torch.int64)
    dist.all_reduce(d2h)
    dist.all_reduce(h2d)
    if rank == 0:
        line = {"metric": "C-loop Mvoxels/s per iteration", "value": value, "unit": "Mvoxels/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"{cfg.name} {cfg.family} {'x'.join(map(str, f.shape))} rel eps {cfg.eps}",
                           "parallelism": f"z-slabs x{world} (NCCL halo send/recv + counter all-reduce per round)",
                           "sweeps_per_step": sweeps, "rounds": st["rounds"],
                           "mode": "frontier + exact change skipping per slab (bit-identical to 1 GPU)",
                           "l2": "inputs larger than L2"},
                "roofline": None, "roofline_note": "kernel rooflines: the N=1 line (same kernels per slab)",
                "cpu_baseline": None,
                "e2e": {"value": f.size * sweeps / (ems * 1e-3) / 1e6, "unit": "Mvoxels/s", "ms_per_step": ems,
                        "h2d_bytes_per_step": int(h2d.item()),
                        "d2h_bytes_per_step": int(d2h.item())},
                "trace": trace, "gpu_launches": launches, "clocks": clk.summary() if clk else None,
                "stats": st}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
