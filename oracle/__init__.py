"""CPU oracle for the DMTz hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2409_17346_b200`` never imports it.  The numerics live in
``oracle/dmtz_oracle.c`` (plain C + OpenMP, literal definitions, see its header);
this module only marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dmtz_oracle.c")
_LIB = os.path.join(_HERE, "libdmtz_oracle.so")

OK, E_ARG, E_DIMS, E_NONFINITE, E_BOUND, E_CAPACITY, E_ITER_CAP, E_STUCK = range(8)
E_INTERNAL = 11
KIND_DESC, KIND_ASC, KIND_CONN = 1, 2, 4
BOUNDARY = np.uint64(0xFFFFFFFFFFFFFFFF)

EDIT_DTYPE = np.dtype([("v", "<u8"), ("q", "<u2"), ("lossless", "u1"), ("pad", "u1"),
                       ("value", "<f4")])
STATS_FIELDS = ["rounds", "n_edited", "n_quantized", "n_lossless", "n_false_round0"]


class _Stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("n_edited", ctypes.c_int64),
                ("n_quantized", ctypes.c_int64), ("n_lossless", ctypes.c_int64),
                ("n_false_round0", ctypes.c_int64),
                ("false_by_kind_round0", ctypes.c_int64 * 8),
                ("status", ctypes.c_int32), ("pad", ctypes.c_int32)]


class _SStats(ctypes.Structure):
    _fields_ = [("c_rounds", ctypes.c_int64), ("s_rounds", ctypes.c_int64),
                ("troublemakers", ctypes.c_int64), ("tm_by_kind", ctypes.c_int64 * 3),
                ("sep_branches", ctypes.c_int64), ("sep_cells", ctypes.c_int64),
                ("tm_round1", ctypes.c_int64), ("pad", ctypes.c_int64 * 7)]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, OpenMP, no FMA contraction, honoured rounding modes)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off",
                               "-frounding-math", "-fPIC", "-shared", "-Wall", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.dmtz_oracle_gradient.argtypes = [P, P, P, P]
        L.dmtz_oracle_complex_info.argtypes = [P, P, P, P, P, P]
        L.dmtz_oracle_cell_counts.argtypes = [P, P]
        L.dmtz_oracle_correct.argtypes = [P, P, P, ctypes.c_float, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, i64, P, P, P, i64, P,
                                          ctypes.POINTER(_Stats)]
        L.dmtz_oracle_correct_ex.argtypes = [P, P, P, ctypes.c_float, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_int32, i64, ctypes.c_int32, P, P, P, i64, P,
                                             ctypes.POINTER(_Stats), P, P, i64, P]
        L.dmtz_oracle_trace_digest.argtypes = [P, P, ctypes.c_uint32, P, P, P]
        L.dmtz_oracle_pairs_batch.argtypes = [P, i64, P, P, P, ctypes.c_int32]
        L.dmtz_oracle_preserve.argtypes = [P, P, P, ctypes.c_float, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32, i64, P, P, P, i64, P,
                                           ctypes.POINTER(_Stats), ctypes.POINTER(_SStats)]
        L.dmtz_oracle_persistence0.argtypes = [P, P, P, i64]
        L.dmtz_oracle_persistence0.restype = ctypes.c_int64
        L.dmtz_oracle_trace.argtypes = [P, P, ctypes.c_uint32, i64, i64, P, P, P, P, P, P, P]
        L.dmtz_oracle_slab_round.argtypes = [P, P, P, ctypes.c_float, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                             i64, i64, i64, i64, P, P, P, P]
        for fn in ("dmtz_oracle_gradient", "dmtz_oracle_complex_info", "dmtz_oracle_cell_counts",
                   "dmtz_oracle_correct", "dmtz_oracle_trace", "dmtz_oracle_num_threads", "dmtz_oracle_slab_round",
                   "dmtz_oracle_preserve", "dmtz_oracle_correct_ex", "dmtz_oracle_trace_digest",
                   "dmtz_oracle_pairs_batch"):
            getattr(L, fn).restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dims(shape) -> np.ndarray:
    """numpy shape (nz, ny, nx) or (ny, nx) -> int64[3] {nx, ny, nz}."""
    if len(shape) == 2:
        return np.array([shape[1], shape[0], 1], dtype=np.int64)
    return np.array([shape[2], shape[1], shape[0]], dtype=np.int64)


def num_threads() -> int:
    return lib().dmtz_oracle_num_threads()


def gradient(field: np.ndarray):
    """Literal discrete gradient of ``field`` -> (codes, crit masks) per anchor."""
    field = np.ascontiguousarray(field, dtype=np.float32)
    d = _dims(field.shape)
    n = field.size
    codes = np.zeros(n, dtype=np.uint64 if d[2] > 1 else np.uint16)
    crit = np.zeros(n, dtype=np.uint32)
    st = lib().dmtz_oracle_gradient(_p(d), _p(field), _p(codes), _p(crit))
    if st:
        raise RuntimeError(f"oracle gradient status {st}")
    return codes.reshape(field.shape), crit.reshape(field.shape)


def complex_info(shape):
    d = _dims(shape)
    T = ctypes.c_int32()
    dim = np.zeros(26, np.int32)
    nlink = np.zeros(26, np.int32)
    offs = np.zeros((26, 4, 3), np.int32)
    links = np.zeros((26, 14, 3), np.int32)
    lib().dmtz_oracle_complex_info(_p(d), ctypes.byref(T), _p(dim), _p(nlink), _p(offs), _p(links))
    t = T.value
    return dict(T=t, dim=dim[:t].copy(), nlink=nlink[:t].copy(), offsets=offs[:t].copy(),
                links=links[:t].copy())


def cell_counts(shape):
    d = _dims(shape)
    c = np.zeros(4, np.int64)
    st = lib().dmtz_oracle_cell_counts(_p(d), _p(c))
    if st:
        raise RuntimeError(f"oracle cell_counts status {st}")
    return c


def correct(f: np.ndarray, fhat: np.ndarray, xi: float, q_max: int = 6, q_cap: int | None = None,
            tier: int = 2, max_rounds: int = 0, edits_capacity: int | None = None,
            frontier: bool = False, round_log: bool = False, diag: bool = False):
    """Literal synchronous C-loop.  Returns dict(status, g, state, edits, stats).

    ``frontier``: after round 1 re-pair and classify only the cells anchored within
    [-2,1]^D of a target of the previous round (``dmtz_oracle_correct_ex``; equal to
    the full loop, tests/test_oracle_frontier.py).  ``round_log``: also return the
    number of false cells of every round (``false_per_round``).  ``diag``: also return
    ``diag`` = dict(targets_at_lb, r1, r2, r3a, r3b, targets) summed over the rounds."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    fhat = np.ascontiguousarray(fhat, dtype=np.float32)
    assert f.shape == fhat.shape
    if q_cap is None:
        q_cap = q_max
    d = _dims(f.shape)
    n = f.size
    cap = n if edits_capacity is None else edits_capacity
    g = np.empty_like(f)
    state = np.zeros(f.shape, dtype=np.uint32)
    edits = np.zeros(max(cap, 1), dtype=EDIT_DTYPE)
    ne = ctypes.c_int64()
    stats = _Stats()
    log_cap = 1 << 20 if round_log else 0
    log = np.full(max(log_cap, 1), -2, np.int64)
    sec = np.zeros(max(log_cap, 1), np.float64)
    dg = np.zeros(6, np.int64)
    st = lib().dmtz_oracle_correct_ex(_p(d), _p(f), _p(fhat), ctypes.c_float(xi), q_max, q_cap, tier,
                                      max_rounds, int(bool(frontier)), _p(g), _p(state), _p(edits), cap,
                                      ctypes.byref(ne), ctypes.byref(stats), _p(log), _p(sec), log_cap,
                                      _p(dg) if diag else None)
    out = {k: getattr(stats, k) for k in STATS_FIELDS}
    out["false_by_kind_round0"] = list(stats.false_by_kind_round0)
    out["status"] = st
    res = dict(status=st, g=g, state=state, edits=edits[:min(ne.value, cap)].copy(),
               n_edits=ne.value, stats=out)
    if diag:
        res["diag"] = dict(zip(("targets_at_lb", "r1", "r2", "r3a", "r3b", "targets"), (int(x) for x in dg)))
    if round_log:
        nr = int((log != -2).sum())
        res["false_per_round"] = [int(x) for x in log[:nr]]
        res["round_seconds"] = [float(x) for x in sec[:nr]]
    return res


def preserve(f: np.ndarray, fhat: np.ndarray, xi: float, tier: int = 4, q_max: int = 6,
             q_cap: int | None = None, max_rounds: int = 0, edits_capacity: int | None = None):
    """Literal alternating C-/S-loop workflow (tiers 1-5; 5 = pre-clamp + tier 4).  Returns dict(status, g, state,
    edits, stats) with stats also holding c_rounds, s_rounds, troublemakers, tm_by_kind,
    sep_branches, sep_cells, tm_round1."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    fhat = np.ascontiguousarray(fhat, dtype=np.float32)
    assert f.shape == fhat.shape
    if q_cap is None:
        q_cap = q_max
    d = _dims(f.shape)
    n = f.size
    cap = n if edits_capacity is None else edits_capacity
    g = np.empty_like(f)
    state = np.zeros(f.shape, dtype=np.uint32)
    edits = np.zeros(max(cap, 1), dtype=EDIT_DTYPE)
    ne = ctypes.c_int64()
    stats, ss = _Stats(), _SStats()
    st = lib().dmtz_oracle_preserve(_p(d), _p(f), _p(fhat), ctypes.c_float(xi), q_max, q_cap, tier,
                                    max_rounds, _p(g), _p(state), _p(edits), cap,
                                    ctypes.byref(ne), ctypes.byref(stats), ctypes.byref(ss))
    out = {k: getattr(stats, k) for k in STATS_FIELDS}
    out["false_by_kind_round0"] = list(stats.false_by_kind_round0)
    out["status"] = st
    for k in ("c_rounds", "s_rounds", "troublemakers", "sep_branches", "sep_cells", "tm_round1"):
        out[k] = getattr(ss, k)
    out["tm_by_kind"] = list(ss.tm_by_kind)
    return dict(status=st, g=g, state=state, edits=edits[:min(ne.value, cap)].copy(),
                n_edits=ne.value, stats=out)


def persistence0(field: np.ndarray) -> np.ndarray:
    """0-dim sublevel persistence pairs (birth vertex, death vertex), union-find + elder rule."""
    field = np.ascontiguousarray(field, dtype=np.float32)
    d = _dims(field.shape)
    n = lib().dmtz_oracle_persistence0(_p(d), _p(field), None, 0)
    out = np.zeros((max(n, 1), 2), np.int64)
    lib().dmtz_oracle_persistence0(_p(d), _p(field), _p(out), n)
    return out[:n]


def trace(field: np.ndarray, kinds: int = KIND_DESC | KIND_ASC | KIND_CONN,
          cap_branches: int | None = None, cap_cells: int | None = None):
    """Literal V-path traces of the gradient of ``field`` (CSR)."""
    field = np.ascontiguousarray(field, dtype=np.float32)
    d = _dims(field.shape)
    L = lib()

    def run(cb, cc):
        off = np.zeros(cb + 1, np.int64)
        cells = np.zeros(max(cc, 1), np.uint64)
        origin = np.zeros(max(cb, 1), np.uint64)
        term = np.zeros(max(cb, 1), np.uint64)
        kind = np.zeros(max(cb, 1), np.uint8)
        nb, nc = ctypes.c_int64(), ctypes.c_int64()
        st = L.dmtz_oracle_trace(_p(d), _p(field), kinds, cb, cc, _p(off), _p(cells), _p(origin),
                                 _p(term), _p(kind), ctypes.byref(nb), ctypes.byref(nc))
        return st, nb.value, nc.value, off, cells, origin, term, kind

    cb = cap_branches if cap_branches is not None else 1024
    cc = cap_cells if cap_cells is not None else 65536
    st, nb, nc, off, cells, origin, term, kind = run(cb, cc)
    if st == E_CAPACITY and cap_branches is None and cap_cells is None:
        st, nb, nc, off, cells, origin, term, kind = run(nb, nc)
    if st not in (OK,):
        raise RuntimeError(f"oracle trace status {st}")
    return dict(offsets=off[:nb + 1], cells=cells[:nc], origin=origin[:nb], terminal=term[:nb],
                kind=kind[:nb])


def trace_digest(field: np.ndarray, kinds: int = KIND_DESC | KIND_ASC | KIND_CONN):
    """The literal trace of ``field`` without storing it: (n_branches, n_cells, digests)
    with digests = {offsets, cells, origin, terminal, kind} as defined in tests/digest.py."""
    field = np.ascontiguousarray(field, dtype=np.float32)
    d = _dims(field.shape)
    dig = np.zeros(5, np.uint64)
    nb, nc = ctypes.c_int64(), ctypes.c_int64()
    st = lib().dmtz_oracle_trace_digest(_p(d), _p(field), kinds, _p(dig), ctypes.byref(nb), ctypes.byref(nc))
    if st:
        raise RuntimeError(f"oracle trace_digest status {st}")
    names = ("offsets", "cells", "origin", "terminal", "kind")
    return nb.value, nc.value, {k: int(v) for k, v in zip(names, dig)}


def pairs_batch(fields: np.ndarray, cap: int = 48):
    """Literal gradient pairs of many fields on one tiny grid (fields: (nf, *shape)).
    Returns (pairs uint32 (nf, cap), count int32 (nf)); a pair is (cell mask << 16) |
    (cofacet mask), vertex-id bitmasks, sorted per field."""
    fields = np.ascontiguousarray(fields, dtype=np.float32)
    d = _dims(fields.shape[1:])
    nf = fields.shape[0]
    out = np.zeros((nf, cap), np.uint32)
    cnt = np.zeros(nf, np.int32)
    st = lib().dmtz_oracle_pairs_batch(_p(d), nf, _p(fields), _p(out), _p(cnt), cap)
    if st:
        raise RuntimeError(f"oracle pairs_batch status {st}")
    return out, cnt


def slab_round(f, fhat, xi, g, state, anchor_planes, owned_planes, q_max=6, q_cap=None, tier=2):
    """One literal C-loop round on a z-slab (local arrays incl. halos; g, state updated
    in place).  Returns (n_false, n_changed, n_targets, kinds[8])."""
    f = np.ascontiguousarray(f, dtype=np.float32)
    fhat = np.ascontiguousarray(fhat, dtype=np.float32)
    assert g.dtype == np.float32 and g.flags.c_contiguous and state.dtype == np.uint32
    d = _dims(f.shape)
    out = np.zeros(3, np.int64)
    kinds = np.zeros(8, np.int64)
    st = lib().dmtz_oracle_slab_round(_p(d), _p(f), _p(fhat), ctypes.c_float(xi), q_max,
                                      q_max if q_cap is None else q_cap, tier, anchor_planes[0],
                                      anchor_planes[1], owned_planes[0], owned_planes[1], _p(g), _p(state),
                                      _p(out), _p(kinds))
    if st:
        raise RuntimeError(f"oracle slab_round status {st}")
    return int(out[0]), int(out[1]), int(out[2]), kinds
