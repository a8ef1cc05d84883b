"""Exhaustive-order pins of the oracle's gradient ("exhaustive over
all orders of 3x3 and 2x2x2 grids"): the oracle's literal pairing equals an independent
C brute force (tests/bf_orders.c: explicit Kuhn complex as vertex bitmasks, the rule of
P:84-92 / P:152-155 read literally) on

* every one of the 8! = 40320 value orders of a 2x2x2 grid and the 9! = 362880 of a
  3x3 grid (distinct values), and
* every tie pattern with values in {0..3} on 2x2x2 (4^8 = 65536 fields) and in {0..2}
  on 3x3 (3^9 = 19683), where the SoS tie-break by vertex index decides.

The pairs are compared as (cell, partner) vertex bitmasks, so neither side's cell
numbering is involved."""
import ctypes
import itertools
import os
import subprocess

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "bf_orders.c")
LIB = os.path.join(HERE, "libbf_orders.so")


def _bf():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-o", LIB, SRC])
    L = ctypes.CDLL(LIB)
    L.bf_pairs.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
    L.bf_pairs.restype = ctypes.c_int
    return L


def _compare(fields):
    shape = fields.shape[1:]
    nx, ny, nz = (shape[1], shape[0], 1) if len(shape) == 2 else (shape[2], shape[1], shape[0])
    cap = 48
    out = np.zeros((fields.shape[0], cap), np.uint32)
    cnt = np.zeros(fields.shape[0], np.int32)
    fl = np.ascontiguousarray(fields, np.float32)
    assert _bf().bf_pairs(nx, ny, nz, fl.shape[0], fl.ctypes.data, out.ctypes.data, cnt.ctypes.data, cap) == 0
    o_out, o_cnt = oracle.pairs_batch(fl, cap)
    assert np.array_equal(cnt, o_cnt)
    assert np.array_equal(out, o_out)
    return cnt


def _all_perms(n):
    return np.array(list(itertools.permutations(range(n))), dtype=np.float32)


def test_all_orders_2x2x2():
    f = _all_perms(8).reshape(-1, 2, 2, 2)
    cnt = _compare(f)
    assert f.shape[0] == 40320
    # 19 edges + 18 triangles + 6 tets + 8 vertices; chi = 1: #crit >= 1, pairs <= 25
    assert cnt.min() >= 1 and cnt.max() <= 25


def test_all_orders_3x3():
    f = _all_perms(9).reshape(-1, 3, 3)
    cnt = _compare(f)
    assert f.shape[0] == 362880 and cnt.max() <= 16


def _all_tie_patterns(nv, k):
    g = np.indices((k,) * nv).reshape(nv, -1).T
    return g.astype(np.float32)


def test_all_tie_patterns_2x2x2():
    _compare(_all_tie_patterns(8, 4).reshape(-1, 2, 2, 2))


def test_all_tie_patterns_3x3():
    _compare(_all_tie_patterns(9, 3).reshape(-1, 3, 3))


def test_bruteforce_is_not_vacuous():
    """A transposed operand in the key comparison would change pairs: the brute force
    and the oracle disagree with a deliberately reversed order (f -> -f)."""
    f = _all_perms(8)[:200].reshape(-1, 2, 2, 2)
    a, _ = oracle.pairs_batch(f)
    b, _ = oracle.pairs_batch(-f)
    assert not np.array_equal(a, b)
