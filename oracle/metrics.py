"""Evaluation metrics of §5.1, plain Python -- TEST INFRASTRUCTURE ONLY.

critical_prf: a cell is "retained" when it is critical in both fields (same anchor and
type: the same bit of the per-anchor critical mask).  separatrix_prf: the unit is one
branch, identified by (kind, origin cell, ordinal among its origin's branches); it is
retained when the other trace holds that branch with the same terminal and cell
sequence.  Recall = matches / original, precision = matches / reconstructed (1 when the
denominator is 0).  Shares no code with the CUDA kernels (csrc/dmtz_metrics.cuh)."""
from __future__ import annotations

import numpy as np


def _ratio(m, d):
    return m / d if d else 1.0


def critical_prf(crit_orig: np.ndarray, crit_rec: np.ndarray) -> dict:
    a = np.unpackbits(np.ascontiguousarray(crit_orig, np.uint32).ravel().view(np.uint8))
    b = np.unpackbits(np.ascontiguousarray(crit_rec, np.uint32).ravel().view(np.uint8))
    na, nb, nm = int(a.sum()), int(b.sum()), int((a & b).sum())
    return dict(n_orig=na, n_rec=nb, n_match=nm, recall=_ratio(nm, na), precision=_ratio(nm, nb))


def _branches(tr):
    off, cells = np.asarray(tr["offsets"]), np.asarray(tr["cells"]).view(np.uint64)
    origin, term, kind = (np.asarray(tr[k]) for k in ("origin", "terminal", "kind"))
    seen, out = {}, {}
    for b in range(len(origin)):
        key0 = (int(kind[b]), int(origin[b].view(np.uint64)) if origin.dtype != np.uint64 else int(origin[b]))
        ordinal = seen.get(key0, 0)
        seen[key0] = ordinal + 1
        t = int(term[b].view(np.uint64)) if term.dtype != np.uint64 else int(term[b])
        out[key0 + (ordinal,)] = (t, tuple(int(c) for c in cells[off[b]:off[b + 1]]))
    return out


def separatrix_prf(tr_orig: dict, tr_rec: dict) -> dict:
    a, b = _branches(tr_orig), _branches(tr_rec)
    nm = sum(1 for k, v in a.items() if b.get(k) == v)
    return dict(n_orig=len(a), n_rec=len(b), n_match=nm, recall=_ratio(nm, len(a)), precision=_ratio(nm, len(b)))
