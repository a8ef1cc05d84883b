"""Explicit-complex brute force (pure Python, tiny inputs) -- pins for the oracle.

Shares no code with ``oracle/`` or the CUDA path.  The complex is built a
different way from the oracle's: every unit cube (square) is cut into the
D! Kuhn simplices  b, b+e_p1, b+e_p1+e_p2, ...  (one per axis permutation p),
and the complex is the set of all faces of those simplices.  Cells are
frozensets of integer coordinate triples; facets and cofacets are set operations.

The gradient is Eq. 1 + the pairing rule read directly off the paper
(P:84-92): keys are the cell's (value, index) pairs sorted
descending; P_a = {b in cofacets(a) : b minus its lowest vertex == a};
a is paired with min-key(P_a) unless already paired with a facet.
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np


class Complex:
    def __init__(self, nx, ny, nz=1, pad=0):
        """Grid complex; ``pad`` > 0 builds it on a grid enlarged by ``pad`` on every
        side (coordinates shifted) so that interior links of boundary cells exist."""
        self.n = (nx, ny, nz)
        self.D = 2 if nz == 1 else 3
        self.pad = pad
        D = self.D
        lo = -pad
        hx, hy = nx + pad, ny + pad
        hz = nz + pad if D == 3 else 1
        zlo = lo if D == 3 else 0
        self.verts = [(x, y, z) for z in range(zlo, hz) for y in range(lo, hy) for x in range(lo, hx)]
        maximal = set()
        for z in range(zlo, hz - (1 if D == 3 else 0)):
            for y in range(lo, hy - 1):
                for x in range(lo, hx - 1):
                    for perm in itertools.permutations(range(D)):
                        p = [x, y, z]
                        simp = [tuple(p)]
                        for ax in perm:
                            p[ax] += 1
                            simp.append(tuple(p))
                        maximal.add(frozenset(simp))
        cells = set()
        for s in maximal:
            for r in range(1, len(s) + 1):
                for sub in itertools.combinations(sorted(s), r):
                    cells.add(frozenset(sub))
        self.cells = cells
        self.by_dim = {d: sorted((c for c in cells if len(c) == d + 1), key=sorted) for d in range(D + 1)}
        self.cofacets = {c: [] for c in cells}
        for c in cells:
            if len(c) > 1:
                for v in c:
                    self.cofacets[c - {v}].append(c)

    def vid(self, p):
        nx, ny, _ = self.n
        return p[0] + nx * (p[1] + ny * p[2])

    def inside(self, p):
        return all(0 <= p[a] < self.n[a] for a in range(3))


def sos_key(f, p, C):
    return (float(f[C.vid(p)]), C.vid(p))


def cell_key(f, cell, C):
    """Eq. 1 as a lexicographic key: vertices sorted descending by (value, index)."""
    return sorted((sos_key(f, p, C) for p in cell), reverse=True)


def gradient(C: Complex, f):
    """Literal pairing.  Returns dict cell -> partner cell (both directions)."""
    fl = np.asarray(f, dtype=np.float32).ravel()
    pair = {}
    for d in range(C.D):
        for a in C.by_dim[d]:
            if a in pair:
                continue
            P = []
            for b in C.cofacets[a]:
                kb = sorted(b, key=lambda p: sos_key(fl, p, C), reverse=True)
                if frozenset(kb[:-1]) == a:          # G0(b) == a
                    P.append(b)
            if P:
                b = min(P, key=lambda c: cell_key(fl, c, C))
                pair[a] = b
                pair[b] = a
    return pair


def critical(C: Complex, pair):
    return {c for c in C.cells if c not in pair}


def ru32(x: Fraction) -> np.float32:
    """Smallest float32 >= x (exact)."""
    c = np.float32(float(x))
    while Fraction(float(c)) < x:
        c = np.nextafter(c, np.float32(np.inf), dtype=np.float32)
    while True:
        p = np.nextafter(c, np.float32(-np.inf), dtype=np.float32)
        if Fraction(float(p)) >= x:
            c = p
        else:
            return c


def c_loop(C: Complex, f, fhat, xi, q_max=6, q_cap=None, tier=2, max_rounds=100000):
    """Synchronous C-loop with the target rules R1/R2/R3a/R3b,
    written independently of the oracle.  Returns (status, g, q, lossless, stats)."""
    if q_cap is None:
        q_cap = q_max
    f = np.asarray(f, np.float32).ravel()
    fhat = np.asarray(fhat, np.float32).ravel()
    xi32 = np.float32(xi)
    step = np.float32(float(Fraction(float(xi32)) / 2 ** q_max))
    assert Fraction(float(step)) == Fraction(float(xi32)) / 2 ** q_max
    lb = np.array([ru32(Fraction(float(v)) - Fraction(float(xi32))) for v in f], np.float32)
    g = fhat.copy()
    q = np.zeros(f.size, np.int64)
    lossless = np.zeros(f.size, bool)
    pf = gradient(C, f)
    cf = critical(C, pf)
    top = C.D
    stats = dict(rounds=0, n_false_round0=0, kinds=[0] * 8)
    rnd = 0
    while True:
        rnd += 1
        pg = gradient(C, g)
        cg = critical(C, pg)
        F = cf ^ cg
        if tier == 1:
            F = {c for c in F if len(c) - 1 in (0, top)}
        if rnd == 1:
            stats["n_false_round0"] = len(F)
            for a in F:
                d = len(a) - 1
                cls = 3 if d == top else d
                stats["kinds"][2 * cls + (1 if a in cf else 0)] += 1
        if not F:
            return "OK", g, q, lossless, stats
        stats["rounds"] = rnd
        T = set()
        for a in F:
            lowest_f = min(a, key=lambda p: sos_key(f, p, C))
            if a in cg:       # FP: critical in g, paired in f  -> R1
                b = pf[a]
                big, small = (b, a) if len(b) > len(a) else (a, b)
                (v,) = big - small
            elif len(pg[a]) > len(a):   # FN, paired up in g -> R2
                v = lowest_f
            else:                       # FN, paired down in g with gamma -> R3
                gamma = pg[a]
                (y,) = a - gamma
                if lowest_f != y:
                    v = lowest_f
                else:
                    (v,) = pf[gamma] - gamma
            T.add(C.vid(v))
        changed = False
        for v in sorted(T):
            if lossless[v]:
                continue
            changed = True
            if q[v] + 1 <= q_cap:
                gp = np.float32(fhat[v] - np.float32(np.float32(q[v] + 1) * step))
                if gp >= lb[v]:
                    q[v] += 1
                    g[v] = gp
                    continue
            g[v] = lb[v]
            lossless[v] = True
        if not changed:
            return "STUCK", g, q, lossless, stats
        if rnd == max_rounds:
            return "ITER_CAP", g, q, lossless, stats


def trace(C: Complex, f, interleaved: bool = False):
    """Descending / ascending / connector traces, returned as python lists of
    (kind, origin, [cells...], terminal) with cells as frozensets.  Connectors:
    cells = the visited triangles in BFS order, terminal = the reached 1-saddles in
    order; with ``interleaved`` cells = the single event log instead -- for each
    dequeued triangle, its facet edges in facet order (the facet omitting the k-th
    vertex by index), a critical edge logged as reached, a new triangle logged when
    it is enqueued."""
    fl = np.asarray(f, np.float32).ravel()
    pair = gradient(C, fl)
    crit = critical(C, pair)
    top = C.D
    out = []

    def order(cells):
        # origin cells ordered by (anchor index, type) is checked by the caller; here by vid tuple
        return sorted(cells, key=lambda c: sorted(C.vid(p) for p in c))

    for e in order(c for c in crit if len(c) == 2):
        for v in sorted(e, key=C.vid):
            cells = [frozenset([v])]
            cur = frozenset([v])
            while cur in pair:
                edge = pair[cur]
                assert len(edge) == 2
                (w,) = edge - cur
                cells += [edge, frozenset([w])]
                cur = frozenset([w])
            out.append(("desc", e, cells, cur))
    for c in order(c for c in crit if len(c) == top):
        for t in sorted(C.cofacets[c], key=lambda t: C.vid(next(iter(t - c)))):
            cells = [t]
            term = None
            while True:
                if t in crit:
                    term = t
                    break
                cc = pair[t]
                cells.append(cc)
                others = [x for x in C.cofacets[cc] if x != t]
                if not others:
                    term = "BOUNDARY"
                    break
                t = others[0]
                cells.append(t)
            out.append(("asc", c, cells, term))
    if C.D == 3:
        for s in order(c for c in crit if len(c) == 3):
            reached, visited, events = [], [s], []
            seen = {s}
            qi = 0
            while qi < len(visited):
                t = visited[qi]
                qi += 1
                for e in (t - {p} for p in sorted(t, key=C.vid)):
                    if e in crit:
                        reached.append(e)
                        events.append(e)
                    elif len(pair[e]) == 3 and pair[e] != t and pair[e] not in seen:
                        seen.add(pair[e])
                        visited.append(pair[e])
                        events.append(pair[e])
            out.append(("conn", s, events if interleaved else visited[1:], reached))
    return out


def cs_loop(C: Complex, f, fhat, xi, q_max=6, q_cap=None, tier=4, max_rounds=100000):
    """Alternating C-/S-loop in synchronous rounds, written
    independently of the oracle: a round with false critical cells is a C-round
    (rules R1-R3b); otherwise (tier >= 3) every separatrix of f is re-checked in the
    gradient of g (tier 4: all; tier 3: those whose end differs in g's trace) and its
    troublemaker -- the first cell along it whose partner differs -- has the vertex of
    its original partner that it does not share decreased.
    Returns (status, g, q, lossless, stats)."""
    if q_cap is None:
        q_cap = q_max
    f = np.asarray(f, np.float32).ravel()
    fhat = np.asarray(fhat, np.float32).ravel()
    xi32 = np.float32(xi)
    step = np.float32(float(Fraction(float(xi32)) / 2 ** q_max))
    lb = np.array([ru32(Fraction(float(v)) - Fraction(float(xi32))) for v in f], np.float32)
    g = fhat.copy()
    q = np.zeros(f.size, np.int64)
    lossless = np.zeros(f.size, bool)
    pf = gradient(C, f)
    cf = critical(C, pf)
    if tier == 5:   # every vertex of every critical cell of f to its lower bound, losslessly
        for c in cf:
            for p in c:
                v = C.vid(p)
                g[v] = lb[v]
                lossless[v] = True
        tier = 4
    sep_f = trace(C, f) if tier >= 3 else []
    stats = dict(c_rounds=0, s_rounds=0, troublemakers=0)

    def partner_vertex(a):
        b = pf[a]
        big, small = (b, a) if len(b) > len(a) else (a, b)
        (v,) = big - small
        return v

    def first_differing(kind, origin, cells, pg):
        if kind == "desc":
            seq = cells[0:-1:2]
        elif kind == "asc":
            seq = cells[1::2]
        else:
            seq = [e for t in [origin] + cells for e in (t - {p} for p in sorted(t, key=C.vid))
                   if e not in cf]
        for a in seq:
            if pf.get(a) != pg.get(a):
                return a
        return None

    rnd = 0
    while True:
        rnd += 1
        pg = gradient(C, g)
        cg = critical(C, pg)
        F = cf ^ cg
        T = set()
        if F:
            stats["c_rounds"] += 1
            for a in F:
                lowest_f = min(a, key=lambda p: sos_key(f, p, C))
                if a in cg:
                    v = partner_vertex(a)
                elif len(pg[a]) > len(a):
                    v = lowest_f
                else:
                    gamma = pg[a]
                    (y,) = a - gamma
                    if lowest_f != y:
                        v = lowest_f
                    else:
                        (v,) = pf[gamma] - gamma
                T.add(C.vid(v))
        elif tier >= 3:
            sep_g = trace(C, g) if tier == 3 else None
            n = 0
            for b, (kind, origin, cells, term) in enumerate(sep_f):
                if tier == 3:
                    kg, og, cg_, tg = sep_g[b]
                    assert (kg, og) == (kind, origin)
                    same = (sorted(map(sorted, tg)) == sorted(map(sorted, term))) if kind == "conn" else tg == term
                    if same:
                        continue
                a = first_differing(kind, origin, cells, pg)
                if a is None:
                    continue
                n += 1
                T.add(C.vid(partner_vertex(a)))
            if not T:
                return "OK", g, q, lossless, stats
            stats["s_rounds"] += 1
            stats["troublemakers"] += n
        else:
            return "OK", g, q, lossless, stats
        changed = False
        for v in sorted(T):
            if lossless[v]:
                continue
            changed = True
            if q[v] + 1 <= q_cap:
                gp = np.float32(fhat[v] - np.float32(np.float32(q[v] + 1) * step))
                if gp >= lb[v]:
                    q[v] += 1
                    g[v] = gp
                    continue
            g[v] = lb[v]
            lossless[v] = True
        if not changed:
            return "STUCK", g, q, lossless, stats
        if rnd == max_rounds:
            return "ITER_CAP", g, q, lossless, stats


def persistence0(C: Complex, f):
    """0-dim sublevel persistence pairs (birth vertex, death vertex) from scratch: add the
    vertices in SoS order, recompute the components of the induced subgraph each time;
    when v merges components, all but the eldest (earliest-born) die at v."""
    fl = np.asarray(f, np.float32).ravel()
    verts = sorted((c for c in C.by_dim[0]), key=lambda c: sos_key(fl, next(iter(c)), C))
    nbrs = {}
    for e in C.by_dim[1]:
        a, b = tuple(e)
        nbrs.setdefault(a, []).append(b)
        nbrs.setdefault(b, []).append(a)
    rank = {}
    comps_prev = {}
    pairs = []
    present = set()
    for i, c in enumerate(verts):
        (p,) = tuple(c)
        rank[p] = i
        present.add(p)
        # components containing p's present neighbours, before p was added
        roots = {comps_prev[q] for q in nbrs.get(p, []) if q in present and q != p}
        if len(roots) > 1:
            eldest = min(roots, key=lambda r: rank[r])
            pairs += [(C.vid(r), C.vid(p)) for r in roots if r != eldest]
        # recompute components (labels = eldest vertex) from scratch
        comps_prev = {}
        seen = set()
        for s0 in present:
            if s0 in seen:
                continue
            stack, comp = [s0], []
            seen.add(s0)
            while stack:
                x = stack.pop()
                comp.append(x)
                for y in nbrs.get(x, []):
                    if y in present and y not in seen:
                        seen.add(y)
                        stack.append(y)
            root = min(comp, key=lambda r: rank[r])
            for x in comp:
                comps_prev[x] = root
    return sorted(pairs)
