/*
 * oracle/dmtz_oracle.c -- plain, slow, literal CPU oracle for the DMTz hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2409_17346_b200/) never links, imports or calls it, and this file
 * includes no header and shares no table, helper or constant generator with the
 * CUDA path.  It re-derives everything it needs from the definitions in
 * PAPER.md (cited as P:<line>) and the readings listed in DESIGN.md section 3.
 *
 * What it computes (each function cites its passage):
 *   - the Freudenthal/Kuhn cell complex of a regular grid
 *   - the discrete gradient by the Shivashankar-Natarajan rule on the
 *     extended function of Eq. 1, LITERALLY: for every
 *     d-cell a (d ascending, cells already paired with a facet skipped) it forms
 *     P_a = { b cofacet of a : G0(b) = a } by sorting b's vertices and dropping
 *     the lowest, and pairs a with the lexicographically smallest key in P_a
 *   - critical cells (unpaired cells)
 *   - the C-loop in synchronous rounds with the
 *     quantized edit of Eq. 2, error bound P:138
 *   - V-path traces: descending, ascending, saddle-saddle connectors
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py against
 * brute force on an explicit complex, closed-form counts, the Euler relation and
 * the paper's worked example (Fig. 3).  Round counts / edit counts on
 * synthetic data have no external pin ("parity unpinned").
 *
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -frounding-math -fPIC -shared
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* fesetround() is honoured because the file is compiled with -frounding-math. */

/* Status values: the numeric codes the C-ABI documents (include/dmtz.h is NOT
 * included; the oracle restates the documented numbers). */
enum {
  OR_OK = 0, OR_E_ARG = 1, OR_E_DIMS = 2, OR_E_NONFINITE = 3, OR_E_BOUND = 4,
  OR_E_CAPACITY = 5, OR_E_ITER_CAP = 6, OR_E_STUCK = 7, OR_E_INTERNAL = 11
};

#define MAXTYPES 26
#define MAXLINK 14
#define BOUNDARY_ID UINT64_MAX

/* ------------------------------------------------------------------------- */
/* The cell complex ("regular grid-based triangulation").        */
/* ------------------------------------------------------------------------- */

typedef struct {
  int dim;              /* number of vertices - 1 */
  int nv;
  int off[4][3];        /* vertex offsets from the anchor, ascending global index */
  int nlink;            /* interior link size (grid assumed unbounded) */
  int link[MAXLINK][3]; /* link vertex offsets, ascending (dz,dy,dx) = slot order */
  int cof_anchor[MAXLINK][3]; /* cofacet cell (cell + link[s]) : its anchor delta */
  int cof_type[MAXLINK];      /*                                   its type      */
  int cof_pos[MAXLINK];       /* position of link[s] inside the cofacet's vertex list */
  int fac_anchor[4][3]; /* facet omitting vertex k : anchor delta */
  int fac_type[4];      /*                           type         */
} ctype_t;

typedef struct {
  int D;                 /* 2 or 3 */
  int64_t n[3];          /* nx, ny, nz (nz == 1 for 2D) */
  int64_t N;             /* vertex count */
  int T;                 /* cell types per anchor */
  int top;               /* top dimension */
  int first_of_dim[5];   /* first type index of each dimension, [dim+1] = end */
  ctype_t t[MAXTYPES];
} cx_t;

static void mask_off(int m, int o[3]) { o[0] = m & 1; o[1] = (m >> 1) & 1; o[2] = (m >> 2) & 1; }

/* A set of lattice points is a simplex of the Kuhn/Freudenthal triangulation
 * iff all points lie in one unit cube above their componentwise minimum and
 * their offsets from it are totally ordered componentwise (a chain from the
 * cube's low corner towards the main diagonal) -- S:47-48, "split on the
 * (lowest-corner -> opposite-corner) diagonal". */
static int is_simplex(int np, int p[][3]) {
  int b[3] = {p[0][0], p[0][1], p[0][2]};
  for (int i = 1; i < np; i++)
    for (int a = 0; a < 3; a++) if (p[i][a] < b[a]) b[a] = p[i][a];
  for (int i = 0; i < np; i++) {
    for (int a = 0; a < 3; a++) { int d = p[i][a] - b[a]; if (d < 0 || d > 1) return 0; }
    for (int j = i + 1; j < np; j++) {
      int le = 1, ge = 1, eq = 1;
      for (int a = 0; a < 3; a++) {
        if (p[i][a] > p[j][a]) le = 0;
        if (p[i][a] < p[j][a]) ge = 0;
        if (p[i][a] != p[j][a]) eq = 0;
      }
      if (eq || (!le && !ge)) return 0;
    }
  }
  return 1;
}

/* (dz,dy,dx) lexicographic order of offsets == ascending global index order */
static int off_less(const int a[3], const int b[3]) {
  if (a[2] != b[2]) return a[2] < b[2];
  if (a[1] != b[1]) return a[1] < b[1];
  return a[0] < b[0];
}

/* Find the (anchor, type) of the cell whose vertex set is pts[0..np) */
static int locate(const cx_t* cx, int np, int pts[][3], int anchor[3], int* pos_of_last) {
  int b[3] = {pts[0][0], pts[0][1], pts[0][2]};
  for (int i = 1; i < np; i++)
    for (int a = 0; a < 3; a++) if (pts[i][a] < b[a]) b[a] = pts[i][a];
  for (int ti = 0; ti < cx->T; ti++) {
    const ctype_t* c = &cx->t[ti];
    if (c->nv != np) continue;
    int all = 1, lastpos = -1;
    for (int i = 0; i < np && all; i++) {
      int found = 0;
      for (int k = 0; k < np; k++)
        if (c->off[k][0] == pts[i][0] - b[0] && c->off[k][1] == pts[i][1] - b[1] &&
            c->off[k][2] == pts[i][2] - b[2]) { found = 1; if (i == np - 1) lastpos = k; }
      all = found;
    }
    if (all) { anchor[0] = b[0]; anchor[1] = b[1]; anchor[2] = b[2]; if (pos_of_last) *pos_of_last = lastpos; return ti; }
  }
  return -1;
}

/* Enumerate the cell types anchored at a vertex: chains 0 = m0 < m1 < ... < md of
 * nested bit masks in {0,1}^D, dims ascending, each dim in lexicographic order of
 * the mask tuple (the type numbering documented in include/dmtz.h, restated). */
static void build_complex(cx_t* cx, int64_t nx, int64_t ny, int64_t nz) {
  memset(cx, 0, sizeof *cx);
  cx->n[0] = nx; cx->n[1] = ny; cx->n[2] = nz;
  cx->N = nx * ny * nz;
  cx->D = (nz == 1) ? 2 : 3;
  cx->top = cx->D;
  int full = (1 << cx->D) - 1;
  int T = 0;
  for (int d = 0; d <= cx->D; d++) {
    cx->first_of_dim[d] = T;
    /* enumerate d-chains by brute force over all mask tuples, lexicographically */
    int m[4] = {0, 0, 0, 0};
    int total = 1;
    for (int i = 0; i < d; i++) total *= (full + 1);
    for (int code = 0; code < total; code++) {
      int c = code, ok = 1;
      /* most significant digit first -> lexicographic order */
      for (int i = d - 1; i >= 0; i--) { m[i] = c % (full + 1); c /= (full + 1); }
      for (int i = 0; i < d && ok; i++) {
        if (m[i] == 0) ok = 0;
        if (i > 0 && !((m[i - 1] & ~m[i]) == 0 && m[i - 1] != m[i])) ok = 0;
      }
      if (!ok) continue;
      ctype_t* ct = &cx->t[T++];
      ct->dim = d; ct->nv = d + 1;
      ct->off[0][0] = ct->off[0][1] = ct->off[0][2] = 0;
      for (int i = 0; i < d; i++) mask_off(m[i], ct->off[i + 1]);
    }
  }
  cx->first_of_dim[cx->D + 1] = T;
  cx->T = T;
  /* links, cofacets and facets, by brute force over nearby lattice points */
  for (int ti = 0; ti < T; ti++) {
    ctype_t* ct = &cx->t[ti];
    int zlo = (cx->D == 3) ? -1 : 0, zhi = (cx->D == 3) ? 2 : 0;
    for (int z = zlo; z <= zhi; z++)
      for (int y = -1; y <= 2; y++)
        for (int x = -1; x <= 2; x++) {
          int w[3] = {x, y, z}, pts[5][3], dup = 0;
          for (int k = 0; k < ct->nv; k++) {
            memcpy(pts[k], ct->off[k], sizeof pts[k]);
            if (!memcmp(ct->off[k], w, sizeof w)) dup = 1;
          }
          if (dup) continue;
          memcpy(pts[ct->nv], w, sizeof w);
          if (!is_simplex(ct->nv + 1, pts)) continue;
          /* insertion into slot order */
          int s = ct->nlink++;
          while (s > 0 && off_less(w, ct->link[s - 1])) { memcpy(ct->link[s], ct->link[s - 1], sizeof w); s--; }
          memcpy(ct->link[s], w, sizeof w);
        }
    for (int s = 0; s < ct->nlink; s++) {
      int pts[5][3];
      for (int k = 0; k < ct->nv; k++) memcpy(pts[k], ct->off[k], sizeof pts[k]);
      memcpy(pts[ct->nv], ct->link[s], sizeof pts[0]);
      ct->cof_type[s] = locate(cx, ct->nv + 1, pts, ct->cof_anchor[s], &ct->cof_pos[s]);
    }
    if (ct->dim > 0)
      for (int k = 0; k < ct->nv; k++) {
        int pts[4][3], np = 0;
        for (int i = 0; i < ct->nv; i++) if (i != k) memcpy(pts[np++], ct->off[i], sizeof pts[0]);
        ct->fac_type[k] = locate(cx, np, pts, ct->fac_anchor[k], NULL);
      }
  }
}

typedef struct { int64_t x, y, z; } co_t;

static inline co_t coords(const cx_t* cx, int64_t v) {
  co_t c; c.x = v % cx->n[0]; c.y = (v / cx->n[0]) % cx->n[1]; c.z = v / (cx->n[0] * cx->n[1]);
  return c;
}
static inline int inside(const cx_t* cx, int64_t x, int64_t y, int64_t z) {
  return x >= 0 && y >= 0 && z >= 0 && x < cx->n[0] && y < cx->n[1] && z < cx->n[2];
}
static inline int64_t vid(const cx_t* cx, int64_t x, int64_t y, int64_t z) {
  return x + cx->n[0] * (y + cx->n[1] * z);
}
/* global vertex ids of cell (anchor A, type ti); returns 0 if the cell leaves the grid */
static int cell_vertices(const cx_t* cx, int64_t A, int ti, int64_t* vs) {
  co_t a = coords(cx, A);
  const ctype_t* ct = &cx->t[ti];
  for (int k = 0; k < ct->nv; k++) {
    int64_t x = a.x + ct->off[k][0], y = a.y + ct->off[k][1], z = a.z + ct->off[k][2];
    if (!inside(cx, x, y, z)) return 0;
    vs[k] = vid(cx, x, y, z);
  }
  return 1;
}

/* ------------------------------------------------------------------------- */
/* Simulation of simplicity and the extended function of Eq. 1.              */
/* ------------------------------------------------------------------------- */

/* u < v in the SoS total order: (value, index) lexicographic (reading A2) */
static inline int sos_less(const float* f, int64_t u, int64_t v) {
  return f[u] < f[v] || (f[u] == f[v] && u < v);
}

/* key of a cell = its vertices sorted descending in SoS order; lexicographic
 * comparison of keys realises Eq. 1 with symbolic epsilon (reading A3) */
static void key_of(const float* f, int n, const int64_t* vs, int64_t* key) {
  for (int i = 0; i < n; i++) key[i] = vs[i];
  for (int i = 1; i < n; i++) {
    int64_t x = key[i]; int j = i;
    while (j > 0 && sos_less(f, key[j - 1], x)) { key[j] = key[j - 1]; j--; }
    key[j] = x;
  }
}
static int key_less(const float* f, int n, const int64_t* a, const int64_t* b) {
  for (int i = 0; i < n; i++) {
    if (a[i] == b[i]) continue;
    return sos_less(f, a[i], b[i]);
  }
  return 0;
}
static int same_set(int n, const int64_t* a, const int64_t* b) {
  for (int i = 0; i < n; i++) {
    int found = 0;
    for (int j = 0; j < n; j++) if (a[i] == b[j]) found = 1;
    if (!found) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------------- */
/* Discrete gradient.                                   */
/* up[A*T+t] = link slot of the cofacet the cell is paired with, or -1;       */
/* dn[A*T+t] = position (in the cell's vertex list) of the vertex that is NOT  */
/*             in the facet it is paired with, or -1.                          */
/* ------------------------------------------------------------------------- */

typedef struct { int8_t* up; int8_t* dn; } grad_t;

static int grad_alloc(const cx_t* cx, grad_t* G) {
  size_t n = (size_t)cx->N * cx->T;
  G->up = (int8_t*)malloc(n); G->dn = (int8_t*)malloc(n);
  return G->up && G->dn;
}
static void grad_free(grad_t* G) { free(G->up); free(G->dn); G->up = G->dn = NULL; }

/* cofacet b = a + {w}; its (anchor id, type) */
static int64_t cofacet_cell(const cx_t* cx, int64_t A, int ti, int s, int* bt) {
  co_t a = coords(cx, A);
  const ctype_t* ct = &cx->t[ti];
  *bt = ct->cof_type[s];
  return vid(cx, a.x + ct->cof_anchor[s][0], a.y + ct->cof_anchor[s][1], a.z + ct->cof_anchor[s][2]);
}
static int64_t facet_cell(const cx_t* cx, int64_t A, int ti, int k, int* ft) {
  co_t a = coords(cx, A);
  const ctype_t* ct = &cx->t[ti];
  *ft = ct->fac_type[k];
  return vid(cx, a.x + ct->fac_anchor[k][0], a.y + ct->fac_anchor[k][1], a.z + ct->fac_anchor[k][2]);
}

/* Pair one d-cell literally.  Returns the chosen slot or -1. */
static int pair_cell(const cx_t* cx, const float* f, int64_t A, int ti) {
  const ctype_t* ct = &cx->t[ti];
  int64_t av[4];
  if (!cell_vertices(cx, A, ti, av)) return -1;
  co_t a = coords(cx, A);
  int n = ct->nv, best = -1;
  int64_t bestkey[5];
  for (int s = 0; s < ct->nlink; s++) {
    int64_t x = a.x + ct->link[s][0], y = a.y + ct->link[s][1], z = a.z + ct->link[s][2];
    if (!inside(cx, x, y, z)) continue;           /* cofacet leaves the grid */
    int64_t bv[5], key[5];
    for (int k = 0; k < n; k++) bv[k] = av[k];
    bv[n] = vid(cx, x, y, z);
    key_of(f, n + 1, bv, key);
    /* G0(b) = b minus its lowest vertex = the first n entries of the key */
    if (!same_set(n, key, av)) continue;          /* a is not the highest facet of b */
    if (best < 0 || key_less(f, n + 1, key, bestkey)) {
      best = s;
      memcpy(bestkey, key, sizeof(int64_t) * (n + 1));
    }
  }
  return best;
}

/* compute_gradient: dimensions ascending; a cell already paired with a facet is
 * not paired again (S:177 / reading A4); P_a empty -> a stays unpaired. */
static void gradient(const cx_t* cx, const float* f, grad_t* G) {
  size_t n = (size_t)cx->N * cx->T;
  memset(G->up, -1, n);
  memset(G->dn, -1, n);
  for (int d = 0; d < cx->top; d++) {
    int t0 = cx->first_of_dim[d], t1 = cx->first_of_dim[d + 1];
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t A = 0; A < cx->N; A++) {
      for (int ti = t0; ti < t1; ti++) {
        if (G->dn[A * cx->T + ti] >= 0) continue;
        int s = pair_cell(cx, f, A, ti);
        if (s < 0) continue;
        G->up[A * cx->T + ti] = (int8_t)s;
        int bt;
        int64_t B = cofacet_cell(cx, A, ti, s, &bt);
        G->dn[B * cx->T + bt] = (int8_t)cx->t[ti].cof_pos[s];
      }
    }
  }
}

static inline int cell_exists(const cx_t* cx, int64_t A, int ti) {
  int64_t vs[4];
  return cell_vertices(cx, A, ti, vs);
}

/* Frontier update of a gradient (the oracle's frontier mode, used for the full-size
 * C3/C4 goldens).  The pairing of a cell anchored at A reads the
 * values of A + [-1,1]^D only (the cell and its link), and whether a cell
 * is paired down reads the pairings of its facets, anchored in A + {0,1}^D.  So
 * when the values changed only at vertices v with a flag in `D` dilated by
 * [-2,1]^D (i.e. D[A] = 1 for every anchor A with a changed vertex in
 * A + [-1,2]^D), every cell whose pair can differ is anchored where D[A] = 1, and
 * recomputing exactly those cells -- with the literal rule, dimensions ascending,
 * a cell paired with a facet not paired again -- gives the gradient a
 * full recomputation gives (tests/test_oracle_frontier.py checks that claim
 * against full mode bit for bit).  dn of a recomputed cell is re-derived from
 * its facets' pairs (the facets may lie outside D and keep their pairs). */
static void gradient_update(const cx_t* cx, const float* f, grad_t* G, const uint8_t* D) {
  const int T = cx->T;
  for (int d = 0; d <= cx->top; d++) {
    int t0 = cx->first_of_dim[d], t1 = cx->first_of_dim[d + 1];
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t A = 0; A < cx->N; A++) {
      if (!D[A]) continue;
      for (int ti = t0; ti < t1; ti++) {
        size_t i = (size_t)A * T + ti;
        G->dn[i] = -1;
        if (d == 0 || !cell_exists(cx, A, ti)) continue;
        for (int k = 0; k <= d; k++) {
          int ft;
          int64_t C = facet_cell(cx, A, ti, k, &ft);
          int s = G->up[(size_t)C * T + ft];
          if (s < 0) continue;
          int bt;
          int64_t B = cofacet_cell(cx, C, ft, s, &bt);
          if (B == A && bt == ti) G->dn[i] = (int8_t)k;
        }
      }
    }
    if (d == cx->top) break;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t A = 0; A < cx->N; A++) {
      if (!D[A]) continue;
      for (int ti = t0; ti < t1; ti++) {
        size_t i = (size_t)A * T + ti;
        G->up[i] = -1;
        if (G->dn[i] >= 0) continue;
        int s = pair_cell(cx, f, A, ti);
        if (s >= 0) G->up[i] = (int8_t)s;
      }
    }
  }
}

/* D[A] = 1 iff some vertex with T[v] = 1 lies in A + [-1,2]^D (see above). */
static void dilate_targets(const cx_t* cx, const uint8_t* T, uint8_t* D) {
  int zlo = cx->D == 3 ? -1 : 0, zhi = cx->D == 3 ? 2 : 0;
#pragma omp parallel for schedule(static)
  for (int64_t A = 0; A < cx->N; A++) {
    co_t a = coords(cx, A);
    uint8_t hit = 0;
    for (int dz = zlo; dz <= zhi && !hit; dz++)
      for (int dy = -1; dy <= 2 && !hit; dy++)
        for (int dx = -1; dx <= 2 && !hit; dx++) {
          int64_t x = a.x + dx, y = a.y + dy, z = a.z + dz;
          if (inside(cx, x, y, z) && T[vid(cx, x, y, z)]) hit = 1;
        }
    D[A] = hit;
  }
}
static inline int is_crit(const cx_t* cx, const grad_t* G, int64_t A, int ti) {
  size_t i = (size_t)A * cx->T + ti;
  return G->up[i] < 0 && G->dn[i] < 0 && cell_exists(cx, A, ti);
}

/* ------------------------------------------------------------------------- */
/* Exported: gradient in the documented packed form.                          */
/*  3D code (u64): bits 0-3 vertex slot (15 = none); edges e_k at 4+3k (7 =  */
/*  none); triangles t_k at 25+2k (3 = none).  2D code (u16): bits 0-2 vertex  */
/*  slot (7 = none); edges at 3+2k (3 = none).                                */
/*  crit mask (u32): bit t set iff cell (anchor, type t) is critical.         */
/* ------------------------------------------------------------------------- */

static int check_dims(const int64_t* dims) {
  if (dims[0] < 2 || dims[1] < 2 || dims[2] < 1) return OR_E_DIMS;
  return OR_OK;
}

static void export_codes(const cx_t* cx, const grad_t* G, void* codes, uint32_t* crit) {
  for (int64_t A = 0; A < cx->N; A++) {
    uint64_t c = 0;
    uint32_t m = 0;
    for (int ti = 0; ti < cx->T; ti++) {
      int d = cx->t[ti].dim;
      int k = ti - cx->first_of_dim[d];
      int s = G->up[A * cx->T + ti];
      if (cx->D == 3) {
        if (d == 0) c |= (uint64_t)(s < 0 ? 15 : s);
        else if (d == 1) c |= (uint64_t)(s < 0 ? 7 : s) << (4 + 3 * k);
        else if (d == 2) c |= (uint64_t)(s < 0 ? 3 : s) << (25 + 2 * k);
      } else {
        if (d == 0) c |= (uint64_t)(s < 0 ? 7 : s);
        else if (d == 1) c |= (uint64_t)(s < 0 ? 3 : s) << (3 + 2 * k);
      }
      if (is_crit(cx, G, A, ti)) m |= 1u << ti;
    }
    if (codes) {
      if (cx->D == 3) ((uint64_t*)codes)[A] = c;
      else ((uint16_t*)codes)[A] = (uint16_t)c;
    }
    if (crit) crit[A] = m;
  }
}

int dmtz_oracle_gradient(const int64_t* dims, const float* field, void* codes, uint32_t* crit) {
  int st = check_dims(dims);
  if (st) return st;
  for (int64_t i = 0; i < dims[0] * dims[1] * dims[2]; i++) if (!isfinite(field[i])) return OR_E_NONFINITE;
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  grad_t G;
  if (!grad_alloc(&cx, &G)) return OR_E_ARG;
  gradient(&cx, field, &G);
  export_codes(&cx, &G, codes, crit);
  grad_free(&G);
  return OR_OK;
}

/* Introspection for tests: the complex as the oracle derived it. */
int dmtz_oracle_complex_info(const int64_t* dims, int32_t* out_T, int32_t* dim_of_type,
                             int32_t* nlink_of_type, int32_t* offsets /* T*4*3 */,
                             int32_t* links /* T*14*3 */) {
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  *out_T = cx.T;
  for (int ti = 0; ti < cx.T; ti++) {
    dim_of_type[ti] = cx.t[ti].dim;
    nlink_of_type[ti] = cx.t[ti].nlink;
    for (int k = 0; k < 4; k++) for (int a = 0; a < 3; a++)
      offsets[(ti * 4 + k) * 3 + a] = k < cx.t[ti].nv ? cx.t[ti].off[k][a] : 0;
    for (int s = 0; s < MAXLINK; s++) for (int a = 0; a < 3; a++)
      links[(ti * MAXLINK + s) * 3 + a] = s < cx.t[ti].nlink ? cx.t[ti].link[s][a] : 0;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* The C-loop with Eq. 2 edits.         */
/* ------------------------------------------------------------------------- */

typedef struct {
  int64_t rounds, n_edited, n_quantized, n_lossless, n_false_round0;
  int64_t false_by_kind_round0[8]; /* FPmin FNmin FP1s FN1s FP2s FN2s FPmax FNmax */
  int32_t status, pad;
} or_stats;

typedef struct { uint64_t v; uint16_t q; uint8_t lossless; uint8_t pad; float value; } or_edit;

/* lb = RU(f - xi): the smallest float >= f - xi, so g >= lb implies |g - f| <= xi
 * exactly (reading A9). */
static float lower_bound_ru(float f, float xi) {
  int old = fegetround();
  fesetround(FE_UPWARD);
  volatile float a = f, b = xi;
  volatile float r = a - b;
  fesetround(old);
  return r;
}
static float upper_bound_rd(float f, float xi) {
  int old = fegetround();
  fesetround(FE_DOWNWARD);
  volatile float a = f, b = xi;
  volatile float r = a + b;
  fesetround(old);
  return r;
}

/* kind index: 2*critical-class + (false negative ? 1 : 0); classes: min, 1-saddle,
 * 2-saddle, max (2D: the triangle is the max) */
static int kind_of(const cx_t* cx, int dim, int fn) {
  int cls = (dim == cx->top) ? 3 : dim;
  return 2 * cls + (fn ? 1 : 0);
}

/* SoS-lowest vertex of a cell under field f */
static int64_t lowest_vertex(const float* f, int n, const int64_t* vs) {
  int64_t m = vs[0];
  for (int i = 1; i < n; i++) if (sos_less(f, vs[i], m)) m = vs[i];
  return m;
}

/* Target vertex for false cell a (rules R1/R2/R3a/R3b):
 *  FP (critical in g, paired in f):
 *     the vertex of the larger cell of a's f-pair that is not in the smaller one.
 *  FN (critical in f, paired in g):
 *     paired up in g             -> m = f-lowest vertex of a             (R2)
 *     paired down in g with c,
 *        y = a \ c, m != y        -> m                                    (R3a)
 *        m == y                   -> the vertex c is paired with in f     (R3b)
 * Returns -1 on an internal inconsistency. */
static int64_t target_of(const cx_t* cx, const float* f, const grad_t* Gf, const grad_t* Gg,
                         int64_t A, int ti, int fn, int* rule) {
  const ctype_t* ct = &cx->t[ti];
  int64_t av[4];
  cell_vertices(cx, A, ti, av);
  size_t i = (size_t)A * cx->T + ti;
  co_t a = coords(cx, A);
  if (!fn) {
    *rule = 1;
    if (Gf->up[i] >= 0) {
      int s = Gf->up[i];
      return vid(cx, a.x + ct->link[s][0], a.y + ct->link[s][1], a.z + ct->link[s][2]);
    }
    return av[(int)Gf->dn[i]];
  }
  int64_t m = lowest_vertex(f, ct->nv, av);
  *rule = 2;
  if (Gg->up[i] >= 0) return m;
  int k = Gg->dn[i];
  int64_t y = av[k];
  *rule = 3;
  if (m != y) return m;
  *rule = 4;
  int ft;
  int64_t C = facet_cell(cx, A, ti, k, &ft);
  int s = Gf->up[(size_t)C * cx->T + ft];
  if (s < 0) return -1;
  co_t c = coords(cx, C);
  const ctype_t* fc = &cx->t[ft];
  return vid(cx, c.x + fc->link[s][0], c.y + fc->link[s][1], c.z + fc->link[s][2]);
}

/* One literal round of classification: F = C_f xor C_g (tier 1: dims 0 and top,
 * P:140-141), target set T (a set: each vertex at most once per round).
 * Returns |F| (or -1 on internal error); kinds[8] accumulates counts. */
static int64_t classify(const cx_t* cx, const float* f, const grad_t* Gf, const grad_t* Gg,
                        int tier, uint8_t* T, int64_t* kinds, const uint8_t* D, int64_t* rules) {
  int64_t nF = 0, bad = 0;
  int64_t kk[8] = {0}, rr[5] = {0};
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : nF, bad) reduction(+ : kk[:8], rr[:5])
  for (int64_t A = 0; A < cx->N; A++) {
    if (D && !D[A]) continue;  /* frontier mode: no false cell is anchored outside D */
    for (int ti = 0; ti < cx->T; ti++) {
      int d = cx->t[ti].dim;
      if (tier == 1 && d != 0 && d != cx->top) continue;
      if (!cell_exists(cx, A, ti)) continue;
      int cf = is_crit(cx, Gf, A, ti), cg = is_crit(cx, Gg, A, ti);
      if (cf == cg) continue;
      int fn = cf;  /* critical in f, paired in g: false negative */
      nF++;
      kk[kind_of(cx, d, fn)]++;
      int rule = 0;
      int64_t v = target_of(cx, f, Gf, Gg, A, ti, fn, &rule);
      rr[rule]++;
      if (v < 0) { bad++; continue; }
#pragma omp atomic write
      T[v] = 1;
    }
  }
  for (int k = 0; k < 8; k++) kinds[k] += kk[k];
  if (rules) for (int k = 1; k < 5; k++) rules[k - 1] += rr[k];
  return bad ? -1 : nF;
}

/* diag (optional, int64[6], accumulated over the rounds; instrumentation for the
 * progress-lemma pin): [0] targets whose g was not above lb when selected, [1..4]
 * false cells resolved by rule R1 / R2 / R3a / R3b, [5] targets (set members).
 * frontier = 0: every round recomputes the whole gradient of g and classifies every
 * cell (the literal loop).  frontier = 1: round 1 does; round r > 1 recomputes the
 * cells anchored in D_r = { A : a target of round r-1 lies in A + [-1,2]^D } (the
 * only cells whose pair can change, see gradient_update) and classifies the cells
 * anchored in D_r: a false cell of round r was either false in round r-1 -- it is
 * anchored within [-2,1]^D of its own target (its target is one of its vertices,
 * of its pair's vertices or of its facet's pair's vertices) -- or became false
 * because a vertex it reads (A + [-1,2]^D) changed, and every changed vertex was
 * a target.  Checked equal to frontier = 0 in tests/test_oracle_frontier.py. */
int dmtz_oracle_correct_ex(const int64_t* dims, const float* f, const float* fhat, float xi,
                           int32_t q_max, int32_t q_cap, int32_t tier, int64_t max_rounds, int32_t frontier,
                           float* g_out, uint32_t* state_out, or_edit* edits, int64_t edits_capacity,
                           int64_t* n_edits, or_stats* stats, int64_t* round_log, double* round_sec,
                           int64_t round_log_cap, int64_t* diag) {
  memset(stats, 0, sizeof *stats);
  *n_edits = 0;
  int st = check_dims(dims);
  if (st) { stats->status = st; return st; }
  if (!(xi > 0.0f) || !isfinite(xi) || q_max < 0 || q_max > 30 || q_cap < 1 || q_cap > 65535 ||
      (tier != 1 && tier != 2) || max_rounds < 0) {
    stats->status = OR_E_ARG; return OR_E_ARG;
  }
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  int64_t N = cx.N;
  for (int64_t v = 0; v < N; v++)
    if (!isfinite(f[v]) || !isfinite(fhat[v])) { stats->status = OR_E_NONFINITE; return OR_E_NONFINITE; }
  /* |fhat - f| <= xi exactly  <=>  RU(f - xi) <= fhat <= RD(f + xi) */
  for (int64_t v = 0; v < N; v++)
    if (fhat[v] < lower_bound_ru(f[v], xi) || fhat[v] > upper_bound_rd(f[v], xi)) {
      stats->status = OR_E_BOUND; return OR_E_BOUND;
    }
  if (max_rounds == 0) max_rounds = N * (int64_t)(q_cap + 1);
  float step = ldexpf(xi, -q_max);           /* xi / 2^q_max, exact */
  float* lb = (float*)malloc(sizeof(float) * N);
  uint16_t* q = (uint16_t*)calloc(N, sizeof(uint16_t));
  uint8_t* lossless = (uint8_t*)calloc(N, 1);
  uint8_t* T = (uint8_t*)calloc(N, 1);
  grad_t Gf, Gg;
  if (!lb || !q || !lossless || !T || !grad_alloc(&cx, &Gf) || !grad_alloc(&cx, &Gg)) {
    stats->status = OR_E_ARG; return OR_E_ARG;
  }
  for (int64_t v = 0; v < N; v++) { lb[v] = lower_bound_ru(f[v], xi); g_out[v] = fhat[v]; }
  uint8_t* Dm = frontier ? (uint8_t*)malloc(N) : NULL;
  if (frontier && !Dm) { stats->status = OR_E_ARG; return OR_E_ARG; }
  gradient(&cx, f, &Gf);
  int status = OR_OK;
  for (int64_t round = 1;; round++) {
#ifdef _OPENMP
    double t_round0 = omp_get_wtime();  /* instrumentation only: wall time of each round */
#endif
    if (round == 1 || !frontier) {
      gradient(&cx, g_out, &Gg);
    } else {
      dilate_targets(&cx, T, Dm);
      gradient_update(&cx, g_out, &Gg, Dm);
    }
    memset(T, 0, N);
    int64_t kinds[8] = {0};
    int64_t nF = classify(&cx, f, &Gf, &Gg, tier, T, kinds, (round == 1 || !frontier) ? NULL : Dm,
                          diag ? diag + 1 : NULL);
    if (round_log && round - 1 < round_log_cap) round_log[round - 1] = nF;
    if (nF < 0) { status = OR_E_INTERNAL; break; }
    if (round == 1) {
      stats->n_false_round0 = nF;
      memcpy(stats->false_by_kind_round0, kinds, sizeof kinds);
    }
    if (nF == 0) break;
    stats->rounds = round;
    int changed = 0;
    for (int64_t v = 0; v < N; v++) {
      if (diag && T[v]) {                 /* diagnostics: targets, and targets already at lb */
        diag[5]++;
        if (!(g_out[v] > lb[v])) diag[0]++;
      }
      if (!T[v] || lossless[v]) continue;
      changed = 1;
      /* Eq. 2: one step of xi/2^q_max, recomputed from fhat:
       * g' = RN(fhat - RN((q+1) * step)), accepted iff q+1 <= q_cap and g' >= lb;
       * otherwise clamp to the lower bound and store losslessly. */
      if (q[v] + 1 <= q_cap) {
        float s = (float)(q[v] + 1) * step;
        float gp = fhat[v] - s;
        if (gp >= lb[v]) { q[v]++; g_out[v] = gp; continue; }
      }
      g_out[v] = lb[v];
      lossless[v] = 1;
    }
#ifdef _OPENMP
    if (round_sec && round - 1 < round_log_cap) round_sec[round - 1] = omp_get_wtime() - t_round0;
#endif
    if (!changed) { status = OR_E_STUCK; break; }
    if (round == max_rounds) { status = OR_E_ITER_CAP; break; }
  }
  int64_t ne = 0;
  for (int64_t v = 0; v < N; v++) {
    if (state_out) state_out[v] = (uint32_t)q[v] | ((uint32_t)lossless[v] << 16);
    if (q[v] == 0 && !lossless[v]) continue;
    stats->n_edited++;
    if (lossless[v]) stats->n_lossless++; else stats->n_quantized++;
    if (edits && ne < edits_capacity) {
      edits[ne].v = (uint64_t)v; edits[ne].q = q[v]; edits[ne].lossless = lossless[v];
      edits[ne].pad = 0; edits[ne].value = g_out[v];
    }
    ne++;
  }
  *n_edits = ne;
  if (status == OR_OK && edits && ne > edits_capacity) status = OR_E_CAPACITY;
  stats->status = status;
  free(lb); free(q); free(lossless); free(T); free(Dm);
  grad_free(&Gf); grad_free(&Gg);
  return status;
}

int dmtz_oracle_correct(const int64_t* dims, const float* f, const float* fhat, float xi,
                        int32_t q_max, int32_t q_cap, int32_t tier, int64_t max_rounds,
                        float* g_out, uint32_t* state_out, or_edit* edits, int64_t edits_capacity,
                        int64_t* n_edits, or_stats* stats) {
  return dmtz_oracle_correct_ex(dims, f, fhat, xi, q_max, q_cap, tier, max_rounds, 0, g_out, state_out,
                                edits, edits_capacity, n_edits, stats, NULL, NULL, 0, NULL);
}

/* ------------------------------------------------------------------------- */
/* V-path traces (P:82 gradient paths; P:228 ascending/descending paths and   */
/* saddle-saddle connectors).                                                 */
/* cell id = (dim << 56) | (anchor * T_dim + index of the type within dim).   */
/* ------------------------------------------------------------------------- */

enum { KIND_DESC = 1, KIND_ASC = 2, KIND_CONN = 4 };

static uint64_t cell_id(const cx_t* cx, int64_t A, int ti) {
  int d = cx->t[ti].dim;
  int Td = cx->first_of_dim[d + 1] - cx->first_of_dim[d];
  return ((uint64_t)d << 56) | (uint64_t)(A * Td + (ti - cx->first_of_dim[d]));
}

typedef struct {
  int64_t cap_b, cap_c, nb, nc;
  int64_t* off; uint64_t* cells; uint64_t* origin; uint64_t* terminal; uint8_t* kind;
  uint64_t* dig;  /* non-NULL: digest mode -- nothing is stored, see csr_digest_mix */
} csr_t;

/* Digest mode (for the full-size goldens, whose CSR does not fit in host memory):
 * instead of storing array X, accumulate sum_i mix(X[i] ^ (i * 0x9E3779B97F4A7C15))
 * mod 2^64, mix = the splitmix64 finalizer.  dig[0..4] = offsets, cells, origin,
 * terminal, kind.  A checksum of the output, not part of the method; the tests
 * compute the same sums over the GPU's arrays (tests/digest.py). */
static uint64_t csr_digest_mix(uint64_t x, uint64_t i) {
  uint64_t z = x ^ (i * 0x9E3779B97F4A7C15ull);
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void csr_begin(csr_t* o, uint64_t origin, uint8_t kind) {
  if (o->dig) {
    o->dig[2] += csr_digest_mix(origin, (uint64_t)o->nb);
    o->dig[4] += csr_digest_mix(kind, (uint64_t)o->nb);
    return;
  }
  if (o->nb < o->cap_b) { o->off[o->nb] = o->nc; o->origin[o->nb] = origin; o->kind[o->nb] = kind; }
}
static void csr_push(csr_t* o, uint64_t c) {
  if (o->dig) o->dig[1] += csr_digest_mix(c, (uint64_t)o->nc);
  else if (o->nc < o->cap_c) o->cells[o->nc] = c;
  o->nc++;
}
static void csr_end(csr_t* o, uint64_t terminal) {
  if (o->dig) {
    o->dig[3] += csr_digest_mix(terminal, (uint64_t)o->nb);
    o->dig[0] += csr_digest_mix((uint64_t)o->nc, (uint64_t)o->nb + 1);
  } else if (o->nb < o->cap_b) {
    o->terminal[o->nb] = terminal; o->off[o->nb + 1] = o->nc;
  }
  o->nb++;
}

/* top cofacets of a (top-1)-cell (at most 2), in slot order */
static int top_cofacets(const cx_t* cx, int64_t A, int ti, int64_t* Bs, int* bts) {
  const ctype_t* ct = &cx->t[ti];
  co_t a = coords(cx, A);
  int n = 0;
  for (int s = 0; s < ct->nlink; s++) {
    if (!inside(cx, a.x + ct->link[s][0], a.y + ct->link[s][1], a.z + ct->link[s][2])) continue;
    Bs[n] = cofacet_cell(cx, A, ti, s, &bts[n]);
    n++;
  }
  return n;
}

/* Growable CSR for the oracle's internal traces (the exported trace writes into
 * caller buffers with fixed capacities instead). */
static int csr_grow(csr_t* o) {
  if (o->nb + 1 >= o->cap_b) {
    int64_t nb = o->cap_b ? 2 * o->cap_b : 1024;
    o->off = (int64_t*)realloc(o->off, sizeof(int64_t) * (nb + 1));
    o->origin = (uint64_t*)realloc(o->origin, sizeof(uint64_t) * nb);
    o->terminal = (uint64_t*)realloc(o->terminal, sizeof(uint64_t) * nb);
    o->kind = (uint8_t*)realloc(o->kind, nb);
    if (!o->off || !o->origin || !o->terminal || !o->kind) return 0;
    o->cap_b = nb;
  }
  if (o->nc + 4 >= o->cap_c) {
    int64_t nc = o->cap_c ? 2 * o->cap_c : 65536;
    o->cells = (uint64_t*)realloc(o->cells, sizeof(uint64_t) * nc);
    if (!o->cells) return 0;
    o->cap_c = nc;
  }
  return 1;
}
static void csr_free(csr_t* o) {
  free(o->off); free(o->cells); free(o->origin); free(o->terminal); free(o->kind);
  memset(o, 0, sizeof *o);
}
#define CSR_ROOM(o) do { if (grow && !csr_grow(o)) return OR_E_ARG; } while (0)

/* The traces of gradient G into o (grow = 1: o is reallocated as needed).
 * Returns OR_OK, or OR_E_INTERNAL on a cycle (never expected: paths strictly
 * decrease the extended function). */
static int trace_grad(const cx_t* cxp, const grad_t* Gp, uint32_t kinds, csr_t* op, int grow) {
  const cx_t cx = *cxp;
  const grad_t G = *Gp;
  csr_t* po = op;
#define o (*po)
  if (o.dig) o.dig[0] += csr_digest_mix(0, 0);  /* offsets[0] = 0 */
  else if (o.cap_b > 0) o.off[0] = 0;
  int64_t maxsteps = cx.N * cx.T + 1;
  int err = 0;
  int T = cx.T;
  /* descending: from each endpoint of each critical edge (1-saddle), follow
   * vertex -> paired edge -> its other vertex until a critical vertex */
  if (kinds & KIND_DESC) {
    for (int64_t A = 0; A < cx.N && !err; A++)
      for (int ti = cx.first_of_dim[1]; ti < cx.first_of_dim[2] && !err; ti++) {
        if (!is_crit(&cx, &G, A, ti)) continue;
        int64_t ev[2];
        cell_vertices(&cx, A, ti, ev);
        for (int b = 0; b < 2; b++) {
          CSR_ROOM(&o); csr_begin(&o, cell_id(&cx, A, ti), KIND_DESC);
          int64_t v = ev[b];
          CSR_ROOM(&o); csr_push(&o, cell_id(&cx, v, 0));
          int64_t steps = 0;
          while (G.up[(size_t)v * T + 0] >= 0) {
            int s = G.up[(size_t)v * T + 0], bt;
            int64_t E = cofacet_cell(&cx, v, 0, s, &bt);
            co_t c = coords(&cx, v);
            int64_t w = vid(&cx, c.x + cx.t[0].link[s][0], c.y + cx.t[0].link[s][1], c.z + cx.t[0].link[s][2]);
            CSR_ROOM(&o); csr_push(&o, cell_id(&cx, E, bt));
            CSR_ROOM(&o); csr_push(&o, cell_id(&cx, w, 0));
            v = w;
            if (++steps > maxsteps) { err = 1; break; }
          }
          csr_end(&o, cell_id(&cx, v, 0));
        }
      }
  }
  /* ascending: from each critical (top-1)-cell, through each top cofacet t:
   * t critical -> maximum; else t is paired down with facet c; continue
   * through c's other top cofacet; none -> the path leaves the domain */
  if ((kinds & KIND_ASC) && !err) {
    int d = cx.top - 1;
    for (int64_t A = 0; A < cx.N && !err; A++)
      for (int ti = cx.first_of_dim[d]; ti < cx.first_of_dim[d + 1] && !err; ti++) {
        if (!is_crit(&cx, &G, A, ti)) continue;
        int64_t Bs[2]; int bts[2];
        int nb = top_cofacets(&cx, A, ti, Bs, bts);
        for (int b = 0; b < nb; b++) {
          CSR_ROOM(&o); csr_begin(&o, cell_id(&cx, A, ti), KIND_ASC);
          int64_t B = Bs[b]; int bt = bts[b];
          uint64_t term = BOUNDARY_ID;
          int64_t steps = 0;
          for (;;) {
            CSR_ROOM(&o); csr_push(&o, cell_id(&cx, B, bt));
            if (is_crit(&cx, &G, B, bt)) { term = cell_id(&cx, B, bt); break; }
            int k = G.dn[(size_t)B * T + bt];
            if (k < 0) { err = 1; break; }
            int ct;
            int64_t C = facet_cell(&cx, B, bt, k, &ct);
            CSR_ROOM(&o); csr_push(&o, cell_id(&cx, C, ct));
            int64_t Cs[2]; int cts[2];
            int nc = top_cofacets(&cx, C, ct, Cs, cts);
            int moved = 0;
            for (int j = 0; j < nc; j++)
              if (!(Cs[j] == B && cts[j] == bt)) { B = Cs[j]; bt = cts[j]; moved = 1; break; }
            if (!moved) break;  /* boundary facet: BOUNDARY terminal */
            if (++steps > maxsteps) { err = 1; break; }
          }
          csr_end(&o, term);
        }
      }
  }
  /* saddle-saddle connectors (3D): breadth-first from each critical triangle over
   * facet edges: critical edge -> reached 1-saddle (recorded each time met);
   * edge paired up with a triangle t' != current -> enqueue t' if unvisited */
  if ((kinds & KIND_CONN) && !err && cx.D == 3) {
    int64_t qcap = 1024;
    int64_t* qa = (int64_t*)malloc(sizeof(int64_t) * qcap);
    int* qt = (int*)malloc(sizeof(int) * qcap);
    uint8_t* seen = (uint8_t*)calloc((size_t)cx.N * T, 1);
    for (int64_t A = 0; A < cx.N && !err; A++)
      for (int ti = cx.first_of_dim[2]; ti < cx.first_of_dim[3] && !err; ti++) {
        if (!is_crit(&cx, &G, A, ti)) continue;
        CSR_ROOM(&o); csr_begin(&o, cell_id(&cx, A, ti), KIND_CONN);
        int64_t head = 0, tail = 0;
        qa[tail] = A; qt[tail] = ti; tail++;
        seen[(size_t)A * T + ti] = 1;
        while (head < tail) {
          int64_t B = qa[head]; int bt = qt[head]; head++;
          for (int k = 0; k < 3; k++) {
            int et;
            int64_t E = facet_cell(&cx, B, bt, k, &et);
            if (is_crit(&cx, &G, E, et)) { CSR_ROOM(&o); csr_push(&o, cell_id(&cx, E, et)); continue; }
            int s = G.up[(size_t)E * T + et];
            if (s < 0) continue;  /* paired down with a vertex: the path stops */
            int nt;
            int64_t Nb = cofacet_cell(&cx, E, et, s, &nt);
            if (Nb == B && nt == bt) continue;
            if (seen[(size_t)Nb * T + nt]) continue;
            seen[(size_t)Nb * T + nt] = 1;
            CSR_ROOM(&o); csr_push(&o, cell_id(&cx, Nb, nt));
            if (tail == qcap) {
              qcap *= 2;
              qa = (int64_t*)realloc(qa, sizeof(int64_t) * qcap);
              qt = (int*)realloc(qt, sizeof(int) * qcap);
            }
            qa[tail] = Nb; qt[tail] = nt; tail++;
          }
        }
        for (int64_t j = 0; j < tail; j++) seen[(size_t)qa[j] * T + qt[j]] = 0;
        csr_end(&o, BOUNDARY_ID);
      }
    free(qa); free(qt); free(seen);
  }
#undef o
  return err ? OR_E_INTERNAL : OR_OK;
}

/* The trace in digest mode: n_branches, n_cells, per-kind branch counts are not
 * separated (the kind digest covers them); dig[5] as in csr_t. */
int dmtz_oracle_trace_digest(const int64_t* dims, const float* field, uint32_t kinds, uint64_t* dig,
                             int64_t* n_branches, int64_t* n_cells) {
  int st = check_dims(dims);
  if (st) return st;
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  grad_t G;
  if (!grad_alloc(&cx, &G)) return OR_E_ARG;
  gradient(&cx, field, &G);
  for (int k = 0; k < 5; k++) dig[k] = 0;
  csr_t o = {0, 0, 0, 0, NULL, NULL, NULL, NULL, NULL, dig};
  int err = trace_grad(&cx, &G, kinds, &o, 0);
  grad_free(&G);
  *n_branches = o.nb;
  *n_cells = o.nc;
  return err;
}

int dmtz_oracle_trace(const int64_t* dims, const float* field, uint32_t kinds,
                      int64_t cap_branches, int64_t cap_cells, int64_t* branch_offsets,
                      uint64_t* cells, uint64_t* origin, uint64_t* terminal, uint8_t* kind,
                      int64_t* n_branches, int64_t* n_cells) {
  int st = check_dims(dims);
  if (st) return st;
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  grad_t G;
  if (!grad_alloc(&cx, &G)) return OR_E_ARG;
  gradient(&cx, field, &G);
  csr_t o = {cap_branches, cap_cells, 0, 0, branch_offsets, cells, origin, terminal, kind, NULL};
  if (cap_branches > 0) branch_offsets[0] = 0;
  int err = trace_grad(&cx, &G, kinds, &o, 0);
  grad_free(&G);
  *n_branches = o.nb;
  *n_cells = o.nc;
  if (err) return err;
  if (o.nb > cap_branches || o.nc > cap_cells) return OR_E_CAPACITY;
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* S-loops and the alternating C/S driver (Fig. 2).         */
/* ------------------------------------------------------------------------- */

/* (anchor, type) of a cell id */
static void id_to_cell(const cx_t* cx, uint64_t id, int64_t* A, int* ti) {
  int d = (int)(id >> 56);
  int Td = cx->first_of_dim[d + 1] - cx->first_of_dim[d];
  int64_t r = (int64_t)(id & ((1ull << 56) - 1));
  *A = r / Td;
  *ti = cx->first_of_dim[d] + (int)(r % Td);
}

/* "whose pairing partner differs": the cell's pair in Gg is not its pair in Gf
 * (pairs up: the same cofacet slot; pairs down: the same facet). */
static int pair_differs(const cx_t* cx, const grad_t* Gf, const grad_t* Gg, int64_t A, int ti) {
  size_t i = (size_t)A * cx->T + ti;
  return Gf->up[i] != Gg->up[i] || Gf->dn[i] != Gg->dn[i];
}

/* The troublemaker of branch b of the original separatrices Sf: the
 * first cell along the branch, in its walk order, whose pairing in g differs from
 * the original pairing.  Cells examined (the critical cells at the ends are the
 * C-loop's business and are skipped):
 *   DESC (cells v0 e1 v1 ... v_min): the vertices before the minimum -- a
 *        0-dimensional troublemaker "paired with an incorrect 1-cell";
 *   ASC  (cells t0 c1 t1 c2 ...): the (top-1)-cells c_k -- the 2-cell (3D) "paired
 *        with an incorrect 3-cell", or in 2D the edge paired with a triangle;
 *   CONN (breadth-first event log): the triangles in queue order (the origin,
 *        then the logged triangles), and of each its facet edges in facet order,
 *        f-critical edges skipped -- the 1-cell "paired with an incorrect 2-cell".
 * Returns 1 and the cell, or 0. */
static int troublemaker(const cx_t* cx, const grad_t* Gf, const grad_t* Gg, const csr_t* S, int64_t b,
                        int64_t* tA, int* tt) {
  int64_t i0 = S->off[b], i1 = S->off[b + 1];
  int kind = S->kind[b];
  if (kind == KIND_DESC) {
    for (int64_t i = i0; i + 1 < i1; i += 2) {   /* v0, v1, ... ; the last cell is the minimum */
      int64_t A; int ti;
      id_to_cell(cx, S->cells[i], &A, &ti);
      if (pair_differs(cx, Gf, Gg, A, ti)) { *tA = A; *tt = ti; return 1; }
    }
    return 0;
  }
  if (kind == KIND_ASC) {
    for (int64_t i = i0 + 1; i < i1; i += 2) {   /* c1, c2, ... */
      int64_t A; int ti;
      id_to_cell(cx, S->cells[i], &A, &ti);
      if (pair_differs(cx, Gf, Gg, A, ti)) { *tA = A; *tt = ti; return 1; }
    }
    return 0;
  }
  /* CONN */
  int64_t B; int bt;
  id_to_cell(cx, S->origin[b], &B, &bt);
  for (int64_t i = i0 - 1; i < i1; i++) {
    if (i >= i0) {
      if ((int)(S->cells[i] >> 56) != 2) continue;      /* logged critical edge */
      id_to_cell(cx, S->cells[i], &B, &bt);
    }
    for (int k = 0; k < 3; k++) {
      int et;
      int64_t E = facet_cell(cx, B, bt, k, &et);
      if (is_crit(cx, Gf, E, et)) continue;
      if (pair_differs(cx, Gf, Gg, E, et)) { *tA = E; *tt = et; return 1; }
    }
  }
  return 0;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* Tier 3: does branch b of Sg reach the same extremum / the same multiset
 * of 1-saddles (connectors, reading A14) as branch b of Sf?  Both are traced from
 * the same critical cells (F = empty), so their branch lists correspond 1:1. */
static int same_ends(const csr_t* Sf, const csr_t* Sg, int64_t b) {
  if (Sf->kind[b] != KIND_CONN) return Sf->terminal[b] == Sg->terminal[b];
  int64_t n[2] = {0, 0};
  uint64_t* e[2];
  const csr_t* S[2] = {Sf, Sg};
  for (int s = 0; s < 2; s++) {
    int64_t i0 = S[s]->off[b], i1 = S[s]->off[b + 1];
    e[s] = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(i1 - i0 + 1));
    for (int64_t i = i0; i < i1; i++)
      if ((int)(S[s]->cells[i] >> 56) == 1) e[s][n[s]++] = S[s]->cells[i];
    qsort(e[s], (size_t)n[s], sizeof(uint64_t), cmp_u64);
  }
  int same = n[0] == n[1] && (n[0] == 0 || memcmp(e[0], e[1], sizeof(uint64_t) * (size_t)n[0]) == 0);
  free(e[0]); free(e[1]);
  return same;
}

typedef struct {
  int64_t c_rounds, s_rounds, troublemakers, tm_by_kind[3];  /* DESC ASC CONN */
  int64_t sep_branches, sep_cells;                           /* of the original field */
  int64_t tm_round1;                                         /* troublemakers of the first S-round */
  int64_t pad[7];
} or_sstats;

/* The DMTz workflow for tiers 1-4 (Fig. 2): C-loops and S-loops
 * alternate until no false critical cell and no false separatrix is left.
 * Synchronous rounds (reading A7, A17):
 *   every round recomputes the gradient of g;
 *   F != empty (tiers >= 3 use tier 2's F)  -> C-round: T = targets of F (R1-R3b);
 *   else, tier >= 3                          -> S-round: T = { R1 target of the
 *        troublemaker of b : b an original separatrix branch, checked when
 *        tier 4 -- always; tier 3 -- when b's traced end in g differs };
 *        T = empty -> done;
 *   else done;
 *   each non-lossless v in T takes one Eq. 2 step.
 * A troublemaker's target is "the vertex of its original partner it does not
 * share" (decrease j / k / l), i.e. rule R1 of the C-loop. */
int dmtz_oracle_preserve(const int64_t* dims, const float* f, const float* fhat, float xi,
                         int32_t q_max, int32_t q_cap, int32_t tier, int64_t max_rounds,
                         float* g_out, uint32_t* state_out, or_edit* edits, int64_t edits_capacity,
                         int64_t* n_edits, or_stats* stats, or_sstats* ss) {
  memset(stats, 0, sizeof *stats);
  memset(ss, 0, sizeof *ss);
  *n_edits = 0;
  int st = check_dims(dims);
  if (st) { stats->status = st; return st; }
  if (!(xi > 0.0f) || !isfinite(xi) || q_max < 0 || q_max > 30 || q_cap < 1 || q_cap > 65535 ||
      tier < 1 || tier > 5 || max_rounds < 0) {
    stats->status = OR_E_ARG; return OR_E_ARG;
  }
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  int64_t N = cx.N;
  for (int64_t v = 0; v < N; v++)
    if (!isfinite(f[v]) || !isfinite(fhat[v])) { stats->status = OR_E_NONFINITE; return OR_E_NONFINITE; }
  for (int64_t v = 0; v < N; v++)
    if (fhat[v] < lower_bound_ru(f[v], xi) || fhat[v] > upper_bound_rd(f[v], xi)) {
      stats->status = OR_E_BOUND; return OR_E_BOUND;
    }
  if (max_rounds == 0) max_rounds = N * (int64_t)(q_cap + 1);
  float step = ldexpf(xi, -q_max);
  float* lb = (float*)malloc(sizeof(float) * N);
  uint16_t* q = (uint16_t*)calloc(N, sizeof(uint16_t));
  uint8_t* lossless = (uint8_t*)calloc(N, 1);
  uint8_t* T = (uint8_t*)calloc(N, 1);
  grad_t Gf, Gg;
  if (!lb || !q || !lossless || !T || !grad_alloc(&cx, &Gf) || !grad_alloc(&cx, &Gg)) {
    stats->status = OR_E_ARG; return OR_E_ARG;
  }
  for (int64_t v = 0; v < N; v++) { lb[v] = lower_bound_ru(f[v], xi); g_out[v] = fhat[v]; }
  gradient(&cx, f, &Gf);
  if (tier == 5) {
    /* T5: "we edit the scalar values of all vertices that constitute the
     * critical cells in the original data to their lower bound f - xi before the
     * iterative process begins"; stored losslessly.  Then the tier-4 workflow. */
    for (int64_t A = 0; A < N; A++)
      for (int ti = 0; ti < cx.T; ti++) {
        if (!is_crit(&cx, &Gf, A, ti)) continue;
        int64_t vs[4];
        cell_vertices(&cx, A, ti, vs);
        for (int k = 0; k <= cx.t[ti].dim; k++) { g_out[vs[k]] = lb[vs[k]]; lossless[vs[k]] = 1; }
      }
    tier = 4;
  }
  const uint32_t all = KIND_DESC | KIND_ASC | KIND_CONN;
  csr_t Sf = {0}, Sg = {0};
  int status = OR_OK;
  if (tier >= 3) {
    status = trace_grad(&cx, &Gf, all, &Sf, 1);
    ss->sep_branches = Sf.nb;
    ss->sep_cells = Sf.nc;
  }
  const int ctier = tier >= 2 ? 2 : 1;
  for (int64_t round = 1; status == OR_OK; round++) {
    gradient(&cx, g_out, &Gg);
    memset(T, 0, N);
    int64_t kinds[8] = {0};
    int64_t nF = classify(&cx, f, &Gf, &Gg, ctier, T, kinds, NULL, NULL);
    if (nF < 0) { status = OR_E_INTERNAL; break; }
    if (round == 1) {
      stats->n_false_round0 = nF;
      memcpy(stats->false_by_kind_round0, kinds, sizeof kinds);
    }
    if (nF > 0) {
      ss->c_rounds++;
    } else if (tier >= 3) {
      if (tier == 3) {
        Sg.nb = Sg.nc = 0;
        status = trace_grad(&cx, &Gg, all, &Sg, 1);
        if (status) break;
        if (Sg.nb != Sf.nb) { status = OR_E_INTERNAL; break; }
      }
      int64_t ntm = 0, bad = 0;
      for (int64_t b = 0; b < Sf.nb; b++) {
        if (tier == 3 && same_ends(&Sf, &Sg, b)) continue;
        int64_t A; int ti;
        if (!troublemaker(&cx, &Gf, &Gg, &Sf, b, &A, &ti)) continue;
        int rule_unused;
        int64_t v = target_of(&cx, f, &Gf, &Gg, A, ti, 0, &rule_unused);
        if (v < 0) { bad++; continue; }
        T[v] = 1;
        ntm++;
        ss->tm_by_kind[Sf.kind[b] == KIND_DESC ? 0 : Sf.kind[b] == KIND_ASC ? 1 : 2]++;
      }
      if (bad) { status = OR_E_INTERNAL; break; }
      if (ntm == 0) break;
      if (ss->s_rounds == 0) ss->tm_round1 = ntm;
      ss->s_rounds++;
      ss->troublemakers += ntm;
    } else {
      break;
    }
    int changed = 0;
    for (int64_t v = 0; v < N; v++) {
      if (!T[v] || lossless[v]) continue;
      changed = 1;
      if (q[v] + 1 <= q_cap) {
        float s = (float)(q[v] + 1) * step;
        float gp = fhat[v] - s;
        if (gp >= lb[v]) { q[v]++; g_out[v] = gp; continue; }
      }
      g_out[v] = lb[v];
      lossless[v] = 1;
    }
    if (!changed) { status = OR_E_STUCK; break; }
    if (round == max_rounds) { status = OR_E_ITER_CAP; break; }
  }
  stats->rounds = ss->c_rounds;
  int64_t ne = 0;
  for (int64_t v = 0; v < N; v++) {
    if (state_out) state_out[v] = (uint32_t)q[v] | ((uint32_t)lossless[v] << 16);
    if (q[v] == 0 && !lossless[v]) continue;
    stats->n_edited++;
    if (lossless[v]) stats->n_lossless++; else stats->n_quantized++;
    if (edits && ne < edits_capacity) {
      edits[ne].v = (uint64_t)v; edits[ne].q = q[v]; edits[ne].lossless = lossless[v];
      edits[ne].pad = 0; edits[ne].value = g_out[v];
    }
    ne++;
  }
  *n_edits = ne;
  if (status == OR_OK && edits && ne > edits_capacity) status = OR_E_CAPACITY;
  stats->status = status;
  free(lb); free(q); free(lossless); free(T);
  grad_free(&Gf); grad_free(&Gg);
  csr_free(&Sf); csr_free(&Sg);
  return status;
}

/* ------------------------------------------------------------------------- */
/* 0-dimensional persistence of the sublevel filtration (tier 5's check,       */
/* P:143 "persistence diagram"): vertices in SoS order, union-find   */
/* over the edges of the complex, elder rule.  pairs[2k], pairs[2k+1] = (birth  */
/* vertex, death vertex) of each finite pair; returns the number of pairs.      */
/* ------------------------------------------------------------------------- */
static int64_t uf_find(int64_t* parent, int64_t x) {
  while (parent[x] != x) { parent[x] = parent[parent[x]]; x = parent[x]; }
  return x;
}
static const float* g_sort_f;
static int cmp_sos(const void* a, const void* b) {
  int64_t u = *(const int64_t*)a, v = *(const int64_t*)b;
  return sos_less(g_sort_f, u, v) ? -1 : sos_less(g_sort_f, v, u) ? 1 : 0;
}
int64_t dmtz_oracle_persistence0(const int64_t* dims, const float* field, int64_t* pairs, int64_t cap) {
  if (check_dims(dims)) return -1;
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  int64_t N = cx.N;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * N);
  int64_t* parent = (int64_t*)malloc(sizeof(int64_t) * N);
  int64_t* root_birth = (int64_t*)malloc(sizeof(int64_t) * N);  /* oldest vertex of a root's component */
  uint8_t* in = (uint8_t*)calloc(N, 1);
  for (int64_t v = 0; v < N; v++) { order[v] = v; parent[v] = v; root_birth[v] = v; }
  g_sort_f = field;
  qsort(order, (size_t)N, sizeof(int64_t), cmp_sos);
  int64_t np = 0;
  for (int64_t i = 0; i < N; i++) {
    int64_t v = order[i];
    in[v] = 1;
    co_t c = coords(&cx, v);
    const ctype_t* vt = &cx.t[0];
    for (int s = 0; s < vt->nlink; s++) {        /* edges {v, w}: the vertex's link */
      int64_t x = c.x + vt->link[s][0], y = c.y + vt->link[s][1], z = c.z + vt->link[s][2];
      if (!inside(&cx, x, y, z)) continue;
      int64_t w = vid(&cx, x, y, z);
      if (!in[w]) continue;
      int64_t a = uf_find(parent, v), b = uf_find(parent, w);
      if (a == b) continue;
      int64_t ba = root_birth[a], bb = root_birth[b];
      /* elder rule: the younger component (later birth) dies at v */
      int64_t young = sos_less(field, ba, bb) ? b : a, old = young == a ? b : a;
      if (root_birth[young] != v) {              /* v's own singleton merging is not a pair */
        if (np < cap) { pairs[2 * np] = root_birth[young]; pairs[2 * np + 1] = v; }
        np++;
      }
      parent[young] = old;
    }
  }
  free(order); free(parent); free(root_birth); free(in);
  return np;
}

/* Test interface for the exhaustive-order pins (tests/test_oracle_orders.py): the
 * literal gradient of each of nf fields on one tiny grid (<= 16 vertices), as the list
 * of pairs (vertex-id bitmask of the cell, bitmask of its partner cofacet) sorted by
 * the cell's bitmask; out[f * cap ...] holds field f's pairs, count[f] their number. */
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}
int dmtz_oracle_pairs_batch(const int64_t* dims, int64_t nf, const float* fields, uint32_t* out, int32_t* count,
                            int32_t cap) {
  int st = check_dims(dims);
  if (st) return st;
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  if (cx.N > 16) return OR_E_ARG;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : bad)
  for (int64_t k = 0; k < nf; k++) {
    grad_t G;
    if (!grad_alloc(&cx, &G)) { bad++; continue; }
    gradient(&cx, fields + k * cx.N, &G);
    int n = 0;
    uint32_t* o = out + k * (int64_t)cap;
    for (int64_t A = 0; A < cx.N; A++)
      for (int ti = 0; ti < cx.T; ti++) {
        int s = G.up[(size_t)A * cx.T + ti];
        if (s < 0) continue;
        int64_t vs[5];
        cell_vertices(&cx, A, ti, vs);
        uint32_t cm = 0;
        for (int i = 0; i <= cx.t[ti].dim; i++) cm |= 1u << vs[i];
        co_t a = coords(&cx, A);
        const ctype_t* ct = &cx.t[ti];
        int64_t w = vid(&cx, a.x + ct->link[s][0], a.y + ct->link[s][1], a.z + ct->link[s][2]);
        if (n < cap) o[n] = (cm << 16) | cm | (1u << w);
        n++;
      }
    if (n > cap) { bad++; n = cap; }
    qsort(o, (size_t)n, sizeof(uint32_t), cmp_u32);
    count[k] = n;
    grad_free(&G);
  }
  return bad ? OR_E_CAPACITY : OR_OK;
}

int dmtz_oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Number of cells of each dimension of the grid complex (for the closed-form
 * count pins S:60-62 and the Euler characteristic). */
int dmtz_oracle_cell_counts(const int64_t* dims, int64_t* counts /* [4] */) {
  int st = check_dims(dims);
  if (st) return st;
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  for (int d = 0; d < 4; d++) counts[d] = 0;
  for (int64_t A = 0; A < cx.N; A++)
    for (int ti = 0; ti < cx.T; ti++)
      if (cell_exists(&cx, A, ti)) counts[cx.t[ti].dim]++;
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* One synchronous C-loop round on a z-slab (for the multi-rank tests).        */
/* The local grid is the slab plus halo planes; only cells anchored in local   */
/* planes [az0, az1) are classified and only targets in planes [oz0, oz1)      */
/* (the owned planes) are edited.  Same literal rules as dmtz_oracle_correct.  */
/* out = {n_false (anchored in owned planes), n_changed, n_targets}; kinds[8]. */
/* ------------------------------------------------------------------------- */
int dmtz_oracle_slab_round(const int64_t* dims, const float* f, const float* fhat, float xi, int32_t q_max,
                           int32_t q_cap, int32_t tier, int64_t az0, int64_t az1, int64_t oz0, int64_t oz1,
                           float* g, uint32_t* state, int64_t* out, int64_t* kinds) {
  int st = check_dims(dims);
  if (st) return st;
  cx_t cx; build_complex(&cx, dims[0], dims[1], dims[2]);
  int64_t N = cx.N, plane = cx.n[0] * cx.n[1];
  grad_t Gf, Gg;
  uint8_t* T = (uint8_t*)calloc(N, 1);
  if (!T || !grad_alloc(&cx, &Gf) || !grad_alloc(&cx, &Gg)) return OR_E_ARG;
  gradient(&cx, f, &Gf);
  gradient(&cx, g, &Gg);
  int64_t nF = 0, bad = 0;
  for (int64_t A = az0 * plane; A < az1 * plane && A < N; A++) {
    for (int ti = 0; ti < cx.T; ti++) {
      int d = cx.t[ti].dim;
      if (tier == 1 && d != 0 && d != cx.top) continue;
      if (!cell_exists(&cx, A, ti)) continue;
      int cf = is_crit(&cx, &Gf, A, ti), cg = is_crit(&cx, &Gg, A, ti);
      if (cf == cg) continue;
      if (A >= oz0 * plane && A < oz1 * plane) {  /* each anchor is counted by its owner */
        nF++;
        kinds[kind_of(&cx, d, cf)]++;
      }
      int rule_unused;
      int64_t v = target_of(&cx, f, &Gf, &Gg, A, ti, cf, &rule_unused);
      if (v < 0) { bad++; continue; }
      if (v >= oz0 * plane && v < oz1 * plane) T[v] = 1;
    }
  }
  float step = ldexpf(xi, -q_max);
  int64_t changed = 0, targets = 0;
  for (int64_t v = 0; v < N; v++) {
    if (!T[v]) continue;
    targets++;
    uint32_t q = state[v] & 0xFFFFu, ll = state[v] >> 16;
    if (ll) continue;
    changed++;
    float lb = lower_bound_ru(f[v], xi);
    if ((int64_t)q + 1 <= q_cap) {
      float s = (float)(q + 1) * step;
      float gp = fhat[v] - s;
      if (gp >= lb) { state[v] = q + 1; g[v] = gp; continue; }
    }
    g[v] = lb;
    state[v] = q | (1u << 16);
  }
  out[0] = nF; out[1] = changed; out[2] = targets;
  free(T); grad_free(&Gf); grad_free(&Gg);
  return bad ? OR_E_INTERNAL : OR_OK;
}
