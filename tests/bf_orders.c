/*
 * tests/bf_orders.c -- an independent brute force of the discrete gradient on tiny
 * grids, for the exhaustive-order pins (tests/test_oracle_orders.py).  TEST ONLY.
 *
 * Shares nothing with oracle/ or the CUDA path.  The complex is built from its
 * definition as a simplicial complex: every unit cube (square)
 * is cut into the D! Kuhn simplices  b, b+e_p1, b+e_p1+e_p2, ...  (one per axis
 * permutation p); the cells are all non-empty faces of those simplices, held as
 * bitmasks of vertex ids (<= 16 vertices).  The pairing is the rule of P:84-92 /
 * P:152-155 read literally: for d = 0, 1, ..., a d-cell a not yet paired with a facet
 * is paired with the cofacet b of least key among P_a = { b : b minus its SoS-lowest
 * vertex = a }, where a cell's key is its vertex list sorted descending in the SoS
 * order (value, then vertex id) and keys compare lexicographically (Eq. 1).
 *
 * bf_pairs(nx, ny, nz, nf, fields, out, count, cap): for each field, its pairs as
 * (cell mask << 16) | cofacet mask, sorted ascending.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const float* F;

static int sos_less(int u, int v) { return F[u] < F[v] || (F[u] == F[v] && u < v); }

/* vertices of mask m sorted descending in SoS order */
static int key_of(uint32_t m, int* key) {
  int n = 0;
  for (int v = 0; v < 32; v++)
    if (m >> v & 1u) key[n++] = v;
  for (int i = 1; i < n; i++)
    for (int j = i; j > 0 && sos_less(key[j - 1], key[j]); j--) {
      int t = key[j]; key[j] = key[j - 1]; key[j - 1] = t;
    }
  return n;
}

static int key_less(uint32_t a, uint32_t b) {
  int ka[8], kb[8];
  int n = key_of(a, ka);
  key_of(b, kb);
  for (int i = 0; i < n; i++) {
    if (ka[i] == kb[i]) continue;
    return sos_less(ka[i], kb[i]);
  }
  return 0;
}

static int lowest(uint32_t m) {
  int best = -1;
  for (int v = 0; v < 32; v++)
    if (m >> v & 1u)
      if (best < 0 || sos_less(v, best)) best = v;
  return best;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

int bf_pairs(int nx, int ny, int nz, int64_t nf, const float* fields, uint32_t* out, int32_t* count, int32_t cap) {
  const int D = nz == 1 ? 2 : 3, N = nx * ny * nz;
  if (N > 16) return 1;
  uint8_t* is_cell = (uint8_t*)calloc(1u << N, 1);
  /* maximal simplices: cube base b, axis permutation */
  int perms[6][3], np = 0;
  for (int a = 0; a < D; a++)
    for (int b = 0; b < D; b++)
      for (int c = 0; c < (D == 3 ? 3 : 1); c++) {
        if (a == b || (D == 3 && (a == c || b == c))) continue;
        perms[np][0] = a; perms[np][1] = b; perms[np][2] = c; np++;
      }
  for (int z = 0; z < (D == 3 ? nz - 1 : 1); z++)
    for (int y = 0; y < ny - 1; y++)
      for (int x = 0; x < nx - 1; x++)
        for (int p = 0; p < np; p++) {
          int c[3] = {x, y, z}, vs[4];
          vs[0] = c[0] + nx * (c[1] + ny * c[2]);
          for (int k = 0; k < D; k++) {
            c[perms[p][k]]++;
            vs[k + 1] = c[0] + nx * (c[1] + ny * c[2]);
          }
          for (int sub = 1; sub < (1 << (D + 1)); sub++) {  /* every face */
            uint32_t m = 0;
            for (int k = 0; k <= D; k++)
              if (sub >> k & 1) m |= 1u << vs[k];
            is_cell[m] = 1;
          }
        }
  uint32_t* cells = (uint32_t*)malloc(sizeof(uint32_t) << N);
  int nc = 0;
  for (uint32_t m = 1; m < (1u << N); m++)
    if (is_cell[m]) cells[nc++] = m;
  uint32_t* partner = (uint32_t*)malloc(sizeof(uint32_t) << N);
  int bad = 0;
  for (int64_t f = 0; f < nf; f++) {
    F = fields + f * N;
    memset(partner, 0, sizeof(uint32_t) << N);
    int n = 0;
    uint32_t* o = out + f * (int64_t)cap;
    for (int d = 0; d < D; d++)
      for (int i = 0; i < nc; i++) {
        uint32_t a = cells[i];
        if (__builtin_popcount(a) != d + 1 || partner[a]) continue;
        uint32_t best = 0;
        for (int v = 0; v < N; v++) {
          if (a >> v & 1u) continue;
          uint32_t b = a | (1u << v);
          if (!is_cell[b]) continue;
          if ((b & ~(1u << lowest(b))) != a) continue;  /* G0(b) = b minus its lowest vertex */
          if (!best || key_less(b, best)) best = b;
        }
        if (!best) continue;
        partner[a] = best;
        partner[best] = a;
        if (n < cap) o[n] = (a << 16) | best;
        n++;
      }
    if (n > cap) { bad = 1; n = cap; }
    qsort(o, (size_t)n, sizeof(uint32_t), cmp_u32);
    count[f] = n;
  }
  free(is_cell); free(cells); free(partner);
  return bad;
}
