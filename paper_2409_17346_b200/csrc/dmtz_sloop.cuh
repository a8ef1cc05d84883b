// dmtz_sloop.cuh -- S-loop rounds for sm_100a.
//
// The separatrices of the ORIGINAL field f are traced once (dmtz_trace.cuh) into a
// CSR that stays resident.  An S-round then asks, for every branch b of that CSR,
// for its TROUBLEMAKER: the first cell along b (walk order) whose pairing in the
// current gradient of g differs from its pairing in f, and marks the
// vertex of the cell's original partner that the cell does not share (P:235-243:
// "decrease j" / "decrease k" / "decrease l" -- the C-loop's rule R1) in the
// round's target bitmap.  k_edit_rows then applies Eq. 2 to the marked vertices.
//
// Cells examined (as in oracle/dmtz_oracle.c troublemaker()):
//   DESC  cells v0 e1 v1 ... v_min : the vertices before the minimum;
//   ASC   cells t0 c1 t1 c2 ...    : the (top-1)-cells c_k;
//   CONN  event log of the BFS     : the triangles in queue order (the origin, then the
//         logged triangles), and of each its 3 facet edges in facet order, f-critical
//         edges skipped.
// "First" is found in two steps: k_tm_cells keeps one mismatch bit per CSR cell
// (re-evaluating only cells whose codes changed since the last S-round), and
// k_tm_targets (one thread per branch) takes the first set bit of its range.  Which
// cells are examined is precomputed once per CSR cell (k_cell_desc_*).
#pragma once

#include "dmtz_kernels.cuh"
#include "dmtz_sweep.cuh"
#include "dmtz_trace.cuh"

namespace dmtz {

// ----------------------------------------------------------------------------- per-cell descriptors
// desc[i] (one byte per CSR cell, built once): 0 = not examined; else the branch
// kind (1 DESC vertex before the minimum, 2 ASC (top-1)-cell, 4 CONN logged
// triangle).  Branches of at most 32 cells are done by their own thread; longer ones
// are listed (long_list) and done by a warp each.
__device__ __forceinline__ uint8_t cell_desc(int k, int64_t pos, int64_t len, uint64_t id) {
  if (k == 1) return (!(pos & 1) && pos + 1 < len) ? 1 : 0;
  if (k == 2) return (pos & 1) ? 2 : 0;
  return (id >> 56) == 2 ? 4 : 0;
}

template <int D>
__device__ __forceinline__ void put_desc(int k, int64_t pos, int64_t len, uint64_t id, uint8_t* desc, uint32_t* anc,
                                         int64_t i);

template <int D>
__global__ void k_cell_desc_short(const long long* __restrict__ off, const uint8_t* __restrict__ kind,
                                  const uint64_t* __restrict__ cells, int64_t nb, uint8_t* __restrict__ desc,
                                  uint32_t* __restrict__ anc, uint32_t* __restrict__ long_list,
                                  unsigned long long* __restrict__ n_long) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = off[b], i1 = off[b + 1];
    const int k = kind[b];
    if (i1 - i0 <= 32) {
      for (int64_t i = i0; i < i1; i++) put_desc<D>(k, i - i0, i1 - i0, cells[i], desc, anc, i);
    } else {
      long_list[atomicAdd(n_long, 1ull)] = (uint32_t)b;
    }
  }
}

template <int D>
__global__ void k_cell_desc_long(const long long* __restrict__ off, const uint8_t* __restrict__ kind,
                                 const uint64_t* __restrict__ cells, const uint32_t* __restrict__ long_list,
                                 const unsigned long long* __restrict__ n_long, uint8_t* __restrict__ desc,
                                 uint32_t* __restrict__ anc) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)*n_long;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t b = long_list[w];
    const int64_t i0 = off[b], i1 = off[b + 1];
    const int k = kind[b];
    for (int64_t i = i0 + lane; i < i1; i += 32) put_desc<D>(k, i - i0, i1 - i0, cells[i], desc, anc, i);
  }
}

// ----------------------------------------------------------------------------- pairing comparison
// The facet of cell (A, t) its code set points at it (down-pair), or -1.
template <int D>
__device__ __forceinline__ int down_facet(const void* codes, const Grid& g, int64_t A, int t) {
  for (int j = 0; j < t_nfacet<D>(t); j++) {
    const int dm = t_facet<D>(t, j, 0), ft = t_facet<D>(t, j, 1), sl = t_facet<D>(t, j, 2);
    if (field_of<D>(code_at<D>(codes, A + mask_delta(g, dm)), ft) == (uint32_t)sl) return j;
  }
  return -1;
}

// Does cell (A, t)'s partner in g differ from its partner in f?  (pairs up: the
// cofacet slot; pairs down: the facet.)  The cell exists (it lies on a path of f).
template <int D>
__device__ __forceinline__ bool pair_differs(const void* cf, const void* cg, const Grid& g, int64_t A, int t) {
  if (t_dim<D>(t) < Tr<D>::TOP) {
    const uint32_t uf = field_of<D>(code_at<D>(cf, A), t), ug = field_of<D>(code_at<D>(cg, A), t);
    if (uf != ug) return true;
    if (uf != (uint32_t)t_none<D>(t)) return false;  // paired up with the same cofacet in both
  }
  return t_dim<D>(t) > 0 && down_facet<D>(cf, g, A, t) != down_facet<D>(cg, g, A, t);
}

// vertex index of the R1 target of cell (A, t): the vertex of its f-partner it does not share
template <int D>
__device__ __forceinline__ int64_t r1_target(const void* cf, const Grid& g, int64_t A, int t) {
  if (t_dim<D>(t) < Tr<D>::TOP) {
    const uint32_t s = field_of<D>(code_at<D>(cf, A), t);
    if (s != (uint32_t)t_none<D>(t))
      return A + t_link<D>(t, (int)s, 0) + t_link<D>(t, (int)s, 1) * g.sy + t_link<D>(t, (int)s, 2) * g.sz;
  }
  const int j = down_facet<D>(cf, g, A, t);
  if (j < 0) return -1;
  return A + mask_delta(g, t_vmask<D>(t, t_facet<D>(t, j, 3)));  // facet j omits vertex t_facet(t, j, 3)
}

// ----------------------------------------------------------------------------- per-cell mismatch bits
// mbits (one bit per CSR cell, persistent across S-rounds): the cell is examined
// (see the header) and its pairing in g differs from f's -- for a CONN triangle:
// one of its facet edges that is not critical in f does.  A cell's bit depends
// only on the codes of g at a few anchors (DESC vertex v: v; ASC cell: its anchor;
// CONN triangle at B: each facet edge's anchor and second vertex, all in
// B + {0,1,2}^3), so after the first S-round (full = 1) only cells whose anchor has
// a changed code in that window since the last S-round (sdirty, fed by every round's
// changed-code bits, dilated by k_sdirty_dilate) are re-evaluated; the others keep
// their bit exactly.
// id_cell with compile-time divisors (multiply-high instead of a 64-bit division)
template <int D>
__device__ __forceinline__ void id_cell_fast(uint64_t id, int64_t& a, int& t) {
  const int d = (int)(id >> 56);
  const uint64_t r = id & ((1ull << 56) - 1);
  uint64_t q;
  if (D == 3) q = d == 0 ? r : d == 1 ? r / 7u : d == 2 ? r / 12u : r / 6u;
  else q = d == 0 ? r : d == 1 ? r / 3u : r / 2u;
  a = (int64_t)q;
  t = t_first_of_dim_c<D>(d) + (int)(r - q * (uint64_t)types_of_dim<D>(d));
}

// desc[i] and, for examined cells, anc[i] = the cell's anchor (grids below 2^32 vertices)
template <int D>
__device__ __forceinline__ void put_desc(int k, int64_t pos, int64_t len, uint64_t id, uint8_t* desc, uint32_t* anc,
                                         int64_t i) {
  const uint8_t d = cell_desc(k, pos, len, id);
  desc[i] = d;
  if (d) {
    int64_t A; int t;
    id_cell_fast<D>(id, A, t);
    anc[i] = (uint32_t)A;
  }
}

__device__ __forceinline__ bool dbit(const uint32_t* __restrict__ d, int64_t v) {
  return (__ldg(d + (v >> 5)) >> (v & 31)) & 1u;
}

template <int D>
__device__ __forceinline__ bool conn_tri_differs(const void* cf, const void* cg, const uint32_t* __restrict__ crit_f,
                                                 const Grid& g, int64_t B, int bt, int* jfirst) {
  for (int j = 0; j < 3; j++) {
    const int64_t E = B + mask_delta(g, t_facet<D>(bt, j, 0));
    const int et = t_facet<D>(bt, j, 1);
    if ((__ldg(crit_f + E) >> et) & 1u) continue;
    if (pair_differs<D>(cf, cg, g, E, et)) { *jfirst = j; return true; }
  }
  return false;
}

// A warp takes TM_U consecutive mbits words (32 x TM_U cells, one per lane per word)
// and issues every load of the batch before using any (the kernel is bound by the
// latency of its dependent loads otherwise).
constexpr int TM_U = 4;
template <int D>
__global__ void __launch_bounds__(256)
k_tm_cells(const uint64_t* __restrict__ cells, int64_t n_cells, const uint8_t* __restrict__ desc,
           const uint32_t* __restrict__ anc, const void* __restrict__ cf, const void* __restrict__ cg,
           const uint32_t* __restrict__ crit_f, Grid g, const uint32_t* __restrict__ sdirty /* dilated */, int full,
           uint32_t* __restrict__ mbits, Counters* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * TM_U;  // first word of the warp
  int k[TM_U];
  uint32_t a[TM_U];
#pragma unroll
  for (int u = 0; u < TM_U; u++) {
    const int64_t i = (w0 + u) * 32 + lane;
    k[u] = i < n_cells ? __ldg(desc + i) : 0;
  }
#pragma unroll
  for (int u = 0; u < TM_U; u++) {
    const int64_t i = (w0 + u) * 32 + lane;
    a[u] = k[u] ? __ldg(anc + i) : 0u;
  }
  bool dirty[TM_U];
#pragma unroll
  for (int u = 0; u < TM_U; u++)
    dirty[u] = full ? ((w0 + u) * 32 + lane < n_cells) : (k[u] && dbit(sdirty, (int64_t)a[u]));
  unsigned long long nre = 0;
#pragma unroll
  for (int u = 0; u < TM_U; u++) {
    bool mis = false;
    if (k[u] && dirty[u]) {
      nre++;
      int64_t A; int t;
      id_cell_fast<D>(__ldg(cells + (w0 + u) * 32 + lane), A, t);
      int j;
      mis = k[u] == 4 ? conn_tri_differs<D>(cf, cg, crit_f, g, A, t, &j) : pair_differs<D>(cf, cg, g, A, t);
    }
    const unsigned dm = __ballot_sync(0xffffffffu, dirty[u]), mm = __ballot_sync(0xffffffffu, mis);
    if (lane == 0 && dm) {
      uint32_t* w = mbits + w0 + u;
      *w = (*w & ~dm) | mm;
    }
  }
  warp_add(&cnt->pad[7], nre);
}

// first set bit of mbits in [i0, i1), or -1
__device__ __forceinline__ int64_t first_bit(const uint32_t* __restrict__ mbits, int64_t i0, int64_t i1) {
  for (int64_t w = i0 >> 5; (w << 5) < i1; w++) {
    uint32_t m = mbits[w];
    const int64_t lo = w << 5;
    if (lo < i0) m &= ~0u << (i0 - lo);
    if (lo + 32 > i1) m &= (i1 - lo) >= 32 ? ~0u : ((1u << (i1 - lo)) - 1u);
    if (m) return lo + __ffs(m) - 1;
  }
  return -1;
}

// ----------------------------------------------------------------------------- per-branch targets
// One thread per branch: its troublemaker = the first set mismatch bit (CONN: the
// origin's facets first), its target -> the round's target bitmap.
// cnt->pad[3] += troublemakers, cnt->pad[4 + kind index] += per kind.
// flag (tier 3, else nullptr): only branches with flag[b] != 0 count.
template <int D>
__global__ void k_tm_targets(const uint64_t* __restrict__ cells, const long long* __restrict__ off,
                             const uint8_t* __restrict__ kind, const uint64_t* __restrict__ origin, int64_t nb,
                             const void* __restrict__ cf, const void* __restrict__ cg,
                             const uint32_t* __restrict__ crit_f, Grid g, RowGeom rg,
                             const uint32_t* __restrict__ mbits, const uint8_t* __restrict__ flag,
                             const uint32_t* __restrict__ sdirty, int full, uint8_t* __restrict__ omis,
                             uint32_t* __restrict__ tbits, Counters* __restrict__ cnt) {
  unsigned long long ntm = 0, nk[3] = {0, 0, 0}, bad = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int k = kind[b];
    int64_t A = -1;
    int t = 0;
    if (k == 4) {
      int64_t B; int bt;
      id_cell_fast<D>(origin[b], B, bt);
      int j = -1;
      // the origin's facets come first; their mismatch (omis) is kept like mbits
      bool om;
      if (full || dbit(sdirty, B)) {
        om = conn_tri_differs<D>(cf, cg, crit_f, g, B, bt, &j);
        omis[b] = om;
      } else {
        om = omis[b] != 0;
        if (om && !conn_tri_differs<D>(cf, cg, crit_f, g, B, bt, &j)) { bad++; continue; }
      }
      if (flag && !flag[b]) continue;  // tier 3: this branch ends where it ends in f
      if (!om) {
        const int64_t i = first_bit(mbits, off[b], off[b + 1]);
        if (i < 0) continue;
        id_cell_fast<D>(cells[i], B, bt);
        if (!conn_tri_differs<D>(cf, cg, crit_f, g, B, bt, &j)) { bad++; continue; }
      }
      A = B + mask_delta(g, t_facet<D>(bt, j, 0));
      t = t_facet<D>(bt, j, 1);
    } else {
      if (flag && !flag[b]) continue;  // tier 3: this branch ends where it ends in f
      const int64_t i = first_bit(mbits, off[b], off[b + 1]);
      if (i < 0) continue;
      id_cell_fast<D>(cells[i], A, t);
    }
    const int64_t v = r1_target<D>(cf, g, A, t);
    if (v < 0) { bad++; continue; }
    int64_t x, y, z;
    coords_of(g, v, x, y, z);
    atomicOr(tbits + dword_index(g, rg, y, z, x >> 5), 1u << (x & 31));
    ntm++;
    nk[k == 1 ? 0 : k == 2 ? 1 : 2]++;
  }
  warp_add(&cnt->pad[3], ntm);
  warp_add(&cnt->pad[4], nk[0]);
  warp_add(&cnt->pad[5], nk[1]);
  warp_add(&cnt->pad[6], nk[2]);
  warp_add(&cnt->n_internal, bad);
}

// dil(A) = OR of changed(A + dx + dy*nx + dz*nx*ny) over (dx, dy, dz) in {0,1,2}^3, in the
// linear bit space (offsets that wrap across a row or plane only add positions): a
// superset of every anchor a cell's mismatch bit reads (DESC/ASC: the cell's anchor;
// CONN: facet edges at A + {0,1}^3 and their second vertices), so one bit decides
// whether a cell must be re-evaluated.
__global__ void k_sdirty_dilate(const uint32_t* __restrict__ chg, int64_t nwords, int64_t sy, int64_t sz,
                                uint32_t* __restrict__ dil) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t acc = 0;
#pragma unroll
    for (int dz = 0; dz < 3; dz++)
#pragma unroll
      for (int dy = 0; dy < 3; dy++) {
        const int64_t o = dy * sy + dz * sz;       // bits w*32 + o + (0..2) + lane
        const int64_t b = w * 32 + o;
        const int64_t q = b >> 5;
        const int r = (int)(b & 31);
        const uint32_t lo = q < nwords ? __ldg(chg + q) : 0u, hi = q + 1 < nwords ? __ldg(chg + q + 1) : 0u;
        const uint32_t h2 = q + 1 < nwords && r > 29 ? (q + 2 < nwords ? __ldg(chg + q + 2) : 0u) : 0u;
        // 64-bit window starting at bit b: bits b .. b + 63 (enough for + 0..2 when r <= 29)
        const unsigned long long win = ((unsigned long long)hi << 32 | lo) >> r;
        const unsigned long long ext = r > 29 ? (unsigned long long)h2 << (64 - r) : 0ull;
        const unsigned long long x = win | ext;
        acc |= (uint32_t)(x | (x >> 1) | (x >> 2));
      }
    dil[w] = acc;
  }
}

// changed-code bits of a round (row-padded words) -> the linear per-anchor bitmap sdirty
__global__ void k_sdirty_or(const uint32_t* __restrict__ ebits, int64_t nwords, Grid g, RowGeom rg,
                            uint32_t* __restrict__ sdirty) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = ebits[w];
    if (!m) continue;
    const int64_t row = w / rg.wpr, c = w - row * rg.wpr;
    const int64_t v0 = row * g.nx + c * 32;
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      const int64_t v = v0 + bit;
      atomicOr(sdirty + (v >> 5), 1u << (v & 31));
    }
  }
}

}  // namespace dmtz

namespace dmtz {

// ----------------------------------------------------------------------------- tier 3
// flag[b] = 1 iff branch b of the trace of g ends differently from branch b of the
// trace of f: DESC / ASC -- another terminal; CONN -- another multiset of
// reached 1-saddles (reading A14).  One warp per branch; connector multisets are
// compared by counting each reached edge's occurrences in both logs (shared-memory
// copies when both have at most T3_SMEM edges, else straight from the CSRs).
constexpr int T3_WARPS = 4, T3_SMEM = 256;
__global__ void __launch_bounds__(T3_WARPS * 32)
k_t3_flags(const long long* __restrict__ foff, const uint64_t* __restrict__ fcells,
           const uint64_t* __restrict__ fterm, const uint8_t* __restrict__ kind, const long long* __restrict__ goff,
           const uint64_t* __restrict__ gcells, const uint64_t* __restrict__ gterm, int64_t nb,
           uint8_t* __restrict__ flag) {
  __shared__ unsigned long long sl[T3_WARPS][2][T3_SMEM];
  __shared__ int sn[T3_WARPS][2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (kind[b] != 4) {
      if (lane == 0) flag[b] = fterm[b] != gterm[b];
      continue;
    }
    const int64_t s0[2] = {foff[b], goff[b]}, s1[2] = {foff[b + 1], goff[b + 1]};
    const uint64_t* cs[2] = {fcells, gcells};
    if (lane < 2) sn[wib][lane] = 0;
    __syncwarp();
    int cnt[2];
    for (int h = 0; h < 2; h++) {
      int c = 0;
      for (int64_t i = s0[h] + lane; i < s1[h]; i += 32) {
        const uint64_t id = cs[h][i];
        if ((id >> 56) != 1) continue;
        c++;
        const int p = atomicAdd(&sn[wib][h], 1);
        if (p < T3_SMEM) sl[wib][h][p] = id;
      }
      cnt[h] = __reduce_add_sync(0xffffffffu, c);
    }
    __syncwarp();
    bool differ = cnt[0] != cnt[1];
    if (!differ && cnt[0] > 0) {
      const bool smem = cnt[0] <= T3_SMEM;
      bool bad = false;
      if (smem) {
        for (int i = lane; i < cnt[0]; i += 32) {
          const unsigned long long x = sl[wib][0][i];
          int a = 0, c = 0;
          for (int j = 0; j < cnt[0]; j++) {
            a += sl[wib][0][j] == x;
            c += sl[wib][1][j] == x;
          }
          bad |= a != c;
        }
      } else {
        for (int64_t i = s0[0] + lane; i < s1[0]; i += 32) {
          const uint64_t x = fcells[i];
          if ((x >> 56) != 1) continue;
          int64_t a = 0, c = 0;
          for (int64_t j = s0[0]; j < s1[0]; j++) a += fcells[j] == x;
          for (int64_t j = s0[1]; j < s1[1]; j++) c += gcells[j] == x;
          bad |= a != c;
        }
      }
      differ = __any_sync(0xffffffffu, bad);
    }
    if (lane == 0) flag[b] = differ ? 1 : 0;
    __syncwarp();
  }
}

}  // namespace dmtz

namespace dmtz {

// Tier 5: every vertex of every critical cell of f goes to its lower
// bound before the loop, stored losslessly.  Several anchors may write the
// same vertex: the writes are identical.
template <int D>
__global__ void k_t5_clamp(const uint32_t* __restrict__ crit_f, const float* __restrict__ lb, float* __restrict__ gf,
                           uint32_t* __restrict__ state, Grid g) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.N; v += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = crit_f[v];
    while (m) {
      const int t = __ffs(m) - 1;
      m &= m - 1;
      for (int k = 0; k < t_nv<D>(t); k++) {
        const int64_t w = v + mask_delta(g, t_vmask<D>(t, k));
        gf[w] = lb[w];
        state[w] = 1u << 16;
      }
    }
  }
}

}  // namespace dmtz

namespace dmtz {

// ----------------------------------------------------------------------------- tier 3, candidates
// A branch whose f-path shows no mismatch (no troublemaker) follows the same path in g
// and ends the same; only the others (the candidates) are traced in g.
// cidx[b] = 1 for a candidate (then exclusive-scanned into its index); cnt->pad[4 + kind
// index] counts them per kind.
// With the end cache (t3st != nullptr): a candidate whose cached end comparison is still
// valid takes it (flag[b] = t3st[b] == 2) and is not traced; *hits counts them.
template <int D>
__global__ void k_t3_cand(const uint64_t* __restrict__ cells, const long long* __restrict__ off,
                          const uint8_t* __restrict__ kind, const uint64_t* __restrict__ origin, int64_t nb,
                          const void* __restrict__ cf, const void* __restrict__ cg, const uint32_t* __restrict__ crit_f,
                          Grid g, const uint32_t* __restrict__ mbits, long long* __restrict__ cidx,
                          Counters* __restrict__ cnt, const uint8_t* __restrict__ t3st, uint8_t* __restrict__ flag,
                          unsigned long long* __restrict__ hits) {
  unsigned long long nk[3] = {0, 0, 0}, nh = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x) {
    if (b == nb) { cidx[nb] = 0; continue; }
    const int k = kind[b];
    bool c = first_bit(mbits, off[b], off[b + 1]) >= 0;
    if (!c && k == 4) {
      int64_t B; int bt; int j;
      id_cell_fast<D>(origin[b], B, bt);
      c = conn_tri_differs<D>(cf, cg, crit_f, g, B, bt, &j);
    }
    if (c && t3st) {
      const uint8_t st = t3st[b];
      if (st) {
        flag[b] = st == 2 ? 1 : 0;
        nh++;
        c = false;
      }
    }
    cidx[b] = c ? 1 : 0;
    if (c) nk[k == 1 ? 0 : k == 2 ? 1 : 2]++;
  }
  if (t3st) warp_add(hits, nh);
  warp_add(&cnt->pad[4], nk[0]);
  warp_add(&cnt->pad[5], nk[1]);
  warp_add(&cnt->pad[6], nk[2]);
}

// candidate i = cidx[b] (after the scan): its origin, kind, branch index j (DESC: which
// endpoint; ASC: the raw cofacet slot of its first cell; CONN: 0) and cmap[i] = b
template <int D>
__global__ void k_t3_fill(const uint64_t* __restrict__ cells, const long long* __restrict__ off,
                          const uint8_t* __restrict__ kind, const uint64_t* __restrict__ origin, int64_t nb,
                          const long long* __restrict__ cidx, Grid g, uint64_t* __restrict__ corigin,
                          uint8_t* __restrict__ ckind, uint64_t* __restrict__ cj, uint32_t* __restrict__ cmap) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const long long i = cidx[b];
    if (cidx[b + 1] == i) continue;  // not a candidate
    const int k = kind[b];
    const uint64_t o = origin[b];
    uint64_t j = 0;
    if (k == 1) {
      j = (b > 0 && origin[b - 1] == o && kind[b - 1] == 1) ? 1 : 0;
    } else if (k == 2) {
      int64_t A; int t;
      id_cell_fast<D>(o, A, t);
      const uint64_t t0 = cells[off[b]];
      for (int sl = 0; sl < t_nlink<D>(t); sl++)
        if (cell_id<D>(cof_anchor<D>(g, A, t, sl), t_cof_type<D>(t, sl)) == t0) { j = (uint64_t)sl; break; }
    }
    corigin[i] = o;
    ckind[i] = (uint8_t)k;
    cj[i] = j;
    cmap[i] = (uint32_t)b;
  }
}

// The box of the anchors a traced branch visited (its origin and every cell of its
// g-CSR entry), for the end cache
struct T3Box {
  uint16_t lo[3], hi[3];
};

// flag[b] for the candidates: like k_t3_flags, candidate i of the g-CSR against branch
// cmap[i] of the f-CSR (the other branches keep flag 0).  With the end cache (box !=
// nullptr): box[b] and t3st[b] = 1 (same end) / 2 (another end).
template <int D>
__global__ void __launch_bounds__(T3_WARPS * 32)
k_t3_flags_cand(const long long* __restrict__ foff, const uint64_t* __restrict__ fcells,
                const uint64_t* __restrict__ fterm, const uint8_t* __restrict__ kind,
                const long long* __restrict__ goff, const uint64_t* __restrict__ gcells,
                const uint64_t* __restrict__ gterm, const uint32_t* __restrict__ cmap, int64_t nc,
                uint8_t* __restrict__ flag, const uint64_t* __restrict__ gorigin, Grid g, T3Box* __restrict__ box,
                uint8_t* __restrict__ t3st) {
  __shared__ unsigned long long sl[T3_WARPS][2][T3_SMEM];
  __shared__ int sn[T3_WARPS][2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nc;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = cmap[i];
    if (box) {
      uint32_t lo[3] = {0xFFFFu, 0xFFFFu, 0xFFFFu}, hi[3] = {0u, 0u, 0u};
      for (int64_t q = goff[i] + lane - 1; q < goff[i + 1]; q += 32) {
        const uint64_t id = q < goff[i] ? gorigin[i] : gcells[q];
        int64_t A; int t;
        id_cell_fast<D>(id, A, t);
        int64_t x, y, z;
        coords_of(g, A, x, y, z);
        const uint32_t c3[3] = {(uint32_t)x, (uint32_t)y, (uint32_t)z};
#pragma unroll
        for (int a = 0; a < 3; a++) {
          lo[a] = c3[a] < lo[a] ? c3[a] : lo[a];
          hi[a] = c3[a] > hi[a] ? c3[a] : hi[a];
        }
      }
      T3Box bx;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        bx.lo[a] = (uint16_t)__reduce_min_sync(0xffffffffu, lo[a]);
        bx.hi[a] = (uint16_t)__reduce_max_sync(0xffffffffu, hi[a]);
      }
      if (lane == 0) box[b] = bx;
    }
    if (kind[b] != 4) {
      if (lane == 0) {
        const bool differ = fterm[b] != gterm[i];
        flag[b] = differ;
        if (box) t3st[b] = differ ? 2 : 1;
      }
      continue;
    }
    const int64_t s0[2] = {foff[b], goff[i]}, s1[2] = {foff[b + 1], goff[i + 1]};
    const uint64_t* cs[2] = {fcells, gcells};
    if (lane < 2) sn[wib][lane] = 0;
    __syncwarp();
    int cnt[2];
    for (int h = 0; h < 2; h++) {
      int c = 0;
      for (int64_t q = s0[h] + lane; q < s1[h]; q += 32) {
        const uint64_t id = cs[h][q];
        if ((id >> 56) != 1) continue;
        c++;
        const int p = atomicAdd(&sn[wib][h], 1);
        if (p < T3_SMEM) sl[wib][h][p] = id;
      }
      cnt[h] = __reduce_add_sync(0xffffffffu, c);
    }
    __syncwarp();
    bool differ = cnt[0] != cnt[1];
    if (!differ && cnt[0] > 0) {
      bool bad = false;
      if (cnt[0] <= T3_SMEM) {
        for (int q = lane; q < cnt[0]; q += 32) {
          const unsigned long long x = sl[wib][0][q];
          int a = 0, c = 0;
          for (int r = 0; r < cnt[0]; r++) {
            a += sl[wib][0][r] == x;
            c += sl[wib][1][r] == x;
          }
          bad |= a != c;
        }
      } else {
        for (int64_t q = s0[0] + lane; q < s1[0]; q += 32) {
          const uint64_t x = fcells[q];
          if ((x >> 56) != 1) continue;
          int64_t a = 0, c = 0;
          for (int64_t r = s0[0]; r < s1[0]; r++) a += fcells[r] == x;
          for (int64_t r = s0[1]; r < s1[1]; r++) c += gcells[r] == x;
          bad |= a != c;
        }
      }
      differ = __any_sync(0xffffffffu, bad);
    }
    if (lane == 0) {
      flag[b] = differ ? 1 : 0;
      if (box) t3st[b] = differ ? 2 : 1;
    }
    __syncwarp();
  }
}

// P = the inclusive 3D prefix sums of the per-anchor bits `bits` (x, then y, then z)
__global__ void k_t3_psum_x(const uint32_t* __restrict__ bits, Grid g, int32_t* __restrict__ P) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = g.ny * g.nz;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t v0 = r * g.nx;
    int32_t carry = 0;
    for (int64_t x0 = 0; x0 < g.nx; x0 += 32) {
      const int64_t v = v0 + x0 + lane;
      int32_t s = x0 + lane < g.nx ? (int32_t)((bits[v >> 5] >> (v & 31)) & 1u) : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += u;
      }
      if (x0 + lane < g.nx) P[v] = carry + s;
      carry += __shfl_sync(0xffffffffu, s, 31);
    }
  }
}
// axis 1: along y for every (x, z); axis 2: along z for every (x, y)
__global__ void k_t3_psum_yz(Grid g, int axis, int32_t* __restrict__ P) {
  const int64_t n_lines = axis == 1 ? g.nx * g.nz : g.nx * g.ny;
  const int64_t len = axis == 1 ? g.ny : g.nz, stride = axis == 1 ? g.sy : g.sz;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n_lines; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = l % g.nx, o = l / g.nx;   // o = z (axis 1) or y (axis 2)
    int64_t v = x + (axis == 1 ? o * g.sz : o * g.sy);
    int32_t acc = 0;
    for (int64_t k = 0; k < len; k++, v += stride) {
      acc += P[v];
      P[v] = acc;
    }
  }
}

__device__ __forceinline__ int64_t psum_at(const int32_t* P, const Grid& g, int64_t x, int64_t y, int64_t z) {
  return (x < 0 || y < 0 || z < 0) ? 0 : (int64_t)P[x + y * g.sy + z * g.sz];
}

// the cached end comparisons still valid: no changed-code window (bits of sdil) within
// the branch's box grown by 2 on every side; the others are dropped
__global__ void k_t3_valid(const int32_t* __restrict__ P, Grid g, int64_t nb, const T3Box* __restrict__ box,
                           uint8_t* __restrict__ t3st) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    if (!t3st[b]) continue;
    const T3Box bx = box[b];
    const int64_t n[3] = {g.nx, g.ny, g.nz};
    int64_t lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      lo[a] = (int64_t)bx.lo[a] - 2 > 0 ? (int64_t)bx.lo[a] - 2 : 0;
      hi[a] = (int64_t)bx.hi[a] + 2 < n[a] - 1 ? (int64_t)bx.hi[a] + 2 : n[a] - 1;
    }
    const int64_t s = psum_at(P, g, hi[0], hi[1], hi[2]) - psum_at(P, g, lo[0] - 1, hi[1], hi[2]) -
                      psum_at(P, g, hi[0], lo[1] - 1, hi[2]) - psum_at(P, g, hi[0], hi[1], lo[2] - 1) +
                      psum_at(P, g, lo[0] - 1, lo[1] - 1, hi[2]) + psum_at(P, g, lo[0] - 1, hi[1], lo[2] - 1) +
                      psum_at(P, g, hi[0], lo[1] - 1, lo[2] - 1) - psum_at(P, g, lo[0] - 1, lo[1] - 1, lo[2] - 1);
    if (s) t3st[b] = 0;
  }
}

}  // namespace dmtz
