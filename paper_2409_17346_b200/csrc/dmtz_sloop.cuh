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
// "First" is found cell-parallel: k_tm_cells (one thread per CSR cell) takes an
// atomicMin of the cell's position key into its branch's slot; k_tm_targets (one
// thread per branch) turns the winning key into the target.  The branch of each
// CSR cell is precomputed once (k_cell_branch_*).
#pragma once

#include "dmtz_kernels.cuh"
#include "dmtz_sweep.cuh"
#include "dmtz_trace.cuh"

namespace dmtz {

constexpr uint32_t TM_NONE = 0xFFFFFFFFu;

// ----------------------------------------------------------------------------- cell -> branch
// Branches of at most 32 cells are filled by their own thread; longer ones are
// listed (long_list) and filled by a warp each.
__global__ void k_cell_branch_short(const long long* __restrict__ off, int64_t nb, uint32_t* __restrict__ cb,
                                    uint32_t* __restrict__ long_list, unsigned long long* __restrict__ n_long) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = off[b], i1 = off[b + 1];
    if (i1 - i0 <= 32) {
      for (int64_t i = i0; i < i1; i++) cb[i] = (uint32_t)b;
    } else {
      long_list[atomicAdd(n_long, 1ull)] = (uint32_t)b;
    }
  }
}

__global__ void k_cell_branch_long(const long long* __restrict__ off, const uint32_t* __restrict__ long_list,
                                   const unsigned long long* __restrict__ n_long, uint32_t* __restrict__ cb) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)*n_long;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t b = long_list[w];
    const int64_t i0 = off[b], i1 = off[b + 1];
    for (int64_t i = i0 + lane; i < i1; i += 32) cb[i] = b;
  }
}

__global__ void k_fill_u32(uint32_t* __restrict__ a, int64_t n, uint32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
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

// ----------------------------------------------------------------------------- per-cell keys
// key of a mismatch: DESC / ASC: the cell's position in its branch; CONN: 3 * (queue
// position) + facet, queue position 0 = the origin (k_tm_targets), logged triangle at
// branch position p -> queue position p + 1.
template <int D>
__global__ void k_tm_cells(const uint64_t* __restrict__ cells, int64_t n_cells, const uint32_t* __restrict__ cb,
                           const long long* __restrict__ off, const uint8_t* __restrict__ kind,
                           const void* __restrict__ cf, const void* __restrict__ cg,
                           const uint32_t* __restrict__ crit_f, Grid g, uint32_t* __restrict__ first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_cells;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = cb[i];
    const int k = kind[b];
    const int64_t i0 = off[b];
    const int64_t pos = i - i0;
    const uint64_t id = cells[i];
    const int d = (int)(id >> 56);
    uint32_t key = TM_NONE;
    if (k == 1) {  // DESC: vertices at even positions, not the minimum at the end
      if ((pos & 1) || i + 1 >= off[b + 1]) continue;
      int64_t A; int t;
      id_cell<D>(id, A, t);
      if (pair_differs<D>(cf, cg, g, A, t)) key = (uint32_t)pos;
    } else if (k == 2) {  // ASC: (top-1)-cells at odd positions
      if (!(pos & 1)) continue;
      int64_t A; int t;
      id_cell<D>(id, A, t);
      if (pair_differs<D>(cf, cg, g, A, t)) key = (uint32_t)pos;
    } else {  // CONN: the facet edges of a logged triangle
      if (d != 2) continue;
      int64_t B; int bt;
      id_cell<D>(id, B, bt);
      for (int j = 0; j < 3; j++) {
        const int64_t E = B + mask_delta(g, t_facet<D>(bt, j, 0));
        const int et = t_facet<D>(bt, j, 1);
        if ((__ldg(crit_f + E) >> et) & 1u) continue;
        if (pair_differs<D>(cf, cg, g, E, et)) { key = (uint32_t)(3 * (pos + 1) + j); break; }
      }
    }
    if (key != TM_NONE && key < first[b]) atomicMin(first + b, key);
  }
}

// ----------------------------------------------------------------------------- per-branch targets
// cnt->pad[3] += troublemakers, cnt->pad[4 + kind index] += per kind; first[] reset.
// flag (tier 3, else nullptr): only branches with flag[b] != 0 count.
template <int D>
__global__ void k_tm_targets(const uint64_t* __restrict__ cells, const long long* __restrict__ off,
                             const uint8_t* __restrict__ kind, const uint64_t* __restrict__ origin, int64_t nb,
                             const void* __restrict__ cf, const void* __restrict__ cg,
                             const uint32_t* __restrict__ crit_f, Grid g, RowGeom rg, uint32_t* __restrict__ first,
                             const uint8_t* __restrict__ flag, uint32_t* __restrict__ tbits,
                             Counters* __restrict__ cnt) {
  unsigned long long ntm = 0, nk[3] = {0, 0, 0}, bad = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t key = first[b];
    if (key != TM_NONE) first[b] = TM_NONE;
    if (flag && !flag[b]) continue;  // tier 3: this branch ends where it ends in f
    const int k = kind[b];
    int64_t A = -1;
    int t = 0;
    if (k == 4) {
      int64_t B; int bt;
      id_cell<D>(origin[b], B, bt);
      for (int j = 0; j < 3; j++) {  // the origin's facets come first (queue position 0)
        const int64_t E = B + mask_delta(g, t_facet<D>(bt, j, 0));
        const int et = t_facet<D>(bt, j, 1);
        if ((__ldg(crit_f + E) >> et) & 1u) continue;
        if (pair_differs<D>(cf, cg, g, E, et)) { key = (uint32_t)j; break; }
      }
      if (key == TM_NONE) continue;
      const uint32_t qp = key / 3, j = key - qp * 3;
      if (qp > 0) id_cell<D>(cells[off[b] + qp - 1], B, bt);
      A = B + mask_delta(g, t_facet<D>(bt, (int)j, 0));
      t = t_facet<D>(bt, (int)j, 1);
    } else {
      if (key == TM_NONE) continue;
      id_cell<D>(cells[off[b] + key], A, t);
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
