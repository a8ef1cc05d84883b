// dmtz_trace.cuh -- V-path separatrix traces (a9-a11) for sm_100a; see include/dmtz.h.
//
// Gradient paths from the saddles, on the gradient given as codes:
//   DESC  vertex -> paired edge -> other vertex ... -> minimum      (pointer chase)
//   ASC   top cell -> paired facet -> other top cofacet ... -> maximum | BOUNDARY
//   CONN  breadth-first over triangle -> facet edge -> paired triangle (3D)
// Layout of the work:
//   1. crit masks of the codes (k_critmask)
//   2. per kind: per-anchor branch counts -> exclusive scan -> emit branch
//      descriptors (origin id, kind, branch index j) in (origin id, j) order
//   3. per branch: walk once to count cells -> scan -> walk again writing cells
// One thread per branch for the walks; connector BFS runs per saddle with a
// private queue + open-addressing visited set in workspace scratch (saddles
// whose search outgrows the slot are redone alone with the whole scratch).
#pragma once
#include <chrono>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include <cstdlib>

#include "dmtz_kernels.cuh"

namespace dmtz {

struct TraceArgs {
  Grid g;
  const void* codes;
  uint32_t kinds;
  long long* pre;            // >= N x 8 B workspace region: per-anchor branch counts, then overflow flags
  size_t pre_bytes;
  unsigned long long* bfs;   // >= N x 8 B workspace region: connector BFS slots (zeroed, self-cleaning)
  size_t bfs_bytes;
  uint32_t* crit;            // N x 4 B workspace region
  unsigned long long* bsum;  // scan block sums (>= N / 8192 + 2 entries)
  Counters* cnt;
  Counters* host_cnt;
  int64_t* out_offsets;
  uint64_t* out_cells;
  uint64_t* out_origin;
  uint64_t* out_terminal;
  uint8_t* out_kind;
  int64_t cap_b, cap_c;
  int64_t a_lo = 0, a_hi = INT64_MAX;   // origin anchors traced: [a_lo, a_hi)
  // given branches (given_nbk[0] >= 0): the caller filled out_origin / out_kind /
  // out_terminal (= the branch index j) for given_nbk[k] branches of each kind, grouped
  // DESC, ASC, CONN; only those are traced
  int64_t given_nbk[3] = {-1, -1, -1};
  bool unordered = false;    // connectors' events in any order (k_walk_block UN; tier-3 candidates)
  int verbose = 0;
  int64_t n_branches = 0, n_cells = 0, n_internal = 0;
  int64_t n_overflow = 0;  // connectors whose BFS outgrew all scratch (-> DMTZ_E_CAPACITY)
  // connectors handled per escalation level in the count pass: [0] all (thread queues),
  // [1] warp queues, [2..] block BFS levels (slots growing by 16x)
  int64_t level_counts[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
};

constexpr uint64_t CELL_BOUNDARY = ~0ull;
constexpr int SCAN_CHUNK = 8192;

template <int D> __host__ __device__ constexpr int types_of_dim(int d) {
  return D == 3 ? (d == 0 ? 1 : d == 1 ? 7 : d == 2 ? 12 : 6) : (d == 0 ? 1 : d == 1 ? 3 : 2);
}

template <int D>
__device__ __forceinline__ uint64_t cell_id(int64_t anchor, int t) {
  const int d = t_dim<D>(t);
  const int k = t - t_first_of_dim<D>(d);
  return ((uint64_t)d << 56) | (uint64_t)(anchor * types_of_dim<D>(d) + k);
}

template <int D>
__device__ __forceinline__ uint64_t code_at(const void* codes, int64_t a) {
  return D == 3 ? (uint64_t)((const unsigned long long*)codes)[a] : (uint64_t)((const unsigned short*)codes)[a];
}

__device__ __forceinline__ void coords_of(const Grid& g, int64_t v, int64_t& x, int64_t& y, int64_t& z) {
  if (g.fast) {  // 32-bit multiply-high divisions
    const uint32_t v32 = (uint32_t)v, z32 = g.dsz.div(v32), r = v32 - z32 * (uint32_t)g.sz;
    const uint32_t y32 = g.dnx.div(r);
    z = z32;
    y = y32;
    x = r - y32 * (uint32_t)g.nx;
    return;
  }
  z = v / g.sz;
  const int64_t r = v - z * g.sz;
  y = r / g.nx;
  x = r - y * g.nx;
}

template <int D>
__device__ __forceinline__ bool link_in_grid_xyz(const Grid& g, int64_t x, int64_t y, int64_t z, int t, int s) {
  x += t_link<D>(t, s, 0);
  y += t_link<D>(t, s, 1);
  z += t_link<D>(t, s, 2);
  return x >= 0 && y >= 0 && z >= 0 && x < g.nx && y < g.ny && z < g.nz;
}

template <int D>
__device__ __forceinline__ bool link_in_grid(const Grid& g, int64_t a, int t, int s) {
  int64_t x, y, z;
  coords_of(g, a, x, y, z);
  x += t_link<D>(t, s, 0);
  y += t_link<D>(t, s, 1);
  z += t_link<D>(t, s, 2);
  return x >= 0 && y >= 0 && z >= 0 && x < g.nx && y < g.ny && z < g.nz;
}

template <int D>
__device__ __forceinline__ int64_t cof_anchor(const Grid& g, int64_t a, int t, int s) {
  return a + t_cof_anchor<D>(t, s, 0) + t_cof_anchor<D>(t, s, 1) * g.sy + t_cof_anchor<D>(t, s, 2) * g.sz;
}

// facet of top cell (B, bt) paired with it (its code points at B), or -1 if critical
template <int D>
__device__ __forceinline__ int paired_facet(const void* codes, const Grid& g, int64_t B, int bt, int64_t& fa,
                                            int& ftype) {
  for (int j = 0; j < t_nfacet<D>(bt); j++) {
    const int dm = t_facet<D>(bt, j, 0), ft = t_facet<D>(bt, j, 1), sl = t_facet<D>(bt, j, 2);
    const int64_t a = B + mask_delta(g, dm);
    if (field_of<D>(code_at<D>(codes, a), ft) == (uint32_t)sl) { fa = a; ftype = ft; return j; }
  }
  return -1;
}

// ----------------------------------------------------------------------------- counting / emission
// every link vertex (offsets in [-1, 1]^D) of a cell anchored at (x, y, z) is in the grid
template <int D>
__device__ __forceinline__ bool links_interior(const Grid& g, int64_t x, int64_t y, int64_t z) {
  return x >= 1 && y >= 1 && x + 1 < g.nx && y + 1 < g.ny && (D == 2 || (z >= 1 && z + 1 < g.nz));
}
// the types of dimension d as a bit mask, and cell_id for a type of known dimension d
template <int D, int d> __device__ __forceinline__ constexpr uint32_t dim_mask() {
  return ((1u << t_first_of_dim_c<D>(d + 1)) - 1u) & ~((1u << t_first_of_dim_c<D>(d)) - 1u);
}
template <int D, int d> __device__ __forceinline__ uint64_t cell_id_dim(int64_t a, int t) {
  return ((uint64_t)d << 56) | (uint64_t)(a * types_of_dim<D>(d) + (t - t_first_of_dim_c<D>(d)));
}

template <int D>
__device__ __forceinline__ int branch_count(const Grid& g, int kind, uint32_t cm, int64_t x, int64_t y, int64_t z) {
  const int top = Tr<D>::TOP;
  // (top-1)-cells have 2 link vertices in both dimensions: interior anchors need no check
  if (kind == 2 && links_interior<D>(g, x, y, z)) return 2 * __popc(cm & dim_mask<D, Tr<D>::TOP - 1>());
  if (kind == 1) {  // DESC: two branches per critical edge
    const uint32_t em = ((1u << t_first_of_dim<D>(2)) - 1u) & ~1u;
    return 2 * __popc(cm & em);
  }
  if (kind == 2) {  // ASC: one branch per in-grid top cofacet of each critical (top-1)-cell
    int n = 0;
    for (int t = t_first_of_dim<D>(top - 1); t < t_first_of_dim<D>(top); t++) {
      if (!((cm >> t) & 1u)) continue;
      for (int s = 0; s < t_nlink<D>(t); s++) n += link_in_grid_xyz<D>(g, x, y, z, t, s) ? 1 : 0;
    }
    return n;
  }
  // CONN: one branch per critical triangle (3D)
  if (D != 3) return 0;
  const uint32_t tm = ((1u << t_first_of_dim<D>(3)) - 1u) & ~((1u << t_first_of_dim<D>(2)) - 1u);
  return __popc(cm & tm);
}

// exclusive scan helper: one-block scan of block totals (the branch-origin tiles)
__global__ void k_scan_top(unsigned long long* __restrict__ bsum, int64_t nb, unsigned long long* __restrict__ total) {
  // exclusive scan of nb block sums by one block of 1024 threads (contiguous ranges)
  __shared__ unsigned long long part[1024];
  const int64_t per = (nb + 1023) / 1024;
  const int64_t lo = threadIdx.x * per, hi = lo + per < nb ? lo + per : nb;
  unsigned long long acc = 0;
  for (int64_t i = lo; i < hi; i++) acc += bsum[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned long long v = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0ull;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned long long run = part[threadIdx.x] - acc;
  for (int64_t i = lo; i < hi; i++) { const unsigned long long v = bsum[i]; bsum[i] = run; run += v; }
  if (threadIdx.x == 1023) *total = part[1023];
}

// Single-pass exclusive scan (decoupled look-back): block b (in the order blocks start,
// ticket state[0]) scans its SCAN_CHUNK elements, publishes its aggregate in state[1 + b]
// (flag 1 << 62), sums its predecessors' words back to the first inclusive prefix (flag
// 2 << 62), publishes its own inclusive prefix and writes its elements once.  state:
// 1 + ceil(n / SCAN_CHUNK) words, zeroed.  Values < 2^62.
constexpr int SCL_THREADS = 512, SCL_PER = SCAN_CHUNK / SCL_THREADS;
__global__ void __launch_bounds__(SCL_THREADS)
k_scan_lb(long long* __restrict__ a, int64_t n, unsigned long long* __restrict__ state,
          unsigned long long* __restrict__ total) {
  __shared__ long long s_w[SCL_THREADS / 32];
  __shared__ long long s_excl;
  __shared__ int64_t s_bid;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_bid = (int64_t)atomicAdd(state, 1ull);
  __syncthreads();
  const int64_t bid = s_bid;
  const int64_t base = bid * SCAN_CHUNK + (int64_t)tid * SCL_PER;
  long long v[SCL_PER];
  long long sum = 0;
  const bool vec = base + SCL_PER <= n && ((uintptr_t)a & 15u) == 0;
  if (vec) {
    const longlong2* p2 = reinterpret_cast<const longlong2*>(a + base);   // base is even: 16-byte aligned
#pragma unroll
    for (int k = 0; k < SCL_PER / 2; k++) {
      const longlong2 w = p2[k];
      v[2 * k] = w.x;
      v[2 * k + 1] = w.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < SCL_PER; k++) v[k] = base + k < n ? a[base + k] : 0;
  }
#pragma unroll
  for (int k = 0; k < SCL_PER; k++) sum += v[k];
  long long inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_w[wid] = inc;
  __syncthreads();
  long long wbase = 0, agg = 0;
#pragma unroll
  for (int w2 = 0; w2 < SCL_THREADS / 32; w2++) {
    const long long x = s_w[w2];
    if (w2 < wid) wbase += x;
    agg += x;
  }
  if (tid == 0) {
    volatile unsigned long long* st = state + 1;
    long long excl = 0;
    if (bid == 0) {
      st[0] = (2ull << 62) | (unsigned long long)agg;
    } else {
      st[bid] = (1ull << 62) | (unsigned long long)agg;
      __threadfence();
      for (int64_t j = bid - 1;; ) {
        const unsigned long long w = st[j];
        const unsigned f = (unsigned)(w >> 62);
        if (!f) continue;   // not published yet
        excl += (long long)(w & ((1ull << 62) - 1));
        if (f == 2) break;
        j--;
      }
      __threadfence();
      st[bid] = (2ull << 62) | (unsigned long long)(excl + agg);
    }
    s_excl = excl;
    if ((bid + 1) * SCAN_CHUNK >= n) *total = (unsigned long long)(excl + agg);
  }
  __syncthreads();
  long long run = s_excl + wbase + inc - sum;
  if (vec) {
    longlong2* p2 = reinterpret_cast<longlong2*>(a + base);
#pragma unroll
    for (int k = 0; k < SCL_PER / 2; k++) {
      longlong2 w;
      w.x = run;
      run += v[2 * k];
      w.y = run;
      run += v[2 * k + 1];
      p2[k] = w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < SCL_PER; k++)
      if (base + k < n) { a[base + k] = run; run += v[k]; }
  }
}

// Branch origins without an N-sized count array: a block owns BT_TILE consecutive
// anchors (BT_PER per thread); pass 1 writes the block's branch total, the block
// totals are scanned, pass 2 recomputes the counts, scans them inside the block and
// emits in (anchor, type, branch) order.
constexpr int BT_THREADS = 256, BT_PER = 8, BT_TILE = BT_THREADS * BT_PER;

template <int D>
__device__ __forceinline__ int tile_counts(const uint32_t* __restrict__ crit, const Grid& g, int kind, int64_t a0,
                                           int64_t a_lo, int64_t a_hi, int (&c)[BT_PER]) {
  int64_t x, y, z;
  coords_of(g, a0 < g.N ? a0 : 0, x, y, z);
  int tot = 0;
#pragma unroll
  for (int k = 0; k < BT_PER; k++) {
    const int64_t a = a0 + k;
    c[k] = a < g.N && a >= a_lo && a < a_hi ? branch_count<D>(g, kind, __ldg(crit + a), x, y, z) : 0;
    tot += c[k];
    if (++x == g.nx) { x = 0; if (++y == g.ny) { y = 0; ++z; } }
  }
  return tot;
}

__device__ __forceinline__ long long block_exclusive_scan(long long v, long long* total) {
  __shared__ long long ws[BT_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) ws[wid] = incl;
  __syncthreads();
  long long wbase = 0, tot = 0;
  for (int w = 0; w < BT_THREADS / 32; w++) {
    const long long x = ws[w];
    if (w < wid) wbase += x;
    tot += x;
  }
  __syncthreads();
  *total = tot;
  return wbase + incl - v;
}

template <int D>
__global__ void __launch_bounds__(BT_THREADS)
k_branch_tiles(const uint32_t* __restrict__ crit, Grid g, int kind, int64_t a_lo, int64_t a_hi,
               unsigned long long* __restrict__ bsum, int64_t tile0) {
  int c[BT_PER];
  const int t = tile_counts<D>(crit, g, kind, (tile0 + (int64_t)blockIdx.x) * BT_TILE + threadIdx.x * BT_PER, a_lo,
                               a_hi, c);
  long long tot;
  block_exclusive_scan(t, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = (unsigned long long)tot;
}

// Emission: warp w of the block takes anchors [w * 256, w * 256 + 256) of the tile in
// 8 steps of 32 consecutive anchors (lane = anchor), so every step writes one dense
// range of the outputs (coalesced) in (anchor, type, branch) order.
template <int D>
__global__ void __launch_bounds__(BT_THREADS)
k_branch_tiles_emit(const uint32_t* __restrict__ crit, Grid g, int kind, int64_t a_lo, int64_t a_hi,
                    const unsigned long long* __restrict__ bscan, int64_t base, uint64_t* __restrict__ origin,
                    uint8_t* __restrict__ kout, uint64_t* __restrict__ jout, int64_t tile0) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t w0 = (tile0 + (int64_t)blockIdx.x) * BT_TILE + (int64_t)wid * 32 * BT_PER;  // the warp's first anchor
  int c[BT_PER];
  uint32_t cm[BT_PER];
  int wtot = 0;
#pragma unroll
  for (int k = 0; k < BT_PER; k++) {
    const int64_t a = w0 + k * 32 + lane;
    int64_t x, y, z;
    coords_of(g, a < g.N ? a : 0, x, y, z);
    cm[k] = a < g.N && a >= a_lo && a < a_hi ? __ldg(crit + a) : 0u;
    c[k] = cm[k] ? branch_count<D>(g, kind, cm[k], x, y, z) : 0;
    wtot += __reduce_add_sync(0xffffffffu, (unsigned)c[k]);
  }
  long long tot;
  // exclusive scan of the warp totals in warp order = anchor order
  const long long wbase = block_exclusive_scan(lane == 0 ? wtot : 0, &tot);
  int64_t b = base + (int64_t)bscan[blockIdx.x] + __shfl_sync(0xffffffffu, wbase, 0);
  const int top = Tr<D>::TOP;
  // a step's branches are staged in shared memory (lane order = anchor order), then
  // written out by consecutive lanes (coalesced; the kind byte too); a step with more
  // than BT_STAGE branches writes directly
  constexpr int BT_STAGE = 512;
  __shared__ unsigned long long s_org[BT_THREADS / 32][BT_STAGE];
  __shared__ uint8_t s_j[BT_THREADS / 32][BT_STAGE];
#pragma unroll 1
  for (int k = 0; k < BT_PER; k++) {
    int pre = c[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += v;
    }
    const int stot = __shfl_sync(0xffffffffu, pre, 31);
    const int64_t p0 = b;
    b += stot;
    if (!stot) continue;   // warp-uniform
    const bool staged = stot <= BT_STAGE;
    int q = pre - c[k];    // my first entry within the step
    auto put = [&](uint64_t org, int j) {
      if (staged) { s_org[wid][q] = org; s_j[wid][q] = (uint8_t)j; }
      else { origin[p0 + q] = org; kout[p0 + q] = (uint8_t)kind; jout[p0 + q] = (uint64_t)j; }
      q++;
    };
    if (c[k]) {
      const int64_t a = w0 + k * 32 + lane;
      if (kind == 1) {
        for (uint32_t m = cm[k] & dim_mask<D, 1>(); m; m &= m - 1u) {
          const uint64_t id = cell_id_dim<D, 1>(a, __ffs(m) - 1);
          put(id, 0);
          put(id, 1);
        }
      } else if (kind == 2) {
        int64_t x, y, z;
        coords_of(g, a, x, y, z);
        if (links_interior<D>(g, x, y, z)) {
          for (uint32_t m = cm[k] & dim_mask<D, Tr<D>::TOP - 1>(); m; m &= m - 1u) {
            const uint64_t id = cell_id_dim<D, Tr<D>::TOP - 1>(a, __ffs(m) - 1);
            put(id, 0);
            put(id, 1);
          }
        } else
        for (int tt = t_first_of_dim<D>(top - 1); tt < t_first_of_dim<D>(top); tt++) {
          if (!((cm[k] >> tt) & 1u)) continue;
          for (int sl = 0; sl < t_nlink<D>(tt); sl++) {
            if (!link_in_grid_xyz<D>(g, x, y, z, tt, sl)) continue;
            put(cell_id<D>(a, tt), sl);
          }
        }
      } else if (D == 3) {
        for (uint32_t m = cm[k] & dim_mask<D, 2>(); m; m &= m - 1u) put(cell_id_dim<D, 2>(a, __ffs(m) - 1), 0);
      }
    }
    if (staged) {
      __syncwarp();
      for (int i = lane; i < stot; i += 32) {
        origin[p0 + i] = s_org[wid][i];
        kout[p0 + i] = (uint8_t)kind;
        jout[p0 + i] = (uint64_t)s_j[wid][i];
      }
      __syncwarp();
    }
  }
}

// decode a cell id back to (anchor, type)
template <int D>
__device__ __forceinline__ void id_cell(uint64_t id, int64_t& a, int& t) {
  const int d = (int)(id >> 56);
  const int64_t r = (int64_t)(id & ((1ull << 56) - 1));
  const int Td = types_of_dim<D>(d);
  a = r / Td;
  t = t_first_of_dim<D>(d) + (int)(r - a * Td);
}

// ----------------------------------------------------------------------------- compact views
// Built once per trace from the codes and criticality, so that a walk step reads
// one small word instead of several 8-byte codes:
//  vnib: 4 bits per vertex = its cand slot (NONE = critical), 64 MB for 512^3 (L2-resident);
//  tpair: per anchor, 3 bits per top cell type = the facet j paired with it, 7 if critical;
//  eview (3D): per anchor, 4 bits per edge type = cand slot | critical << 3.
struct TraceViews {
  uint8_t* vnib;
  uint32_t* tpair;
  uint32_t* eview;
};

// The critical masks and the views in one pass: per anchor its 8 codes are read once,
// decode_crit_dp gives the critical mask and, for every paired-down cell, the facet it
// is paired with (tpair of the top cells)
template <int D>
__global__ void k_trace_views_crit(const void* codes, uint32_t* __restrict__ crit, Grid g, TraceViews V) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * p < g.N; p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t nib = 0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int64_t u = 2 * p + h;
      if (u >= g.N) break;
      int64_t x, y, z;
      coords_of(g, u, x, y, z);
      const int ok = axes_ok(g, x, y, z);
      uint64_t c[Tr<D>::NDELTA];
      load_codes8<D>((const typename Tr<D>::code_t*)codes, g, u, ok, c);
      uint64_t dp;
      const uint32_t cm = decode_crit_dp<D>(c, ok, &dp);
      crit[u] = cm;
      nib |= (field_of<D>(c[0], 0) & 15u) << (4 * h);
      const int tt0 = t_first_of_dim<D>(Tr<D>::TOP);
      const uint32_t ex = t_exist<D>(ok);
      uint32_t tp = 0;
#pragma unroll
      for (int t = tt0; t < Tr<D>::NT; t++) {
        const uint32_t j = (((ex >> t) & 1u) && !((cm >> t) & 1u)) ? (uint32_t)(dp >> (2 * t)) & 3u : 7u;
        tp |= j << (3 * (t - tt0));
      }
      V.tpair[u] = tp;
      if (D == 3) {
        uint32_t ev = 0;
#pragma unroll
        for (int e = 0; e < 7; e++) {
          const int et = t_first_of_dim<D>(1) + e;
          ev |= ((field_of<D>(c[0], et) & 7u) | (((cm >> et) & 1u) << 3)) << (4 * e);
        }
        V.eview[u] = ev;
      }
    }
    V.vnib[p] = (uint8_t)nib;
  }
}

// ----------------------------------------------------------------------------- walks
// write == false: count cells only.  Returns the cell count or -1 on a cycle.
template <int D>
__device__ int64_t walk_desc(const TraceViews& V, const Grid& g, int64_t a, int t, int j, bool write,
                             uint64_t* cells, uint64_t* term, int64_t cap_steps) {
  int64_t v = a + mask_delta(g, t_vmask<D>(t, j));
  int64_t n = 0;
  if (write) cells[n] = cell_id<D>(v, 0);
  n++;
  for (int64_t step = 0;; step++) {
    if (step > cap_steps) return -1;
    const uint32_t s = (__ldg(V.vnib + (v >> 1)) >> (4 * (v & 1))) & 15u;
    if (s == (uint32_t)t_none<D>(0)) break;  // critical vertex (a vertex has no facets)
    const int64_t w = v + t_link<D>(0, s, 0) + t_link<D>(0, s, 1) * g.sy + t_link<D>(0, s, 2) * g.sz;
    if (write) {
      cells[n] = cell_id<D>(cof_anchor<D>(g, v, 0, s), t_cof_type<D>(0, s));
      cells[n + 1] = cell_id<D>(w, 0);
    }
    n += 2;
    v = w;
  }
  if (write) *term = cell_id<D>(v, 0);
  return n;
}

template <int D>
__device__ int64_t walk_asc(const TraceViews& V, const Grid& g, int64_t a, int t, int s0, bool write,
                            uint64_t* cells, uint64_t* term, int64_t cap_steps) {
  int64_t x, y, z;
  coords_of(g, a, x, y, z);   // once per branch; every step below moves by table offsets
  x += t_cof_anchor<D>(t, s0, 0);
  y += t_cof_anchor<D>(t, s0, 1);
  z += t_cof_anchor<D>(t, s0, 2);
  int64_t B = x + y * g.sy + z * g.sz;
  int bt = t_cof_type<D>(t, s0);
  const int tt0 = t_first_of_dim<D>(Tr<D>::TOP);
  int64_t n = 0;
  uint64_t terminal = CELL_BOUNDARY;
  for (int64_t step = 0;; step++) {
    if (step > cap_steps) return -1;
    if (write) cells[n] = cell_id<D>(B, bt);
    n++;
    const int j = (int)(__ldg(V.tpair + B) >> (3 * (bt - tt0))) & 7;
    if (j == 7) { terminal = cell_id<D>(B, bt); break; }  // maximum
    const int dm = t_facet<D>(bt, j, 0), ct = t_facet<D>(bt, j, 1);
    const int64_t cx = x + (dm & 1), cy = y + ((dm >> 1) & 1), cz = z + ((dm >> 2) & 1);
    const int64_t ca = B + mask_delta(g, dm);
    if (write) cells[n] = cell_id<D>(ca, ct);
    n++;
    // the other top cofacet of (ca, ct)
    bool moved = false;
    for (int s = 0; s < t_nlink<D>(ct); s++) {
      const int64_t lx = cx + t_link<D>(ct, s, 0), ly = cy + t_link<D>(ct, s, 1), lz = cz + t_link<D>(ct, s, 2);
      if (lx < 0 || ly < 0 || lz < 0 || lx >= g.nx || ly >= g.ny || lz >= g.nz) continue;
      const int nt = t_cof_type<D>(ct, s);
      const int64_t nx_ = cx + t_cof_anchor<D>(ct, s, 0), ny_ = cy + t_cof_anchor<D>(ct, s, 1),
                    nz_ = cz + t_cof_anchor<D>(ct, s, 2);
      const int64_t nb = nx_ + ny_ * g.sy + nz_ * g.sz;
      if (nb == B && nt == bt) continue;
      B = nb; bt = nt; x = nx_; y = ny_; z = nz_; moved = true;
      break;
    }
    if (!moved) break;  // boundary facet: the path leaves the domain
  }
  if (write) *term = terminal;
  return n;
}

template <int D>
__global__ void k_walk(TraceViews V, Grid g, int64_t b0, int64_t nb,
                       const uint64_t* __restrict__ origin, const uint8_t* __restrict__ kind,
                       uint64_t* __restrict__ jterm, long long* __restrict__ off, uint64_t* __restrict__ cells,
                       bool write, Counters* __restrict__ cnt) {
  const int64_t cap_steps = g.N * 26 + 1;
  for (int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t a;
    int t;
    id_cell<D>(origin[b], a, t);
    const int k = kind[b];
    int64_t n;
    uint64_t* out = write ? cells + off[b] : nullptr;
    uint64_t term = CELL_BOUNDARY;
    if (k == 1) n = walk_desc<D>(V, g, a, t, (int)jterm[b], write, out, &term, cap_steps);
    else if (k == 2) n = walk_asc<D>(V, g, a, t, (int)jterm[b], write, out, &term, cap_steps);
    else n = -1;  // connectors run in k_conn_small / k_walk_block
    if (n < 0) { atomicAdd(&cnt->n_internal, 1ull); n = 0; }
    if (!write) off[b] = n;
    else jterm[b] = term;
  }
}

// The same walks with dynamic lane refill: path lengths are heavy-tailed (C5: 36
// cells per branch on average), so with one branch per thread a warp runs as long as
// its longest path while the other lanes idle.  Here every lane advances its walk one
// step per iteration and an idle lane takes the next branch at once (warp-aggregated
// atomicAdd on *ctr, zeroed before the launch); persistent grid.  Same per-branch
// results as k_walk (each branch writes only its own cells / count / terminal).
template <int D>
__global__ void __launch_bounds__(128)
k_walk_dyn(TraceViews V, Grid g, int64_t b0, int64_t nb, const uint64_t* __restrict__ origin, const uint8_t* __restrict__ kind,
           uint64_t* __restrict__ jterm, long long* __restrict__ off, uint64_t* __restrict__ cells, bool write,
           Counters* __restrict__ cnt, unsigned long long* __restrict__ ctr) {
  const int64_t cap_steps = g.N * 26 + 1;
  const int lane = threadIdx.x & 31;
  const int tt0 = t_first_of_dim<D>(Tr<D>::TOP);
  int64_t b = -1;
  bool drained = false;
  int k = 0, bt = 0;
  int64_t v = 0, x = 0, y = 0, z = 0, n = 0, step = 0;
  uint64_t* out = nullptr;
  uint64_t term = CELL_BOUNDARY;
  for (;;) {
    const unsigned idle = __ballot_sync(0xffffffffu, b < 0);
    if (idle && !drained) {  // warp-uniform
      const int leader = __ffs(idle) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(idle));
      base = __shfl_sync(0xffffffffu, base, leader);
      if ((int64_t)(base + (unsigned long long)__popc(idle)) >= nb - b0) drained = true;
      if (b < 0) {
        const int64_t nbi = b0 + (int64_t)base + __popc(idle & ((1u << lane) - 1u));
        if (nbi < nb) {
          b = nbi;
          int64_t a;
          int t;
          id_cell<D>(origin[b], a, t);
          k = kind[b];
          const int jj = (int)jterm[b];
          n = 0;
          step = 0;
          out = write ? cells + off[b] : nullptr;
          term = CELL_BOUNDARY;
          if (k == 1) {
            v = a + mask_delta(g, t_vmask<D>(t, jj));
            if (write) out[0] = cell_id<D>(v, 0);
            n = 1;
          } else if (k == 2) {
            coords_of(g, a, x, y, z);
            x += t_cof_anchor<D>(t, jj, 0);
            y += t_cof_anchor<D>(t, jj, 1);
            z += t_cof_anchor<D>(t, jj, 2);
            v = x + y * g.sy + z * g.sz;
            bt = t_cof_type<D>(t, jj);
          }
        }
      }
    }
    if (__all_sync(0xffffffffu, b < 0)) break;
    if (b < 0) continue;
    bool done = false;
    if (k != 1 && k != 2) {
      n = -1;  // connectors run in k_conn_small / k_walk_block
      done = true;
    } else if (step++ > cap_steps) {
      n = -1;
      done = true;
    } else if (k == 1) {
      const uint32_t s = (__ldg(V.vnib + (v >> 1)) >> (4 * (v & 1))) & 15u;
      if (s == (uint32_t)t_none<D>(0)) {  // critical vertex
        term = cell_id<D>(v, 0);
        done = true;
      } else {
        const int64_t w = v + t_link<D>(0, s, 0) + t_link<D>(0, s, 1) * g.sy + t_link<D>(0, s, 2) * g.sz;
        if (write) {
          out[n] = cell_id<D>(cof_anchor<D>(g, v, 0, s), t_cof_type<D>(0, s));
          out[n + 1] = cell_id<D>(w, 0);
        }
        n += 2;
        v = w;
      }
    } else {
      if (write) out[n] = cell_id<D>(v, bt);
      n++;
      const int j = (int)(__ldg(V.tpair + v) >> (3 * (bt - tt0))) & 7;
      if (j == 7) {  // maximum
        term = cell_id<D>(v, bt);
        done = true;
      } else {
        const int dm = t_facet<D>(bt, j, 0), ct = t_facet<D>(bt, j, 1);
        const int64_t cx = x + (dm & 1), cy = y + ((dm >> 1) & 1), cz = z + ((dm >> 2) & 1);
        const int64_t ca = v + mask_delta(g, dm);
        if (write) out[n] = cell_id<D>(ca, ct);
        n++;
        bool moved = false;  // the other top cofacet of (ca, ct)
        for (int s = 0; s < t_nlink<D>(ct); s++) {
          const int64_t lx = cx + t_link<D>(ct, s, 0), ly = cy + t_link<D>(ct, s, 1), lz = cz + t_link<D>(ct, s, 2);
          if (lx < 0 || ly < 0 || lz < 0 || lx >= g.nx || ly >= g.ny || lz >= g.nz) continue;
          const int nt = t_cof_type<D>(ct, s);
          const int64_t nx_ = cx + t_cof_anchor<D>(ct, s, 0), ny_ = cy + t_cof_anchor<D>(ct, s, 1),
                        nz_ = cz + t_cof_anchor<D>(ct, s, 2);
          const int64_t nbb = nx_ + ny_ * g.sy + nz_ * g.sz;
          if (nbb == v && nt == bt) continue;
          v = nbb; bt = nt; x = nx_; y = ny_; z = nz_; moved = true;
          break;
        }
        if (!moved) done = true;  // boundary facet: terminal stays BOUNDARY
      }
    }
    if (done) {
      if (n < 0) { atomicAdd(&cnt->n_internal, 1ull); n = 0; }
      if (!write) off[b] = n;
      else jterm[b] = term;
      b = -1;
    }
  }
}

// Connector tables in shared memory: triangle type -> its 3 facet edges (dm | edge
// index << 3); edge (index, slot) -> cofacet triangle (type | (anchor delta + 1) << 5, 7, 9).
struct ConnTab {
  uint8_t tf[12 * 3];
  uint16_t ec[7 * 8];
};
template <int D>
__device__ __forceinline__ void conn_tables_init(ConnTab& T) {
  if constexpr (D == 3) {
    constexpr int T0 = t_first_of_dim_c<D>(2), E0 = t_first_of_dim_c<D>(1);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int tt = 0; tt < 12; tt++)
#pragma unroll
        for (int j = 0; j < 3; j++)
          T.tf[tt * 3 + j] = (uint8_t)(t_facet<D>(T0 + tt, j, 0) | ((t_facet<D>(T0 + tt, j, 1) - E0) << 3));
#pragma unroll
      for (int e = 0; e < 7; e++)
#pragma unroll
        for (int sl = 0; sl < 8; sl++)
          T.ec[e * 8 + sl] = sl < t_nlink<D>(E0 + e)
                                 ? (uint16_t)(t_cof_type<D>(E0 + e, sl) | ((t_cof_anchor<D>(E0 + e, sl, 0) + 1) << 5) |
                                              ((t_cof_anchor<D>(E0 + e, sl, 1) + 1) << 7) |
                                              ((t_cof_anchor<D>(E0 + e, sl, 2) + 1) << 9))
                                 : (uint16_t)0;
    }
  }
  __syncthreads();
}

// the 3 facet events of triangle (B, bt): kind 1 = critical edge (id), 2 = next triangle
// (id, key = anchor * 32 + type + 1), 0 = nothing; the three view reads are issued together
template <int D>
__device__ __forceinline__ void conn_expand(const ConnTab& T, const uint32_t* __restrict__ eview, const Grid& g,
                                            int64_t B, int bt, int (&ck)[3], uint64_t (&cid)[3],
                                            unsigned long long (&ckey)[3]) {
  constexpr int T0 = t_first_of_dim_c<D>(2), E0 = t_first_of_dim_c<D>(1);
  uint32_t tf[3], ev[3];
  int64_t E[3];
#pragma unroll
  for (int j = 0; j < 3; j++) {
    tf[j] = T.tf[(bt - T0) * 3 + j];
    E[j] = B + mask_delta(g, (int)(tf[j] & 7));
    ev[j] = (__ldg(eview + E[j]) >> (4 * (int)(tf[j] >> 3))) & 15u;
  }
#pragma unroll
  for (int j = 0; j < 3; j++) {
    ck[j] = 0;
    const int e = (int)(tf[j] >> 3);
    if (ev[j] & 8u) { ck[j] = 1; cid[j] = cell_id<D>(E[j], E0 + e); continue; }
    const uint32_t sl = ev[j] & 7u;
    if (sl == 7u) continue;
    const uint32_t ec = T.ec[e * 8 + sl];
    const int nt = (int)(ec & 31);
    const int64_t Nb = E[j] + ((int)((ec >> 5) & 3) - 1) + ((int)((ec >> 7) & 3) - 1) * g.sy +
                       ((int)((ec >> 9) & 3) - 1) * g.sz;
    if (Nb == B && nt == bt) continue;
    ck[j] = 2;
    cid[j] = cell_id<D>(Nb, nt);
    ckey[j] = (unsigned long long)(Nb * 32 + nt) + 1ull;
  }
}

// Connector BFS, small case: one thread per 2-saddle, its queue (= its visited set:
// every visited triangle is enqueued exactly once) in shared memory, keys relative
// to the origin anchor (7 bits per axis + type; BFS depth <= CQ bounds the offsets),
// membership by a linear scan.  Saddles that reach more than CQ triangles set their
// overflow bit and go to the block-parallel pass.
#ifndef DMTZ_CQ
#define DMTZ_CQ 48
#endif
constexpr int CQ = DMTZ_CQ;
constexpr int CONN_THREADS = 128;
constexpr int CONN_CHUNK = 1024;                       // pool entries taken per atomic
constexpr uint64_t CONN_NOT_STORED = ~0ull - 1;        // terminal slot: events not in the pool
// a pool list of full 64-bit cell ids (two u32 per event; the warp-level connectors,
// whose extent can exceed the 7-bit relative keys of the thread level)
constexpr uint64_t CONN_WIDE = 1ull << 62;
constexpr long long CONN_BIG = 256;
// a list in the scratch pool (the upper part of the BFS scratch, which the write pass
// does not touch): always intact
constexpr uint64_t CONN_SCR = 1ull << 61;
constexpr uint64_t CONN_POS = ~(CONN_WIDE | CONN_SCR);   // stored lists longer than this: k_conn_copy_big (a warp each)
// the terminal slot of connector b says its events are in the pool, below pool_limit
// (u32 entries: the paths' region, written last) or at or above top_ok (2 x the CSR's
// cell count: never written) -- the write pass copies them (k_conn_copy) instead of
// redoing the BFS
__device__ __forceinline__ bool conn_stored(uint64_t p, long long len, int64_t pool_limit, int64_t top_ok) {
  if (p >= CONN_NOT_STORED) return false;
  if (p & CONN_SCR) return true;
  const int64_t w = (p & CONN_WIDE) ? 2 : 1;
  const int64_t q = (int64_t)(p & CONN_POS);
  return q + w * len <= pool_limit || q >= top_ok;
}
// IDX: int when the grid has < 2^31 vertices (32-bit index arithmetic), else int64_t
template <int D, typename IDX>
__global__ void __launch_bounds__(CONN_THREADS)
k_conn_small(const uint32_t* __restrict__ eview, Grid g, int64_t b0, int64_t nb,
             const uint64_t* __restrict__ origin, uint64_t* __restrict__ jterm, long long* __restrict__ off,
             uint64_t* __restrict__ cells, bool write, unsigned int* __restrict__ overflow, int64_t conn_base,
             uint32_t* __restrict__ pool, unsigned long long* __restrict__ pool_top, int64_t pool_cap,
             int64_t pool_limit, int cq_lim, int64_t top_ok) {
  __shared__ uint32_t sq[CQ][CONN_THREADS];
  uint32_t* q = &sq[0][threadIdx.x];   // q[k * CONN_THREADS]: conflict-free columns
  // triangle -> facet edges (dm | edge index << 3); edge slot -> cofacet (type | anchor delta + 1)
  constexpr int T0 = t_first_of_dim_c<D>(2), E0 = t_first_of_dim_c<D>(1);
  __shared__ uint8_t s_tf[12 * 3];
  __shared__ uint16_t s_ec[7 * 8];
  if constexpr (D == 3) {
    if (threadIdx.x == 0) {
#pragma unroll
    for (int tt = 0; tt < 12; tt++)
#pragma unroll
      for (int j = 0; j < 3; j++)
        s_tf[tt * 3 + j] = (uint8_t)(t_facet<D>(T0 + tt, j, 0) | ((t_facet<D>(T0 + tt, j, 1) - E0) << 3));
#pragma unroll
    for (int e = 0; e < 7; e++)
#pragma unroll
      for (int sl = 0; sl < 8; sl++)
        s_ec[e * 8 + sl] = sl < t_nlink<D>(E0 + e)
                               ? (uint16_t)(t_cof_type<D>(E0 + e, sl) | ((t_cof_anchor<D>(E0 + e, sl, 0) + 1) << 5) |
                                            ((t_cof_anchor<D>(E0 + e, sl, 1) + 1) << 7) |
                                            ((t_cof_anchor<D>(E0 + e, sl, 2) + 1) << 9))
                               : (uint16_t)0;
    }
  }
  __shared__ IDX s_dm[8];   // index offset of each corner delta of {0,1}^3
  if (threadIdx.x < 8) s_dm[threadIdx.x] = (IDX)mask_delta(g, (int)threadIdx.x);
  __syncthreads();
  const IDX sy = (IDX)g.sy, sz = (IDX)g.sz;
  auto key = [](int dx, int dy, int dz, int ty) {
    return (uint32_t)(dx + 64) | ((uint32_t)(dy + 64) << 7) | ((uint32_t)(dz + 64) << 14) | ((uint32_t)ty << 21);
  };
  // Event pool (count pass): each thread appends the events of its connectors to a
  // chunk of the pool (taken with one atomic per CONN_CHUNK entries), and the branch's
  // terminal slot keeps the pool position until the write pass, which then copies the
  // events instead of redoing the BFS.  Event = 32-bit key relative to the origin
  // anchor, bit 31 set for a reached critical edge.
  uint32_t* chunk = nullptr;
  int chunk_left = 0;
  for (int64_t b = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t a;
    int t;
    id_cell<D>(origin[b], a, t);
    uint64_t* out = write ? cells + off[b] : nullptr;
    if (write) {   // stored by the count pass: k_conn_copy writes it
      const uint64_t p = jterm[b];
      if (conn_stored(p, off[b + 1] - off[b], pool_limit, top_ok)) continue;
    }
    // count pass: room for the connector's events (<= 3 per visited triangle)
    uint32_t* ev_out = nullptr;
    if (!write && pool) {
      if (chunk_left < 3 * CQ) {
        const unsigned long long p = atomicAdd(pool_top, (unsigned long long)CONN_CHUNK);
        if ((int64_t)(p + CONN_CHUNK) <= pool_cap) { chunk = pool + p; chunk_left = CONN_CHUNK; }
        else { chunk = nullptr; chunk_left = 0; }
      }
      ev_out = chunk;
    }
    int head = 0, tail = 1;
    int64_t n = 0;
    bool ovf = false;
    q[0] = key(0, 0, 0, t);
    // membership filter of the queued keys: two 64-bit Bloom words with independent
    // hashes rule out most new keys without the linear scan (which stays exact)
    uint64_t filt0 = 1ull << ((q[0] * 0x9E3779B1u) >> 26), filt1 = 1ull << ((q[0] * 0x85EBCA6Bu) >> 26);
    const IDX a_ = (IDX)a;
    while (head < tail && !ovf) {
      const uint32_t cur = q[(head++) * CONN_THREADS];
      const int bx = (int)(cur & 127) - 64, by = (int)((cur >> 7) & 127) - 64, bz = (int)((cur >> 14) & 127) - 64;
      const int bt = (int)(cur >> 21);
      const IDX B = a_ + (IDX)bx + (IDX)by * sy + (IDX)bz * sz;
      // the triangle's 3 facet edges: all three views read at once (independent loads)
      uint32_t tf[3], ev[3];
      IDX E[3];
#pragma unroll
      for (int j = 0; j < 3; j++) {
        tf[j] = s_tf[(bt - T0) * 3 + j];
        E[j] = B + s_dm[tf[j] & 7];
        ev[j] = (__ldg(eview + E[j]) >> (4 * (int)(tf[j] >> 3))) & 15u;
      }
#pragma unroll
      for (int j = 0; j < 3; j++) {
        const int dm = (int)(tf[j] & 7), e = (int)(tf[j] >> 3);
        if (ev[j] & 8u) {  // critical edge: a reached 1-saddle
          if (write) out[n] = cell_id<D>((int64_t)E[j], E0 + e);
          else if (ev_out) ev_out[n] = key(bx + (dm & 1), by + ((dm >> 1) & 1), bz + ((dm >> 2) & 1), E0 + e) | 0x80000000u;
          n++;
          continue;
        }
        const uint32_t sl = ev[j] & 7u;
        if (sl == 7u) continue;  // paired down with a vertex: the path stops
        const uint32_t ec = s_ec[e * 8 + sl];
        const int nt = (int)(ec & 31);
        const int nx_ = bx + (dm & 1) + (int)((ec >> 5) & 3) - 1, ny_ = by + ((dm >> 1) & 1) + (int)((ec >> 7) & 3) - 1,
                  nz_ = bz + ((dm >> 2) & 1) + (int)((ec >> 9) & 3) - 1;
        const uint32_t k = key(nx_, ny_, nz_, nt);
        if (k == cur) continue;
        // membership: a 64-bit filter of the queued keys rules out most new keys without
        // the linear scan of the queue (which stays exact for the rest)
        const uint64_t fb0 = 1ull << ((k * 0x9E3779B1u) >> 26), fb1 = 1ull << ((k * 0x85EBCA6Bu) >> 26);
        if ((filt0 & fb0) && (filt1 & fb1)) {
          bool seen = false;
          for (int i = tail - 1; i >= 0 && !seen; i--) seen = q[i * CONN_THREADS] == k;
          if (seen) continue;
        }
        if (tail == cq_lim) { ovf = true; break; }   // cq_lim = CQ (tests: smaller)
        q[(tail++) * CONN_THREADS] = k;
        filt0 |= fb0;
        filt1 |= fb1;
        if (write) out[n] = cell_id<D>((int64_t)(a_ + (IDX)nx_ + (IDX)ny_ * sy + (IDX)nz_ * sz), nt);
        else if (ev_out) ev_out[n] = k;
        n++;
      }
    }
    if (ovf) {
      const int64_t cb = b - conn_base;
      atomicOr(overflow + (cb >> 5), 1u << (cb & 31));
      if (!write) jterm[b] = CONN_NOT_STORED;
      continue;
    }
    if (!write) {
      off[b] = n;
      if (ev_out) {
        jterm[b] = (uint64_t)(ev_out - pool);
        chunk += n;
        chunk_left -= (int)n;
      } else {
        jterm[b] = CONN_NOT_STORED;
      }
    } else {
      jterm[b] = CELL_BOUNDARY;
    }
  }
}

// Write pass of the connectors stored by the count pass: a warp takes 32 consecutive
// connector branches and copies their events (pool keys -> cell ids) cooperatively,
// lane i handling event i of the 32 lists laid end to end, so the cell writes -- the
// lists are contiguous in the CSR -- are coalesced.
template <int D>
__global__ void __launch_bounds__(256)
k_conn_copy(Grid g, int64_t b0, int64_t nb, const uint64_t* __restrict__ origin, uint64_t* __restrict__ jterm,
            const long long* __restrict__ off, uint64_t* __restrict__ cells, const uint32_t* __restrict__ pool,
            int64_t pool_limit, int64_t top_ok, uint32_t* __restrict__ big, unsigned long long* __restrict__ n_big,
            int64_t big_cap, const uint32_t* __restrict__ spool) {
  __shared__ long long s_pre[8][33];
  __shared__ const uint32_t* s_src[8][32];
  __shared__ long long s_out[8][32], s_anc[8][32];
  __shared__ bool s_wide[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = b0 + warp * 32; base < nb; base += nwarps * 32) {
    const int64_t b = base + lane;
    long long len = 0;
    if (b < nb) {
      const uint64_t pp = jterm[b];
      const long long o0 = off[b], o1 = off[b + 1];
      bool mine = conn_stored(pp, o1 - o0, pool_limit, top_ok);
      if (mine && o1 - o0 > CONN_BIG && big) {   // a long list: k_conn_copy_big, many blocks on it
        const unsigned long long k = atomicAdd(n_big, 1ull);
        if ((int64_t)k < big_cap) {
          big[k] = (uint32_t)(b - b0);
          mine = false;
        }
      }
      if (mine) {
        len = o1 - o0;
        int64_t an;
        int t;
        id_cell<D>(origin[b], an, t);
        s_src[w][lane] = ((pp & CONN_SCR) ? spool : pool) + (pp & CONN_POS);
        s_wide[w][lane] = (pp & CONN_WIDE) != 0;
        s_out[w][lane] = o0;
        s_anc[w][lane] = an;
        jterm[b] = CELL_BOUNDARY;
      }
    }
    long long inc = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    s_pre[w][lane + 1] = inc;
    if (lane == 0) s_pre[w][0] = 0;
    __syncwarp();
    const long long total = s_pre[w][32];
    for (long long i = lane; i < total; i += 32) {
      int j = 0;   // the list holding event i: the last j with s_pre[j] <= i
#pragma unroll
      for (int st = 16; st > 0; st >>= 1)
        if (s_pre[w][j + st] <= i) j += st;
      const long long k = i - s_pre[w][j];
      const uint32_t* src = s_src[w][j];
      if (s_wide[w][j]) {   // wide list: the 64-bit cell ids
        cells[s_out[w][j] + k] = (uint64_t)src[2 * k] | ((uint64_t)src[2 * k + 1] << 32);
      } else {
        const uint32_t e = src[k];
        const int ex = (int)(e & 127) - 64, ey = (int)((e >> 7) & 127) - 64, ez = (int)((e >> 14) & 127) - 64;
        cells[s_out[w][j] + k] = cell_id<D>(s_anc[w][j] + ex + ey * g.sy + ez * g.sz, (int)((e >> 21) & 31));
      }
    }
    __syncwarp();
  }
}

// the long stored lists k_conn_copy left (big[0 .. *n_big), connector indices from b0):
// a warp per list (k_conn_copy's 32-lists-per-warp groups serialise long lists)
template <int D>
__global__ void __launch_bounds__(256)
k_conn_copy_big(Grid g, int64_t b0, const uint64_t* __restrict__ origin, uint64_t* __restrict__ jterm,
                const long long* __restrict__ off, uint64_t* __restrict__ cells, const uint32_t* __restrict__ pool,
                const uint32_t* __restrict__ big, const unsigned long long* __restrict__ n_big, int64_t big_cap,
                const uint32_t* __restrict__ spool) {
  const int64_t n = (int64_t)*n_big < big_cap ? (int64_t)*n_big : big_cap;
  const int lane = threadIdx.x & 31;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n;
       it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = b0 + big[it];
    const uint64_t pp = jterm[b];
    const long long o0 = off[b], len = off[b + 1] - o0;
    const uint32_t* src = ((pp & CONN_SCR) ? spool : pool) + (pp & CONN_POS);
    if (pp & CONN_WIDE) {
      for (long long k = lane; k < len; k += 32)
        cells[o0 + k] = (uint64_t)src[2 * k] | ((uint64_t)src[2 * k + 1] << 32);
    } else {   // thread-level list: keys relative to the origin anchor
      int64_t an;
      int t;
      id_cell<D>(origin[b], an, t);
      for (long long k = lane; k < len; k += 32) {
        const uint32_t e = src[k];
        const int ex = (int)(e & 127) - 64, ey = (int)((e >> 7) & 127) - 64, ez = (int)((e >> 14) & 127) - 64;
        cells[o0 + k] = cell_id<D>(an + ex + ey * g.sy + ez * g.sz, (int)((e >> 21) & 31));
      }
    }
  }
}

__global__ void k_conn_big_done(int64_t b0, uint64_t* __restrict__ jterm, const uint32_t* __restrict__ big,
                                const unsigned long long* __restrict__ n_big, int64_t big_cap) {
  const int64_t n = (int64_t)*n_big < big_cap ? (int64_t)*n_big : big_cap;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    jterm[b0 + big[i]] = CELL_BOUNDARY;
}

// Connector BFS, mid-size case: one warp per 2-saddle, queue (WQ entries) and a
// visited hash set (WH slots) in shared memory.  Same batch rule as the block
// kernel below (the batch = the next <= 32 queue entries; a discovered triangle is
// new iff it was not seen before the batch and this is its first occurrence in
// (entry, facet) order, decided by an atomicMin of batch << 7 | candidate on its
// slot's owner word), so the events come out in the sequential FIFO order.
constexpr int WQ = 512, WH = 1024, CONNW_WARPS = 4;
// per warp: hash keys (u32: the triangle relative to the origin anchor, 8 bits per axis
// + type, bit 31 set), owner words (u32), and the queue as hash slots (u16) -- 9 KB, so
// 6 blocks (24 warps) fit an SM (u64 keys: 13 KB, 4 blocks).  A triangle more than 127
// anchors from the origin on an axis sends the saddle to the block level.
constexpr size_t CONNW_WARP_BYTES = (size_t)WH * 4 + WH * 4 + WQ * 2;
constexpr size_t CONNW_SMEM = (size_t)CONNW_WARPS * CONNW_WARP_BYTES;
template <int D>
__global__ void __launch_bounds__(CONNW_WARPS * 32)
k_conn_warp(const uint32_t* __restrict__ eview, Grid g, const uint32_t* __restrict__ list,
            int64_t nlist, int64_t conn_base, const uint64_t* __restrict__ origin, uint64_t* __restrict__ jterm,
            long long* __restrict__ off, uint64_t* __restrict__ cells, bool write,
            unsigned int* __restrict__ overflow, int wq_lim, uint64_t* __restrict__ stage,
            uint32_t* __restrict__ pool, unsigned long long* __restrict__ pool_top, int64_t pool_cap,
            uint64_t pool_flag, unsigned long long* __restrict__ next_item) {
  // count pass with a pool (stage != nullptr): the connector's events (cell ids) go to the
  // warp's staging slot (3 WQ entries) and, once complete, to an exact-size pool list
  extern __shared__ uint32_t smw[];
  __shared__ ConnTab CT;
  __shared__ int64_t s_dmw[8];
  conn_tables_init<D>(CT);
  if (threadIdx.x < 8) s_dmw[threadIdx.x] = mask_delta(g, (int)threadIdx.x);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* keys = smw + (size_t)wid * (CONNW_WARP_BYTES / 4);
  uint32_t* owner = keys + WH;
  uint16_t* queue = (uint16_t*)(owner + WH);  // queue entry = the hash slot of its key
  for (int i = lane; i < WH; i += 32) { keys[i] = 0u; owner[i] = 0xFFFFFFFFu; }
  __syncwarp();
  constexpr int T0 = t_first_of_dim_c<D>(2), E0 = t_first_of_dim_c<D>(1);
  auto rkey = [](int dx, int dy, int dz, int ty) {
    return (uint32_t)(dx + 128) | ((uint32_t)(dy + 128) << 8) | ((uint32_t)(dz + 128) << 16) | ((uint32_t)ty << 24) |
           0x80000000u;
  };
  auto hslot = [](uint32_t k) { return (int)((k * 0x9E3779B1u) >> 22); };  // 10 bits
  auto find_or_insert = [&](uint32_t k) -> int {
    const int h = hslot(k);
    for (int p = 0; p < WH / 2; p++) {
      const int i = (h + p) & (WH - 1);
      const uint32_t v = atomicCAS(keys + i, 0u, k);
      if (v == 0u || v == k) return i;
    }
    return -1;
  };
  const int64_t sy = g.sy, sz = g.sz;
  for (;;) {   // saddles taken dynamically, a warp at a time (next_item zeroed before the launch)
    unsigned long long lv = 0;
    if (lane == 0) lv = atomicAdd(next_item, 1ull);
    const int64_t li = (int64_t)__shfl_sync(0xffffffffu, lv, 0);
    if (li >= nlist) break;
    const int64_t cb = list[li], b = conn_base + cb;
    int64_t a0;
    int t0;
    id_cell<D>(origin[b], a0, t0);
    uint64_t* stg = stage ? stage + (((int64_t)blockIdx.x * CONNW_WARPS + wid) * (3 * WQ)) : nullptr;
    uint64_t* out = write ? cells + off[b] : stg;
    if (lane == 0) {
      const int s0 = find_or_insert(rkey(0, 0, 0, t0));
      owner[s0] = 0u;  // seen before every batch
      queue[0] = (uint16_t)s0;
    }
    __syncwarp();
    int head = 0, tail = 1;
    int64_t nev = 0;
    uint32_t batch = 1;
    bool ovf = false;
    while (head < tail) {
      const int K = tail - head < 32 ? tail - head : 32;
      int ckind[3] = {0, 0, 0}, cslot[3] = {-1, -1, -1};
      uint64_t cid[3] = {0, 0, 0};
      uint32_t ckey[3] = {0, 0, 0};
      bool bad = false;
      if (lane < K) {
        // the entry, relative to the origin anchor; its 3 facet edges read at once
        const uint32_t cur = keys[queue[head + lane]];
        const int bx = (int)(cur & 255) - 128, by = (int)((cur >> 8) & 255) - 128, bz = (int)((cur >> 16) & 255) - 128;
        const int bt = (int)((cur >> 24) & 31);
        const int64_t B = a0 + bx + by * sy + bz * sz;
        uint32_t tf[3], ev[3];
        int64_t E[3];
#pragma unroll
        for (int j = 0; j < 3; j++) {
          tf[j] = CT.tf[(bt - T0) * 3 + j];
          E[j] = B + s_dmw[tf[j] & 7];
          ev[j] = (__ldg(eview + E[j]) >> (4 * (int)(tf[j] >> 3))) & 15u;
        }
#pragma unroll
        for (int j = 0; j < 3; j++) {
          const int dm = (int)(tf[j] & 7), e = (int)(tf[j] >> 3);
          if (ev[j] & 8u) { ckind[j] = 1; cid[j] = cell_id<D>(E[j], E0 + e); continue; }
          const uint32_t sl = ev[j] & 7u;
          if (sl == 7u) continue;
          const uint32_t ec = CT.ec[e * 8 + sl];
          const int nt = (int)(ec & 31);
          const int ox = (dm & 1) + (int)((ec >> 5) & 3) - 1, oy = ((dm >> 1) & 1) + (int)((ec >> 7) & 3) - 1,
                    oz = ((dm >> 2) & 1) + (int)((ec >> 9) & 3) - 1;
          if (ox == 0 && oy == 0 && oz == 0 && nt == bt) continue;
          const int nx_ = bx + ox, ny_ = by + oy, nz_ = bz + oz;
          if (nx_ < -127 || nx_ > 127 || ny_ < -127 || ny_ > 127 || nz_ < -127 || nz_ > 127) { bad = true; continue; }
          ckind[j] = 2;
          cid[j] = cell_id<D>(B + ox + oy * sy + oz * sz, nt);
          ckey[j] = rkey(nx_, ny_, nz_, nt);
          const int slot = find_or_insert(ckey[j]);
          if (slot < 0) { bad = true; continue; }
          cslot[j] = slot;
          atomicMin(owner + slot, (batch << 7) | (uint32_t)(lane * 3 + j));
        }
      }
      __syncwarp();
      if (__any_sync(0xffffffffu, bad)) { ovf = true; break; }
      int ne = 0, nq = 0;
      bool isnew[3] = {false, false, false};
#pragma unroll
      for (int j = 0; j < 3; j++) {
        if (ckind[j] == 2 && owner[cslot[j]] == ((batch << 7) | (uint32_t)(lane * 3 + j))) { isnew[j] = true; nq++; }
        if (ckind[j] == 1 || isnew[j]) ne++;
      }
      int v = ne | (nq << 16), incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      const int tot_e = tot & 0xFFFF, tot_q = tot >> 16;
      if (tail + tot_q > wq_lim) { ovf = true; break; }   // wq_lim = WQ (tests: smaller)
      int pe = (incl - v) & 0xFFFF, pq = (incl - v) >> 16;
#pragma unroll
      for (int j = 0; j < 3; j++) {
        if (ckind[j] == 1 || isnew[j]) {
          if (out) out[nev + pe] = cid[j];
          pe++;
        }
        if (isnew[j]) { queue[tail + pq] = (uint16_t)cslot[j]; pq++; }
      }
      __syncwarp();
      nev += tot_e;
      tail += tot_q;
      head += K;
      batch++;
    }
    __syncwarp();
    if (ovf) {  // keys of the failing batch are not all queued: wipe the table
      for (int i = lane; i < WH; i += 32) { keys[i] = 0u; owner[i] = 0xFFFFFFFFu; }
      if (lane == 0) atomicOr(overflow + (cb >> 5), 1u << (cb & 31));
    } else {
      // clean the visited set: the queue holds exactly the occupied slots
      for (int i = lane; i < tail; i += 32) {
        const int sl = queue[i];
        keys[sl] = 0u;
        owner[sl] = 0xFFFFFFFFu;
      }
      if (lane == 0) {
        if (!write) off[b] = nev;
        else jterm[b] = CELL_BOUNDARY;
      }
      if (!write && stg) {  // the staged events -> an exact-size pool list (2 u32 per event)
        unsigned long long p = 0;
        if (lane == 0) p = atomicAdd(pool_top, (unsigned long long)(2 * nev));
        p = __shfl_sync(0xffffffffu, p, 0);
        const bool fits = (int64_t)(p + 2 * nev) <= pool_cap;
        if (fits)
          for (int64_t i = lane; i < nev; i += 32) {
            const uint64_t c = stg[i];
            pool[p + 2 * i] = (uint32_t)c;
            pool[p + 2 * i + 1] = (uint32_t)(c >> 32);
          }
        if (lane == 0) jterm[b] = fits ? (p | CONN_WIDE | pool_flag) : CONN_NOT_STORED;
      }
    }
    __syncwarp();
  }
}

// Block-parallel connector BFS for the saddles that outgrew a per-thread slot.
// Reproduces the sequential FIFO order exactly: a batch = the next (up to 256)
// queue entries, each producing its facet events in facet order; a discovered
// triangle is new iff it was never seen before this batch and this is its first
// occurrence in (entry, facet) order within the batch -- decided by an atomic
// max of ~(batch << 32 | candidate) on the visited slot's owner word.  A block
// scan then places events and new queue entries in that order.

__device__ __forceinline__ int64_t bfs_find_or_insert(unsigned long long* keys, int64_t hcap, unsigned long long k) {
  const unsigned long long h = (k * 0x9E3779B97F4A7C15ull) >> 20;
  for (int64_t p = 0; p < hcap / 2; p++) {
    const int64_t i = (int64_t)((h + p) & (unsigned long long)(hcap - 1));
    const unsigned long long v = atomicCAS(keys + i, 0ull, k);
    if (v == 0ull || v == k) return i;
  }
  return -1;
}
__device__ __forceinline__ int64_t bfs_find(const unsigned long long* keys, int64_t hcap, unsigned long long k) {
  const unsigned long long h = (k * 0x9E3779B97F4A7C15ull) >> 20;
  for (int64_t p = 0; p < hcap; p++) {
    const int64_t i = (int64_t)((h + p) & (unsigned long long)(hcap - 1));
    if (keys[i] == k) return i;
    if (keys[i] == 0ull) return -1;
  }
  return -1;
}

// set bits of words [w0, w1) -> list of bit indices (any order), words cleared; one atomic per warp
__global__ void k_bits_compact(uint32_t* __restrict__ bits, int64_t w0, int64_t w1, uint32_t* __restrict__ list,
                               unsigned long long* __restrict__ n_out) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = w0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane; base < w1;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = base + lane;
    uint32_t word = 0u;
    if (w < w1) {
      word = bits[w];
      if (word) bits[w] = 0u;
    }
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    unsigned long long pos = 0;
    if (lane == 31 && incl) pos = atomicAdd(n_out, (unsigned long long)incl);
    pos = __shfl_sync(0xffffffffu, pos, 31) + (unsigned long long)(incl - c);
    while (word) {
      const int b = __ffs(word) - 1;
      word &= word - 1u;
      list[pos++] = (uint32_t)(w * 32 + b);
    }
  }
}

// SH: the visited hash in shared memory (SB_HCAP u64 keys + u32 owner words; queues of
// at most SB_QMAX entries), the slot in global memory holding the queue only
constexpr int SB_HCAP = 16384, SB_QMAX = 8192;
constexpr size_t SB_SMEM = (size_t)SB_HCAP * 12;
// UN: unordered fill (tier-3 candidate traces, whose consumers -- the end multiset and
// the box -- do not depend on the order): a discovered triangle is new iff this thread's
// insert put it in the hash, positions come from shared atomics, one barrier per batch
template <int D, int BFS_THREADS, bool SH = false, bool UN = false>
__global__ void __launch_bounds__(BFS_THREADS)
k_walk_block(const uint32_t* __restrict__ eview, Grid g, const uint32_t* __restrict__ list,
             int64_t nlist, int64_t conn_base, const uint64_t* __restrict__ origin, uint64_t* __restrict__ jterm,
             long long* __restrict__ off, uint64_t* __restrict__ cells, bool write,
             unsigned long long* __restrict__ scratch, int64_t qcap, int64_t hcap,
             unsigned int* __restrict__ overflow, Counters* __restrict__ cnt, uint32_t* __restrict__ pool,
             int64_t pool_cap, const unsigned long long* __restrict__ bottom_top,
             unsigned long long* __restrict__ top_used, uint64_t pool_flag,
             unsigned long long* __restrict__ next_item) {
  // Count pass with a pool: each processed queue entry keeps its 3 facet outcomes in
  // the key's top bits (2 bits per facet: 1 reached edge, 2 new triangle), and a
  // completed BFS replays them into a wide event list taken from the top of the pool
  // (growing down); the write pass copies it when it lies above the CSR's cells.
  constexpr int QSH = 58;
  constexpr unsigned long long QMASK = (1ull << QSH) - 1ull;
  __shared__ int s_warp[32];
  __shared__ int s_flag;
  __shared__ long long s_base;
  // UN: (events, enqueues) of batch b in s_cnt[b % 3]; thread 0 zeroes the next one during
  // batch b -- last read before batch b - 1's barrier ended (two would race)
  __shared__ int s_cnt[3][2];
  __shared__ ConnTab CT;
  conn_tables_init<D>(CT);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ unsigned long long s_hash[];
  if (SH) hcap = SB_HCAP;
  // a global slot: the queue, the keys and (FIFO only: UN needs no arbitration) the owners
  unsigned long long* queue = scratch + (int64_t)blockIdx.x * (SH ? qcap : UN ? qcap + hcap : qcap + 2 * hcap);
  unsigned long long* keys = SH ? s_hash : queue + qcap;
  unsigned long long* owner = (SH || UN) ? nullptr : keys + hcap;
  uint32_t* owner_s = SH ? (uint32_t*)(s_hash + SB_HCAP) : nullptr;
  if (SH) {
    for (int i = tid; i < SB_HCAP; i += BFS_THREADS) { keys[i] = 0ull; owner_s[i] = 0u; }
    __syncthreads();
  }
  auto key = [](int64_t an, int ty) { return (unsigned long long)(an * 32 + ty) + 1ull; };
  // connectors are taken dynamically (next_item, zeroed before the launch): a block that
  // finishes a small BFS takes the next saddle at once (static strides left the level
  // waiting for the blocks that drew several large ones)
  __shared__ int64_t s_li;
  for (;;) {
    if (tid == 0) s_li = (int64_t)atomicAdd(next_item, 1ull);
    __syncthreads();
    const int64_t li = s_li;
    if (li >= nlist) break;
    const int64_t cb = list[li], b = conn_base + cb;
    int64_t a0;
    int t0;
    id_cell<D>(origin[b], a0, t0);
    uint64_t* out = write ? cells + off[b] : nullptr;
    if (tid == 0) {
      queue[0] = key(a0, t0);
      const int64_t sl = bfs_find_or_insert(keys, hcap, key(a0, t0));
      if (SH) owner_s[sl] = ~0u;  // seen before every batch
      else if (!UN) owner[sl] = ~0ull;
      s_flag = 0;
    }
    __syncthreads();
    int64_t head = 0, tail = 1, nev = 0;
    unsigned long long batch = 1;
    if constexpr (UN) {
      if (tid < 6) s_cnt[tid >> 1][tid & 1] = 0;
      __syncthreads();
      while (head < tail) {
        const int64_t K = tail - head < BFS_THREADS ? tail - head : BFS_THREADS;
        int ckind[3] = {0, 0, 0};
        uint64_t cid[3] = {0, 0, 0};
        unsigned long long ckey[3] = {0, 0, 0};
        bool isnew[3] = {false, false, false};
        int nmine = 0, qmine = 0;
        if (tid < K) {
          const unsigned long long cur = queue[head + tid] - 1ull;
          conn_expand<D>(CT, eview, g, (int64_t)(cur / 32), (int)(cur % 32), ckind, cid, ckey);
#pragma unroll
          for (int j = 0; j < 3; j++) {
            if (ckind[j] == 1) { nmine++; continue; }
            if (ckind[j] != 2) continue;
            // new iff this insert claimed the empty slot
            const unsigned long long hh = (ckey[j] * 0x9E3779B97F4A7C15ull) >> 20;
            bool done = false;
            for (int64_t p = 0; p < hcap / 2 && !done; p++) {
              const int64_t i = (int64_t)((hh + p) & (unsigned long long)(hcap - 1));
              const unsigned long long v = atomicCAS(keys + i, 0ull, ckey[j]);
              if (v == 0ull) { isnew[j] = true; done = true; }
              else if (v == ckey[j]) done = true;
            }
            if (!done) s_flag = 1;
            if (isnew[j]) { nmine++; qmine++; }
          }
          if (!write && pool) {
            unsigned long long oc = 0;
#pragma unroll
            for (int j = 0; j < 3; j++) oc |= (unsigned long long)(ckind[j] == 1 ? 1 : isnew[j] ? 2 : 0) << (2 * j);
            queue[head + tid] = (queue[head + tid] & QMASK) | (oc << QSH);
          }
        }
        int* C = s_cnt[batch % 3];
        int pe = nmine ? atomicAdd(&C[0], nmine) : 0;
        int pq = qmine ? atomicAdd(&C[1], qmine) : 0;
        if (tail + pq + qmine > qcap) s_flag = 1;
        else {
#pragma unroll
          for (int j = 0; j < 3; j++) {
            if (ckind[j] == 1 || isnew[j]) {
              if (write) out[nev + pe] = cid[j];
              pe++;
            }
            if (isnew[j]) { queue[tail + pq] = ckey[j]; pq++; }
          }
        }
        if (tid == 0) { s_cnt[(batch + 1) % 3][0] = 0; s_cnt[(batch + 1) % 3][1] = 0; }
        __syncthreads();
        if (s_flag) break;
        nev += C[0];
        tail += C[1];
        head += K;
        batch++;
      }
    } else
    while (head < tail) {
      const int64_t K = tail - head < BFS_THREADS ? tail - head : BFS_THREADS;
      // candidates of entry head + tid: per facet j, kind 1 = reached edge, 2 = triangle
      int ckind[3] = {0, 0, 0};
      uint64_t cid[3] = {0, 0, 0};
      unsigned long long ckey[3] = {0, 0, 0};
      int64_t cslot[3] = {-1, -1, -1};
      if (tid < K) {
        const unsigned long long cur = queue[head + tid] - 1ull;
        const int64_t B = (int64_t)(cur / 32);
        const int bt = (int)(cur % 32);
        conn_expand<D>(CT, eview, g, B, bt, ckind, cid, ckey);
#pragma unroll
        for (int j = 0; j < 3; j++) {
          if (ckind[j] != 2) continue;
          const int64_t slot = bfs_find_or_insert(keys, hcap, ckey[j]);
          if (slot < 0) { s_flag = 1; continue; }
          cslot[j] = slot;
          if (SH) atomicMax(owner_s + slot, ~(((uint32_t)batch << 12) | (uint32_t)(tid * 3 + j)));
          else atomicMax(owner + slot, ~((batch << 32) | (unsigned long long)(tid * 3 + j)));
        }
      }
      __syncthreads();
      if (s_flag) break;
      int nmine = 0, qmine = 0;
      bool isnew[3] = {false, false, false};
      for (int j = 0; j < 3; j++) {
        if (ckind[j] == 1) nmine++;
        if (ckind[j] == 2 &&
            (SH ? owner_s[cslot[j]] == ~(((uint32_t)batch << 12) | (uint32_t)(tid * 3 + j))
                : owner[cslot[j]] == ~((batch << 32) | (unsigned long long)(tid * 3 + j)))) {
          isnew[j] = true;
          nmine++;
          qmine++;
        }
      }
      if (!write && pool && tid < K) {   // this entry's outcomes, for the replay into the pool
        unsigned long long oc = 0;
#pragma unroll
        for (int j = 0; j < 3; j++) oc |= (unsigned long long)(ckind[j] == 1 ? 1 : isnew[j] ? 2 : 0) << (2 * j);
        queue[head + tid] = (queue[head + tid] & QMASK) | (oc << QSH);
      }
      // block exclusive scan of (events, enqueues) packed in one int
      int v = nmine | (qmine << 16), incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) s_warp[wid] = incl;
      __syncthreads();
      int wbase = 0, tot = 0;
      for (int w2 = 0; w2 < BFS_THREADS / 32; w2++) {
        const int x = s_warp[w2];
        if (w2 < wid) wbase += x;
        tot += x;
      }
      const int ex = wbase + incl - v;
      int pe = ex & 0xFFFF, pq = ex >> 16;
      const int tot_e = tot & 0xFFFF, tot_q = tot >> 16;
      if (tail + tot_q > qcap) {
        if (tid == 0) s_flag = 1;
      } else {
        for (int j = 0; j < 3; j++) {
          if (ckind[j] == 1 || isnew[j]) {
            if (write) out[nev + pe] = cid[j];
            pe++;
          }
          if (isnew[j]) { queue[tail + pq] = ckey[j]; pq++; }
        }
      }
      __syncthreads();
      if (s_flag) break;
      nev += tot_e;
      tail += tot_q;
      head += K;
      batch++;
      __syncthreads();
    }
    const bool ovf = s_flag != 0;
    __syncthreads();
    bool stored = false;
    if (!ovf && !write && pool) {
      if (tid == 0) {
        const unsigned long long need = 2ull * (unsigned long long)nev;
        const unsigned long long old = atomicAdd(top_used, need);
        const long long q = pool_cap - (long long)(old + need);
        s_base = (nev > 0 && q >= (long long)*(volatile const unsigned long long*)bottom_top) ? q : -1;
      }
      __syncthreads();
      const long long base = s_base;
      stored = base >= 0;
      if (stored) {
        // the events in BFS order: entry by entry, its facets in order
        long long pos = 0;
        for (int64_t i0 = 0; i0 < tail; i0 += BFS_THREADS) {
          const int64_t i = i0 + tid;
          const unsigned long long qe = i < tail ? queue[i] : 0ull;
          const unsigned oc = (unsigned)(qe >> QSH);
          const int c = (oc & 3u ? 1 : 0) + ((oc >> 2) & 3u ? 1 : 0) + ((oc >> 4) & 3u ? 1 : 0);
          int incl = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
          }
          if (lane == 31) s_warp[wid] = incl;
          __syncthreads();
          int wbase = 0, tot = 0;
          for (int w2 = 0; w2 < BFS_THREADS / 32; w2++) {
            const int x = s_warp[w2];
            if (w2 < wid) wbase += x;
            tot += x;
          }
          if (c) {
            const unsigned long long cur = (qe & QMASK) - 1ull;
            int ck[3] = {0, 0, 0};
            uint64_t cid[3] = {0, 0, 0};
            unsigned long long ckey[3] = {0, 0, 0};
            conn_expand<D>(CT, eview, g, (int64_t)(cur / 32), (int)(cur % 32), ck, cid, ckey);
            long long p = base + 2 * (pos + wbase + incl - c);
#pragma unroll
            for (int j = 0; j < 3; j++)
              if ((oc >> (2 * j)) & 3u) {
                pool[p] = (uint32_t)cid[j];
                pool[p + 1] = (uint32_t)(cid[j] >> 32);
                p += 2;
              }
          }
          pos += tot;
          __syncthreads();
        }
      }
    }
    // clean the visited set: find every queued key's slot first, then clear
    for (int64_t i = tid; i < tail; i += BFS_THREADS) {
      const int64_t sl = bfs_find(keys, hcap, queue[i] & QMASK);
      queue[i] = (unsigned long long)sl;
    }
    __syncthreads();
    for (int64_t i = tid; i < tail; i += BFS_THREADS) {
      const long long sl = (long long)queue[i];
      if (sl >= 0) {
        keys[sl] = 0ull;
        if (SH) owner_s[sl] = 0u;
        else if (!UN) owner[sl] = 0ull;
      }
    }
    __syncthreads();
    if (ovf) {
      // keys inserted beyond the queue (the failing batch) are not tracked: wipe the whole slot
      for (int64_t i = tid; i < hcap; i += BFS_THREADS) {
        keys[i] = 0ull;
        if (SH) owner_s[i] = 0u;
        else if (!UN) owner[i] = 0ull;
      }
      if (tid == 0) atomicOr(overflow + (cb >> 5), 1u << (cb & 31));
    } else if (tid == 0) {
      if (!write) {
        off[b] = nev;
        jterm[b] = stored ? ((uint64_t)s_base | CONN_WIDE | pool_flag) : CONN_NOT_STORED;
      } else {
        jterm[b] = CELL_BOUNDARY;
      }
    }
    __syncthreads();
  }
}

inline size_t trace_scratch_bytes(const Grid&, int) { return 0; }  // reuses free workspace regions

// walks of the descending branches [0, nasc0) and the ascending ones [nasc0, nb):
// descending paths by k_walk (one thread per branch: short, cheap steps -- the refill
// bookkeeping of k_walk_dyn doubled their time on C4), ascending ones by k_walk_dyn
// (C4 76 -> 65 ms); DMTZ_WALK_STATIC=1: k_walk for both
template <int D>
cudaError_t launch_walk(const TraceViews& V, const Grid& g, int64_t nasc0, int64_t nb, const TraceArgs& A,
                        long long* off, bool write, Counters* dc, int threads, cudaStream_t s) {
  const char* ws = getenv("DMTZ_WALK_STATIC");
  const bool stat = ws && ws[0] == '1';
  const int64_t n_static = stat ? nb : nasc0;
  if (n_static > 0)
    k_walk<D><<<(unsigned)((n_static + threads - 1) / threads), threads, 0, s>>>(
        V, g, 0, n_static, A.out_origin, A.out_kind, A.out_terminal, off, A.out_cells, write, dc);
  if (n_static < nb) {
    cudaError_t e = cudaMemsetAsync(&dc->pad[8], 0, 8, s);
    if (e != cudaSuccess) return e;
    const int64_t want = (nb - n_static + 127) / 128;
    const unsigned grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
    k_walk_dyn<D><<<grid, 128, 0, s>>>(V, g, n_static, nb, A.out_origin, A.out_kind, A.out_terminal, off,
                                       A.out_cells, write, dc, &dc->pad[8]);
  }
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- driver
#define TCK(x)                                  \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return e_;           \
  } while (0)

inline cudaError_t scan_i64(long long* a, int64_t n, unsigned long long* bsum, unsigned long long* total,
                            unsigned long long* host_total, cudaStream_t s) {
  const int64_t nb = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
  if (n > 0) {
    TCK(cudaMemsetAsync(bsum, 0, (size_t)(nb + 1) * 8, s));
    k_scan_lb<<<(unsigned)nb, SCL_THREADS, 0, s>>>(a, n, bsum, total);
  } else {
    TCK(cudaMemsetAsync(total, 0, 8, s));
  }
  TCK(cudaGetLastError());
  TCK(cudaMemcpyAsync(host_total, total, 8, cudaMemcpyDeviceToHost, s));
  TCK(cudaStreamSynchronize(s));
  return cudaSuccess;
}

inline dim3 trace_anchor_grid(const Grid& g) {
  int64_t bx = (g.nx + 127) / 128, by = g.ny < 65535 ? g.ny : 65535, bz = g.nz < 65535 ? g.nz : 65535;
  return dim3((unsigned)bx, (unsigned)by, (unsigned)bz);
}

template <int D>
cudaError_t run_trace(TraceArgs& A, cudaStream_t s) {
  const Grid& g = A.g;
  Counters* dc = A.cnt;
  Counters* hc = A.host_cnt;
  // DMTZ_TRACE_TIMES=1: phase times on stderr (synchronising after each phase)
  static const bool timing = [] { const char* e = getenv("DMTZ_TRACE_TIMES"); return e && e[0] == '1'; }();
  char tlog[1024];
  int tlen = 0;
  auto t_prev = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    if (tlen < 900)
      tlen += snprintf(tlog + tlen, sizeof tlog - tlen, " %s %.2f", what,
                       std::chrono::duration<double, std::milli>(now - t_prev).count());
    t_prev = now;
  };
  struct Flush {
    bool on; char* buf;
    ~Flush() { if (on) fprintf(stderr, "trace ms:%s\n", buf); }
  } flush_{timing, tlog};
  tlog[0] = 0;
  TCK(cudaMemsetAsync(dc, 0, sizeof(Counters), s));
  // compact views at the front of the BFS scratch (the block BFS gets the rest), with the
  // critical masks in the same pass
  TraceViews V;
  {
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    char* p = (char*)A.bfs;
    const size_t nb_nib = al((size_t)(g.N + 1) / 2), nb_w = al((size_t)g.N * 4);
    const size_t need = nb_nib + nb_w * (D == 3 ? 2 : 1);
    if (need + 64 * 1024 > A.bfs_bytes) return cudaErrorMemoryAllocation;
    V.vnib = (uint8_t*)p;
    V.tpair = (uint32_t*)(p + nb_nib);
    V.eview = D == 3 ? (uint32_t*)(p + nb_nib + nb_w) : nullptr;
    A.bfs = (unsigned long long*)(p + need);
    A.bfs_bytes -= need;
    const int64_t pairs = (g.N + 1) / 2;
    k_trace_views_crit<D><<<(unsigned)((pairs + 255) / 256 < 148 * 32 ? (pairs + 255) / 256 : 148 * 32), 256, 0,
                            s>>>(A.codes, A.crit, g, V);
    TCK(cudaGetLastError());
  }
  mark("views");
  long long* pre = A.pre;
  unsigned long long* total = &dc->pad[0];
  const int kinds_list[3] = {1, 2, 4};
  int64_t nbk[3] = {0, 0, 0};
  // origins: per kind, block totals of BT_TILE-anchor tiles (kept, scanned) -> emission
  // only the tiles holding origin anchors [a_lo, a_hi) (range traces: one slab of the grid)
  const int64_t a_end = A.a_hi < g.N ? A.a_hi : g.N;
  const int64_t tile0 = A.a_lo > 0 ? A.a_lo / BT_TILE : 0;
  const int64_t tile1 = a_end > A.a_lo ? (a_end + BT_TILE - 1) / BT_TILE : tile0 + 1;
  const int64_t ntiles = tile1 - tile0;
  if ((3 * ntiles + 8) * 8 > (int64_t)A.pre_bytes) return cudaErrorMemoryAllocation;
  unsigned long long* tsum[3] = {(unsigned long long*)pre, (unsigned long long*)pre + ntiles,
                                 (unsigned long long*)pre + 2 * ntiles};
  const bool given = A.given_nbk[0] >= 0;
  if (given) {
    for (int ki = 0; ki < 3; ki++) nbk[ki] = A.given_nbk[ki];
  } else {
    for (int ki = 0; ki < 3; ki++) {
      const int kind = kinds_list[ki];
      if (!(A.kinds & (uint32_t)kind) || (kind == 4 && D != 3)) continue;
      k_branch_tiles<D><<<(unsigned)ntiles, BT_THREADS, 0, s>>>(A.crit, g, kind, A.a_lo, A.a_hi, tsum[ki], tile0);
      k_scan_top<<<1, 1024, 0, s>>>(tsum[ki], ntiles, total + ki);
      TCK(cudaGetLastError());
    }
    TCK(cudaMemcpyAsync(&hc->pad[0], total, 3 * 8, cudaMemcpyDeviceToHost, s));
    TCK(cudaStreamSynchronize(s));
    for (int ki = 0; ki < 3; ki++) {
      const int kind = kinds_list[ki];
      nbk[ki] = (!(A.kinds & (uint32_t)kind) || (kind == 4 && D != 3)) ? 0 : (int64_t)hc->pad[ki];
    }
  }
  const int64_t nb = nbk[0] + nbk[1] + nbk[2];
  A.n_branches = nb;
  mark("count-origins");
  if (nb > A.cap_b) return cudaSuccess;  // caller reports DMTZ_E_CAPACITY with the needed size
  if (nb == 0) {
    if (A.out_offsets) TCK(cudaMemsetAsync(A.out_offsets, 0, 8, s));
    TCK(cudaStreamSynchronize(s));
    return cudaSuccess;
  }
  int64_t base = 0;
  for (int ki = 0; ki < 3 && !given; ki++) {
    const int kind = kinds_list[ki];
    if (!nbk[ki]) continue;
    k_branch_tiles_emit<D><<<(unsigned)ntiles, BT_THREADS, 0, s>>>(A.crit, g, kind, A.a_lo, A.a_hi, tsum[ki], base,
                                                                   A.out_origin, A.out_kind, A.out_terminal, tile0);
    TCK(cudaGetLastError());
    base += nbk[ki];
  }
  mark("emit");
  // walks: lengths -> offsets -> cells.  Connector slots: one per thread of the launch.
  int* ovf = (int*)pre;
  unsigned long long* sc = A.bfs;
  const int64_t words_all = (int64_t)(A.bfs_bytes / 8);
  // a connector visits at most the 12 N triangles; small grids get small slots
  const int threads = 128;
  const int64_t conn_base = nbk[0] + nbk[1];
  const int64_t ovf_words = (nbk[2] + 31) / 32;
  const int64_t pre_words = (int64_t)(A.pre_bytes / 8);
  if (nbk[2] && (ovf_words + 2) * 4 + 64 * 8 > pre_words * 8) return cudaErrorMemoryAllocation;
  const int64_t list_cap = (pre_words * 8 - (ovf_words + 2) * 4) / 4;
  const int64_t blocks_path = conn_base > 0 ? (conn_base + threads - 1) / threads : 0;
  long long* off = (long long*)A.out_offsets;
  // connector event pool: the (still unused) output cell buffer during the count pass.
  // The write pass copies the connectors first, then writes the paths over the pool;
  // an event list is copied only if it lies below off[conn_base] (the paths' region),
  // where the connectors' own output cannot overwrite it.
  const char* pe = getenv("DMTZ_CONN_POOL");
  uint32_t* pool = (A.out_cells && A.cap_c > 0 && nbk[2] && !(pe && pe[0] == '0')) ? (uint32_t*)A.out_cells : nullptr;
  int64_t pool_cap = pool ? 2 * A.cap_c : 0;
  if (const char* pc = getenv("DMTZ_CONN_POOL_CAP")) {  // tests: a small pool forces the fallback path
    const long long c = atoll(pc);
    if (c >= 0 && c < pool_cap) pool_cap = c;
  }
  int64_t pool_limit = 0;
  int64_t top_ok = INT64_MAX;   // write pass: 2 x the cell count (top-pool lists above it are intact)
  // test knobs (tests/test_gpu_parity.py forces every escalation level on small grids):
  // DMTZ_TEST_CQ / DMTZ_TEST_WQ shrink the thread / warp queues, DMTZ_TEST_BFS_GROW sets
  // the block level's slot growth (default 16), DMTZ_TEST_BFS_WORDS caps the scratch
  auto env_int = [](const char* n, long long dflt, long long lo, long long hi) {
    const char* e = getenv(n);
    if (!e) return dflt;
    long long v = atoll(e);
    return v < lo ? lo : v > hi ? hi : v;
  };
  const int cq_lim = (int)env_int("DMTZ_TEST_CQ", CQ, 1, CQ);
  const int wq_lim = (int)env_int("DMTZ_TEST_WQ", WQ, 4, WQ);
  const int64_t grow = env_int("DMTZ_TEST_BFS_GROW", 16, 2, 16);
  int64_t words = env_int("DMTZ_TEST_BFS_WORDS", words_all, 1024, words_all);
  // Scratch pool (full and range traces with a large scratch): the upper 3/4 of the BFS
  // scratch, which the write pass never touches, holds the wide event lists of the warp
  // and block levels -- intact whatever the CSR's size, so the write pass copies them
  // instead of redoing those BFS.  The block levels' slots keep the lower quarter.
  // DMTZ_SCRATCH_POOL=0: off (the lists then go to the output buffer's pools).
  uint32_t* spool = nullptr;
  int64_t spool_cap = 0;
  {
    const char* sp = getenv("DMTZ_SCRATCH_POOL");   // 0: off, 2: also on small scratch (tests)
    const int spm = sp ? atoi(sp) : 1;
    if (pool && !given && words == words_all && spm && (words_all >= (1ll << 24) || spm == 2)) {
      const int64_t keep = words_all / 4;
      spool = (uint32_t*)(sc + keep);
      spool_cap = 2 * (words_all - keep);
      words = keep;
    }
  }
  // the pool the warp / block levels use: (base, capacity, bottom counter, flag)
  uint32_t* wpool = spool ? spool : pool;
  const int64_t wpool_cap = spool ? spool_cap : pool_cap;
  unsigned long long* wpool_bottom = spool ? &dc->pad[5] : &dc->pad[2];
  const uint64_t wpool_flag = spool ? CONN_SCR : 0ull;
  for (int i = 0; i < 10; i++) A.level_counts[i] = 0;
  TCK(cudaMemsetAsync(&dc->pad[2], 0, 8, s));
  for (int pass = 0; pass < 2; pass++) {
    const bool write = pass == 1;
    TCK(cudaMemsetAsync(ovf, 0, (size_t)ovf_words * 4 + 4, s));
    if (blocks_path && !write)  // descending / ascending paths
      TCK(launch_walk<D>(V, g, nbk[0], conn_base, A, off, write, dc, threads, s));
    mark(write ? "W:start" : "C:paths");
    if (nbk[2]) {  // connectors: one thread per 2-saddle, small queues in shared memory
      const int64_t nbc = (nbk[2] + CONN_THREADS - 1) / CONN_THREADS;
      const unsigned cgrid = (unsigned)(nbc < 148 * 64 ? nbc : 148 * 64);
      if (g.N < (1ll << 31))
        k_conn_small<D, int><<<cgrid, CONN_THREADS, 0, s>>>(
            V.eview, g, conn_base, nb, A.out_origin, A.out_terminal, off, A.out_cells, write,
            (unsigned int*)ovf, conn_base, pool, &dc->pad[2], pool_cap, pool_limit, cq_lim, top_ok);
      else
        k_conn_small<D, int64_t><<<cgrid, CONN_THREADS, 0, s>>>(
            V.eview, g, conn_base, nb, A.out_origin, A.out_terminal, off, A.out_cells, write,
            (unsigned int*)ovf, conn_base, pool, &dc->pad[2], pool_cap, pool_limit, cq_lim, top_ok);
      if (write && pool) mark("small");
      if (write && pool) {  // the stored event lists (skipped above): a cooperative copy, which
                            // then marks them done -- after the BFS pass, which reads the marks
        const int64_t nw = (nbk[2] + 31) / 32;
        // long lists go to k_conn_copy_big (their indices in the overflow list area, which the
        // escalation below refills only afterwards), then their terminals are set
        uint32_t* big = (uint32_t*)(ovf + ovf_words + 1);
        TCK(cudaMemsetAsync(&dc->pad[4], 0, 8, s));
        k_conn_copy<D><<<(unsigned)((nw + 7) / 8 < 148 * 16 ? (nw + 7) / 8 : 148 * 16), 256, 0, s>>>(
            g, conn_base, nb, A.out_origin, A.out_terminal, off, A.out_cells, pool, pool_limit, top_ok, big,
            &dc->pad[4], list_cap, spool);
        k_conn_copy_big<D><<<148 * 8, 256, 0, s>>>(g, conn_base, A.out_origin, A.out_terminal, off, A.out_cells,
                                                 pool, big, &dc->pad[4], list_cap, spool);
        k_conn_big_done<<<16, 256, 0, s>>>(conn_base, A.out_terminal, big, &dc->pad[4], list_cap);
        mark("copy");
      }
      if (!write) A.level_counts[0] = nbk[2];
    }
    TCK(cudaGetLastError());
    mark("small");
    if (nbk[2]) {  // connectors that outgrew their slot: retry with 16x bigger slots, fewer threads
      // the overflow bitmask is compacted into a list on the device, in word chunks that fit the list area
      int64_t q = cq_lim;  // level 0: k_conn_small's shared-memory queues
      uint32_t* dlist = (uint32_t*)(ovf + ovf_words + 1);
      unsigned long long* dn = &dc->pad[1];
      const int64_t chunk_words = list_cap / 32 > 0 ? list_cap / 32 : 1;
      for (int level = 0; level < 8; level++) {
        const bool warp_level = level == 0;  // mid-size: one warp per saddle, shared memory only
        if (!warp_level && q >= words / 5) {  // larger than all scratch: count what is left as internal failures
          TCK(cudaMemsetAsync(dn, 0, 8, s));
          k_bits_compact<<<(unsigned)((ovf_words + 255) / 256 < 148 * 16 ? (ovf_words + 255) / 256 : 148 * 16), 256, 0,
                           s>>>((uint32_t*)ovf, 0, ovf_words, dlist, dn);  // (list unused beyond the count)
          TCK(cudaMemcpyAsync(&hc->pad[1], dn, 8, cudaMemcpyDeviceToHost, s));
          TCK(cudaStreamSynchronize(s));
          // those connectors have no cell count (their offsets were never written):
          // stop here -- the caller reports DMTZ_E_CAPACITY, the CSR is not produced
          A.n_overflow = (int64_t)hc->pad[1];
          TCK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
          TCK(cudaStreamSynchronize(s));
          A.n_internal = (int64_t)hc->n_internal;
          return cudaSuccess;
        }
        const int64_t qn = warp_level ? wq_lim : (q * grow < words / 5 ? q * grow : words / 5);
        int64_t h = 1;
        while (h < 2 * qn) h *= 2;
        const int64_t hw = A.unordered ? 1 : 2;   // hash words per slot: keys (+ owners for FIFO)
        while (qn + hw * h > words) h /= 2;
        int64_t ns = words / (qn + hw * h);
        if (ns < 1) ns = 1;
        if (ns > 148 * 32) ns = 148 * 32;  // one resident 64-thread block-BFS per slot
        bool any = false, cleared = false;
        for (int64_t w0 = 0; w0 < ovf_words; w0 += chunk_words) {
          const int64_t w1 = w0 + chunk_words < ovf_words ? w0 + chunk_words : ovf_words;
          TCK(cudaMemsetAsync(dn, 0, 8, s));
          const int64_t cb = (w1 - w0 + 255) / 256;
          k_bits_compact<<<(unsigned)(cb < 148 * 16 ? cb : 148 * 16), 256, 0, s>>>((uint32_t*)ovf, w0, w1, dlist, dn);
          TCK(cudaGetLastError());
          TCK(cudaMemcpyAsync(&hc->pad[1], dn, 8, cudaMemcpyDeviceToHost, s));
          TCK(cudaStreamSynchronize(s));
          const int64_t cn = (int64_t)hc->pad[1];
          if (!cn) continue;
          any = true;
          if (!write) A.level_counts[level + 1 < 10 ? level + 1 : 9] += cn;
          if (warp_level) {
            const int64_t nbw = (cn + CONNW_WARPS - 1) / CONNW_WARPS;
            if (A.verbose)
              fprintf(stderr, "dmtz trace pass %d level %d: %lld connectors, warp queues of %d\n", pass, level + 1,
                      (long long)cn, WQ);
            TCK(cudaFuncSetAttribute(k_conn_warp<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CONNW_SMEM));
            const unsigned wgrid = (unsigned)(nbw < 148 * 12 ? nbw : 148 * 12);
            // count pass with a pool: stage the events in the (still unused) BFS scratch
            const size_t stage_bytes = (size_t)wgrid * CONNW_WARPS * 3 * WQ * 8;
            uint64_t* stage = (!write && pool && stage_bytes <= (size_t)words * 8) ? (uint64_t*)sc : nullptr;
            TCK(cudaMemsetAsync(&dc->pad[7], 0, 8, s));
            k_conn_warp<D><<<wgrid, CONNW_WARPS * 32, CONNW_SMEM, s>>>(
                V.eview, g, dlist, cn, conn_base, A.out_origin, A.out_terminal, off, A.out_cells, write,
                (unsigned int*)ovf, wq_lim, stage, wpool, wpool_bottom, wpool_cap, wpool_flag, &dc->pad[7]);
            TCK(cudaGetLastError());
            continue;
          }
          // few connectors (<= 1024) with queues of <= SB_QMAX entries: the visited hash in
          // shared memory, one 256-thread block per SM -- the longest BFS is the critical path
          // (C3 tier 3, late S-rounds: 2.4 -> 1.4 ms); many: more 64-thread blocks in flight
          // with the global hash win (125 K connectors: 32 vs 99 ms).  DMTZ_BFS_SMEM=0: never,
          // 2: always
          const char* e_smem = getenv("DMTZ_BFS_SMEM");
          const int smem_mode = e_smem ? atoi(e_smem) : 1;
          TCK(cudaMemsetAsync(&dc->pad[7], 0, 8, s));   // the block kernels' next-saddle counter
          if (smem_mode && qn <= SB_QMAX && (cn <= 1024 || smem_mode == 2)) {
            const int64_t ns_s = words / qn < 148 * 4 ? words / qn : 148 * 4;
            const int64_t nb_s = cn < ns_s ? cn : ns_s;
            if (A.unordered) {
              TCK(cudaFuncSetAttribute(k_walk_block<D, 256, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SB_SMEM));
              k_walk_block<D, 256, true, true><<<(unsigned)nb_s, 256, SB_SMEM, s>>>(
                  V.eview, g, dlist, cn, conn_base, A.out_origin, A.out_terminal, off, A.out_cells, write, sc, qn,
                  SB_HCAP, (unsigned int*)ovf, dc, wpool, wpool_cap, wpool_bottom, &dc->pad[3], wpool_flag,
                  &dc->pad[7]);
            } else {
              TCK(cudaFuncSetAttribute(k_walk_block<D, 256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SB_SMEM));
              k_walk_block<D, 256, true><<<(unsigned)nb_s, 256, SB_SMEM, s>>>(
                  V.eview, g, dlist, cn, conn_base, A.out_origin, A.out_terminal, off, A.out_cells, write, sc, qn,
                  SB_HCAP, (unsigned int*)ovf, dc, wpool, wpool_cap, wpool_bottom, &dc->pad[3], wpool_flag,
                  &dc->pad[7]);
            }
            TCK(cudaGetLastError());
            continue;
          }
          if (!cleared) {  // block-BFS slots: zero once per level (the kernel leaves them zero)
            TCK(cudaMemsetAsync(sc, 0, (size_t)words * 8, s));
            cleared = true;
          }
          const int64_t nblk = cn < ns ? cn : ns;
          if (A.verbose)
            fprintf(stderr, "dmtz trace pass %d level %d: %lld connectors, q %lld, %lld blocks\n", pass, level + 1,
                    (long long)cn, (long long)qn, (long long)nblk);
          // block size of the BFS: DMTZ_BFS_THREADS=64|128|256|512|1024 (default 64: the
          // connectors of a level are many, so saddles in flight beat threads per saddle --
          // C5 origin planes [427, 597) 1475 -> 1105 ms, C3 342 -> 310 ms vs 256 threads)
          // levels with queues >= 2^17 (few, huge connectors: the longest BFS is the critical
          // path, wider batches shorten it) take DMTZ_BFS_THREADS_BIG, default 512 (C3 tier 3
          // 98 -> 79 s; 256: 79 s, 1024: 81 s)
          const char* bt = getenv("DMTZ_BFS_THREADS");
          const char* btb = getenv("DMTZ_BFS_THREADS_BIG");
          const int bfs_t = qn >= (1 << 17) ? (btb ? atoi(btb) : 512) : bt ? atoi(bt) : 64;
#define DMTZ_BFS_LAUNCH(T)                                                                                  \
  do {                                                                                                      \
    if (A.unordered)                                                                                        \
      k_walk_block<D, T, false, true><<<(unsigned)nblk, T, 0, s>>>(                                         \
          V.eview, g, dlist, cn, conn_base, A.out_origin, A.out_terminal, off, A.out_cells, write, sc, qn, h, \
          (unsigned int*)ovf, dc, wpool, wpool_cap, wpool_bottom, &dc->pad[3], wpool_flag, &dc->pad[7]);    \
    else                                                                                                    \
      k_walk_block<D, T><<<(unsigned)nblk, T, 0, s>>>(                                                      \
          V.eview, g, dlist, cn, conn_base, A.out_origin, A.out_terminal, off, A.out_cells, write, sc, qn, h, \
          (unsigned int*)ovf, dc, wpool, wpool_cap, wpool_bottom, &dc->pad[3], wpool_flag, &dc->pad[7]);    \
  } while (0)
          if (bfs_t == 1024) DMTZ_BFS_LAUNCH(1024);
          else if (bfs_t == 512) DMTZ_BFS_LAUNCH(512);
          else if (bfs_t == 128) DMTZ_BFS_LAUNCH(128);
          else if (bfs_t == 256) DMTZ_BFS_LAUNCH(256);
          else DMTZ_BFS_LAUNCH(64);
#undef DMTZ_BFS_LAUNCH
          TCK(cudaGetLastError());
        }
        mark(warp_level ? "warp" : "block");
        if (!any) break;
        q = qn;
      }
    }
    if (blocks_path && write)  // after the connectors: the paths overwrite the event pool
      TCK(launch_walk<D>(V, g, nbk[0], conn_base, A, off, write, dc, threads, s));
    TCK(cudaGetLastError());
    mark(write ? "W:paths" : "C:end");
    if (!write) {
      TCK(cudaMemsetAsync(off + nb, 0, 8, s));
      TCK(scan_i64(off, nb + 1, A.bsum, total, &hc->pad[0], s));
      mark("scan");
      A.n_cells = (int64_t)hc->pad[0];
      if (A.n_cells > A.cap_c) break;
      if (pool) {
        long long oc = 0;
        TCK(cudaMemcpyAsync(&oc, off + conn_base, 8, cudaMemcpyDeviceToHost, s));
        TCK(cudaStreamSynchronize(s));
        pool_limit = 2 * (int64_t)oc;
        top_ok = 2 * A.n_cells;
      }
    }
  }
  TCK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  TCK(cudaStreamSynchronize(s));
  A.n_internal = (int64_t)hc->n_internal;
  return cudaSuccess;
}

}  // namespace dmtz
