// dmtz_kernels.cuh -- sm_100a kernels of the DMTz hot path (C-loop + trace).
//
// Citations: P:<n> = PAPER.md line n.  The kernels implement, per anchor
// vertex, the local form of the gradient (DESIGN.md §3 "local form"):
//   cand(c) = argmin_SoS(c U link(c)) if that minimum is a link vertex, else NONE
// which equals the Shivashankar-Natarajan pairing of P:84-92 / P:152-155 (proved in
// DESIGN.md §3 and checked element-by-element against the literal CPU oracle).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dmtz_tables.h"

namespace dmtz {

// n / d for a divisor fixed at launch (round-up method: m = 2^32 (2^s - d) / d + 1,
// q = (umulhi(m, n) + n) >> s, exact for every 32-bit n); replaces the ~60-instruction
// 64-bit division in per-element index arithmetic
struct FastDiv {
  uint32_t d, m, s;
  FastDiv() = default;
  __host__ explicit FastDiv(uint32_t dv) : d(dv) {
    s = 0;
    while ((1ull << s) < dv) s++;
    m = (uint32_t)(((1ull << 32) * ((1ull << s) - dv)) / dv + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(m, n) + n) >> s);
  }
};

struct Grid {
  int64_t nx, ny, nz, N, sy, sz;  // sy = nx, sz = nx*ny
  // vertex index -> coordinates without 64-bit divisions when N < 2^32 (fast != 0)
  FastDiv dnx, dsz;
  int fast;
  __host__ void set_fast() {
    fast = N < (1ll << 32) && sz < (1ll << 32);
    if (fast) { dnx = FastDiv((uint32_t)nx); dsz = FastDiv((uint32_t)sz); }
  }
};

struct Counters {                 // device-side round counters (one 256 B block)
  unsigned long long n_false;
  unsigned long long kinds[8];
  unsigned long long n_changed;   // targets that took a step or were clamped
  unsigned long long n_targets;   // distinct targets marked
  unsigned long long n_internal;  // invariant violations (expected 0)
  unsigned long long n_swept;     // anchors evaluated by the round's sweep
  unsigned long long n_recomputed;  // of which their code was recomputed (stencil changed)
  unsigned long long n_decoded;   // anchors whose criticality was decoded this round
  unsigned long long n_items;     // false cells whose target rule was evaluated this round
  unsigned long long n_replayed;  // anchors whose cached targets were replayed this round
  unsigned long long first_nonfinite;
  unsigned long long first_bound;
  unsigned long long n_edits;
  unsigned long long n_lossless;  // lossless entries of the edit list
  unsigned long long n_units;     // active units of the current round (frontier list length)
  unsigned long long n_units2;    // slab mode: units whose cells are classified
  unsigned long long pad[9];
};
static_assert(sizeof(Counters) == 256, "counters are one 256 B block");

// Device-side state of the round loop (a7), updated by k_loop_check after every
// round; lets the loop run inside a CUDA-graph conditional WHILE node.
struct LoopState {
  unsigned long long round;          // the round about to run / running (1-based)
  unsigned long long rounds;         // rounds that found false cells
  unsigned long long sweeps;
  unsigned long long anchors_swept;
  unsigned long long n_false0;       // false cells before any edit
  unsigned long long kinds0[8];
  unsigned long long status;         // dmtz_status of the loop (0 while running / OK)
  unsigned long long last_false, last_changed, last_targets, last_swept;
  unsigned long long recomputed;     // anchors whose code was recomputed, summed over sweeps
  unsigned long long decoded, items, replayed;  // k_decode work, summed over sweeps
  unsigned long long pad[10];
};
static_assert(sizeof(LoopState) == 256, "loop state is one 256 B block");

// Range of the values a call's fields can take (f, and g in [lb, fhat]): the key
// form of the gradient (dmtz_sweep.cuh load_keys) needs every value positive and the
// float bit patterns within 2^25 of the smallest.  Filled by k_setup.
struct KeyInfo {
  int min_bits;           // min over lb (as signed int: <= 0 for a non-positive value)
  unsigned int max_bits;  // max over f and fhat (as unsigned: a negative value is huge)
  unsigned int pad[14];
};
// 32 (max - min) + 26 stays below the outside-grid key 0x7E000000 (dmtz_sweep.cuh load_keys)
constexpr unsigned KEY_RANGE = 1u << 25;
__device__ __forceinline__ bool keys_ok(const KeyInfo* ki, uint32_t* base) {
  const int mn = ki->min_bits;
  const unsigned mx = ki->max_bits;
  *base = (uint32_t)mn;
  return mn > 0 && mx >= (unsigned)mn && mx - (unsigned)mn < KEY_RANGE;
}

__global__ void k_set_round(LoopState* ls, unsigned long long r) {
  if (threadIdx.x == 0) ls->round = r;
}

__global__ void k_loop_reset(LoopState* ls) {
  if (threadIdx.x == 0) {
    LoopState z = {};
    z.round = 1;
    *ls = z;
  }
}

// The stop rule of the C-loop: F empty -> OK; no target
// could move -> STUCK; round cap -> ITER_CAP.  Sets the WHILE condition when use_cond.
__global__ void k_loop_check(struct Counters* cnt, LoopState* ls, unsigned long long max_rounds,
                             cudaGraphConditionalHandle h, int use_cond, unsigned long long* n_units_clear);

template <int D> struct Tr;
template <> struct Tr<3> {
  using code_t = unsigned long long;
  static constexpr int NT = k3d::NT, TOP = 3, NDELTA = 8;
  static constexpr uint64_t ALL_NONE = k3d::ALL_NONE;
};
template <> struct Tr<2> {
  using code_t = unsigned short;
  static constexpr int NT = k2d::NT, TOP = 2, NDELTA = 4;
  static constexpr uint64_t ALL_NONE = k2d::ALL_NONE;
};

__global__ void k_loop_check(Counters* cnt, LoopState* ls, unsigned long long max_rounds,
                             cudaGraphConditionalHandle h, int use_cond, unsigned long long* n_units_clear) {
  if (threadIdx.x != 0) return;
  const unsigned long long r = ls->round;
  ls->sweeps++;
  ls->anchors_swept += cnt->n_swept;
  ls->recomputed += cnt->n_recomputed;
  ls->decoded += cnt->n_decoded;
  ls->items += cnt->n_items;
  ls->replayed += cnt->n_replayed;
  ls->last_false = cnt->n_false;
  ls->last_changed = cnt->n_changed;
  ls->last_targets = cnt->n_targets;
  ls->last_swept = cnt->n_swept;
  bool go = false;
  if (cnt->n_internal) {
    ls->status = 11;  // DMTZ_E_INTERNAL
  } else {
    if (r == 1) {
      ls->n_false0 = cnt->n_false;
      for (int k = 0; k < 8; k++) ls->kinds0[k] = cnt->kinds[k];
    }
    if (cnt->n_false != 0) {
      ls->rounds = r;
      if (cnt->n_changed == 0) ls->status = 7;        // DMTZ_E_STUCK
      else if (r == max_rounds) ls->status = 6;        // DMTZ_E_ITER_CAP
      else { ls->round = r + 1; go = true; }
    }
  }
  if (use_cond) {
    // device-driven loop: clear this round's counters (and the frontier list length)
    // for the next round here instead of with memset nodes
    unsigned long long* p = (unsigned long long*)cnt;
    for (int i = 0; i < (int)(offsetof(Counters, first_nonfinite) / 8); i++) p[i] = 0ull;
    if (n_units_clear) *n_units_clear = 0ull;
    cudaGraphSetConditional(h, go ? 1u : 0u);
  }
}


// the round counters of a slab round into a caller buffer (device): n_false, n_changed,
// n_targets, n_internal, kinds[8] (round 1 only, else 0)
__global__ void k_counters_out(const Counters* __restrict__ cnt, long long round, long long* __restrict__ out) {
  const int i = threadIdx.x;
  if (i == 0) out[0] = (long long)cnt->n_false;
  if (i == 1) out[1] = (long long)cnt->n_changed;
  if (i == 2) out[2] = (long long)cnt->n_targets;
  if (i == 3) out[3] = (long long)cnt->n_internal;
  if (i >= 4 && i < 12) out[i] = round == 1 ? (long long)cnt->kinds[i - 4] : 0ll;
}

// table accessors (constant-folded when t is a compile-time constant after unrolling)
#define DMTZ_TAB(D, name) ((D) == 3 ? k3d::name : k2d::name)
template <int D> __device__ __forceinline__ int t_dim(int t) { return D == 3 ? k3d::DIM[t] : k2d::DIM[t]; }
// types of kind class c (0 = minima, 1 = 1-saddles, 2 = 2-saddles, 3 = maxima = top dimension)
template <int D> __device__ __forceinline__ uint32_t t_dimclass_mask(int c) {
  uint32_t m = 0;
#pragma unroll
  for (int t = 0; t < Tr<D>::NT; t++) {
    const int d = t_dim<D>(t);
    m |= ((d == Tr<D>::TOP ? 3 : d) == c ? 1u : 0u) << t;
  }
  return m;
}
template <int D> __device__ __forceinline__ int t_nv(int t) { return D == 3 ? k3d::NV[t] : k2d::NV[t]; }
template <int D> __device__ __forceinline__ int t_shift(int t) { return D == 3 ? k3d::SHIFT[t] : k2d::SHIFT[t]; }
template <int D> __device__ __forceinline__ int t_none(int t) { return D == 3 ? k3d::NONE[t] : k2d::NONE[t]; }
template <int D> __device__ __forceinline__ int t_nfacet(int t) { return D == 3 ? k3d::NFACET[t] : k2d::NFACET[t]; }
template <int D> __device__ __forceinline__ int t_facet(int t, int j, int c) {
  return D == 3 ? k3d::FACET[t][j][c] : k2d::FACET[t][j][c];
}
template <int D> __device__ __forceinline__ int t_vmask(int t, int k) { return D == 3 ? k3d::VMASK[t][k] : k2d::VMASK[t][k]; }
template <int D> __device__ __forceinline__ int t_link(int t, int s, int a) { return D == 3 ? k3d::LINK[t][s][a] : k2d::LINK[t][s][a]; }
template <int D> __device__ __forceinline__ int t_nlink(int t) { return D == 3 ? k3d::NLINK[t] : k2d::NLINK[t]; }
template <int D> __device__ __forceinline__ int t_cof_type(int t, int s) { return D == 3 ? k3d::COF_TYPE[t][s] : k2d::COF_TYPE[t][s]; }
template <int D> __device__ __forceinline__ int t_cof_anchor(int t, int s, int a) {
  return D == 3 ? k3d::COF_ANCHOR[t][s][a] : k2d::COF_ANCHOR[t][s][a];
}
template <int D> __device__ __forceinline__ uint32_t t_exist(int ok) { return D == 3 ? k3d::EXIST[ok] : k2d::EXIST[ok]; }
template <int D> __device__ __forceinline__ uint64_t t_nonex_fill(int ok) {
  return D == 3 ? k3d::NONEX_FILL[ok] : k2d::NONEX_FILL[ok];
}
template <int D> __host__ __device__ constexpr int t_first_of_dim_c(int d) {
  return D == 3 ? (d == 0 ? 0 : d == 1 ? 1 : d == 2 ? 8 : d == 3 ? 20 : 26) : (d == 0 ? 0 : d == 1 ? 1 : d == 2 ? 4 : 6);
}
template <int D> __device__ __forceinline__ int t_first_of_dim(int d) {
  return D == 3 ? k3d::FIRST_OF_DIM[d] : k2d::FIRST_OF_DIM[d];
}

template <int D> __device__ __forceinline__ uint32_t field_of(uint64_t code, int t) {
  return (uint32_t)(code >> t_shift<D>(t)) & (uint32_t)t_none<D>(t);
}

__device__ __forceinline__ int64_t mask_delta(const Grid& g, int m) {
  return (int64_t)(m & 1) + ((m >> 1) & 1) * g.sy + ((m >> 2) & 1) * g.sz;
}

// 'axes with a +1 neighbour' bit mask of an anchor
__device__ __forceinline__ int axes_ok(const Grid& g, int64_t x, int64_t y, int64_t z) {
  return (x + 1 < g.nx ? 1 : 0) | (y + 1 < g.ny ? 2 : 0) | (z + 1 < g.nz ? 4 : 0);
}

// SoS order (reading A2): (value, index) lexicographic
__device__ __forceinline__ bool sos_less(float a, int64_t ia, float b, int64_t ib) {
  return a < b || (a == b && ia < ib);
}

// --------------------------------------------------------------------------
// Gradient codes of a field (a2/a3): one thread per anchor, 3^D stencil.
// --------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ uint64_t anchor_code(const float* __restrict__ fld, const Grid& g, int64_t v,
                                                int64_t x, int64_t y, int64_t z) {
  const float INF = __int_as_float(0x7f800000);
  float s[27];
#pragma unroll
  for (int dz = -1; dz <= 1; dz++)
#pragma unroll
    for (int dy = -1; dy <= 1; dy++)
#pragma unroll
      for (int dx = -1; dx <= 1; dx++) {
        const int p = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
        if (D == 2 && dz != 0) { s[p] = INF; continue; }
        bool in = (x + dx >= 0) && (x + dx < g.nx) && (y + dy >= 0) && (y + dy < g.ny) &&
                  (z + dz >= 0) && (z + dz < g.nz);
        s[p] = in ? __ldg(fld + v + dx + dy * g.sy + dz * g.sz) : INF;
      }
  uint64_t code = (D == 3) ? k3d::cand_code(s) : k2d::cand_code(s);
  return code | t_nonex_fill<D>(axes_ok(g, x, y, z));
}

// iterate anchors of z-planes [z0, z1) with a 3D launch: x fastest, grid-stride in y/z
#define DMTZ_FOR_ANCHORS(g, z0, z1)                                                        \
  for (int64_t z = (z0) + blockIdx.z; z < (z1); z += gridDim.z)                            \
    for (int64_t y = blockIdx.y; y < (g).ny; y += gridDim.y)                               \
      for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < (g).nx;         \
           x += (int64_t)gridDim.x * blockDim.x)

template <int D>
__global__ void k_codes(const float* __restrict__ fld, typename Tr<D>::code_t* __restrict__ codes,
                        Grid g, int64_t z0, int64_t z1) {
  DMTZ_FOR_ANCHORS(g, z0, z1) {
    int64_t v = x + y * g.sy + z * g.sz;
    codes[v] = (typename Tr<D>::code_t)anchor_code<D>(fld, g, v, x, y, z);
  }
}

// --------------------------------------------------------------------------
// Critical masks from the codes at u + {0,1}^D (a4).
// crit(c) <=> c exists, cand(c) = NONE, and no facet points to c.
// --------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ uint32_t decode_crit(const uint64_t (&c)[Tr<D>::NDELTA], int ok) {
  uint32_t m = 0;
#pragma unroll
  for (int t = 0; t < Tr<D>::NT; t++) {
    bool crit = true;
    if (t_dim<D>(t) < Tr<D>::TOP) crit = field_of<D>(c[0], t) == (uint32_t)t_none<D>(t);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (j < t_nfacet<D>(t)) {
        const int dm = t_facet<D>(t, j, 0), ft = t_facet<D>(t, j, 1), sl = t_facet<D>(t, j, 2);
        crit = crit && (field_of<D>(c[dm], ft) != (uint32_t)sl);
      }
    }
    m |= (crit ? 1u : 0u) << t;
  }
  return m & t_exist<D>(ok);
}

// crit mask, and in *dp for every type the index j (2 bits at 2t) of the facet whose
// code points at the cell -- its down-pair partner when it has one (a gradient pairs
// a cell with at most one facet)
template <int D>
__device__ __forceinline__ uint32_t decode_crit_dp(const uint64_t (&c)[Tr<D>::NDELTA], int ok, uint64_t* dp) {
  uint32_t m = 0;
  uint32_t dlo = 0, dhi = 0;
#pragma unroll
  for (int t = 0; t < Tr<D>::NT; t++) {
    bool crit = true;
    if (t_dim<D>(t) < Tr<D>::TOP) crit = field_of<D>(c[0], t) == (uint32_t)t_none<D>(t);
    uint32_t jsel = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (j < t_nfacet<D>(t)) {
        const int dm = t_facet<D>(t, j, 0), ft = t_facet<D>(t, j, 1), sl = t_facet<D>(t, j, 2);
        const bool hit = field_of<D>(c[dm], ft) == (uint32_t)sl;
        crit = crit && !hit;
        if (j > 0) jsel = hit ? (uint32_t)j : jsel;
      }
    }
    m |= (crit ? 1u : 0u) << t;
    if (t < 16) dlo |= jsel << (2 * t);
    else dhi |= jsel << (2 * (t - 16));
  }
  *dp = ((uint64_t)dhi << 32) | dlo;
  return m & t_exist<D>(ok);
}

template <int D>
__device__ __forceinline__ void load_codes8(const typename Tr<D>::code_t* __restrict__ codes, const Grid& g,
                                            int64_t v, int ok, uint64_t (&c)[Tr<D>::NDELTA]) {
#pragma unroll
  for (int dm = 0; dm < Tr<D>::NDELTA; dm++)
    c[dm] = ((dm & ~ok) == 0) ? (uint64_t)__ldg(codes + v + mask_delta(g, dm)) : Tr<D>::ALL_NONE;
}

template <int D>
__global__ void k_critmask(const typename Tr<D>::code_t* __restrict__ codes, uint32_t* __restrict__ crit,
                           Grid g) {
  DMTZ_FOR_ANCHORS(g, 0, g.nz) {
    int64_t v = x + y * g.sy + z * g.sz;
    int ok = axes_ok(g, x, y, z);
    uint64_t c[Tr<D>::NDELTA];
    load_codes8<D>(codes, g, v, ok, c);
    crit[v] = decode_crit<D>(c, ok);
  }
}

__device__ __forceinline__ void warp_add(unsigned long long* dst, unsigned long long v) {
  // warp-aggregated atomic for a value that may be zero on most lanes
  unsigned mask = __ballot_sync(0xffffffffu, v != 0);
  if (!mask) return;
  unsigned long long s = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1)) atomicAdd(dst, s);
}

// --------------------------------------------------------------------------
// Setup (a1): validate, lb = RU32(f - xi), g = fhat, state = 0.
// |fhat - f| <= xi exactly  <=>  RU(f - xi) <= fhat <= RD(f + xi).
// --------------------------------------------------------------------------
__global__ void k_setup(const float* __restrict__ f, const float* __restrict__ fhat, float xi, int64_t n,
                        float* __restrict__ lb, float* __restrict__ gf, uint32_t* __restrict__ state,
                        Counters* __restrict__ cnt, KeyInfo* __restrict__ ki) {
  int mn = 0x7FFFFFFF;
  unsigned mx = 0u;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const float a = f[v], b = fhat[v];
    if (!isfinite(a) || !isfinite(b)) { atomicMin(&cnt->first_nonfinite, (unsigned long long)v); continue; }
    const float lo = __fsub_ru(a, xi);
    if (b < lo || b > __fadd_rd(a, xi)) atomicMin(&cnt->first_bound, (unsigned long long)v);
    lb[v] = lo;
    gf[v] = b;
    state[v] = 0;
    mn = min(mn, __float_as_int(lo));
    mx = max(mx, max(__float_as_uint(a), __float_as_uint(b)));
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&ki->min_bits, mn);
    atomicMax(&ki->max_bits, mx);
  }
}

// --------------------------------------------------------------------------
// Edit-list emission (a8): ordered stream compaction of {v : state_v != 0}.
// Chunk = EDIT_CHUNK vertices per block; count -> exclusive scan -> write.
// --------------------------------------------------------------------------
constexpr int EDIT_CHUNK = 8192;
constexpr int EDIT_THREADS = 1024;

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  unsigned long long s = 0;
  if (w == 0) {
    s = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  __syncthreads();
  return s;  // valid in warp 0
}

// vertices [v0, n) (slab mode: the owned planes)
__global__ void k_edit_count(const uint32_t* __restrict__ state, int64_t v0, int64_t n,
                             unsigned long long* __restrict__ bc, Counters* __restrict__ cnt) {
  __shared__ unsigned long long sh[32];
  const int64_t base = v0 + (int64_t)blockIdx.x * EDIT_CHUNK;
  unsigned long long c = 0, nl = 0;
  for (int i = threadIdx.x; i < EDIT_CHUNK; i += blockDim.x) {
    const int64_t v = base + i;
    const uint32_t st = v < n ? state[v] : 0u;
    if (st != 0) c++;
    if (st >> 16) nl++;
  }
  warp_add(&cnt->n_lossless, nl);
  c = block_sum(c, sh);
  if (threadIdx.x == 0) bc[blockIdx.x] = c;
}

// exclusive scan of nb block counts in one block; total -> cnt->n_edits
__global__ void k_scan_counts(unsigned long long* __restrict__ bc, int64_t nb, Counters* __restrict__ cnt) {
  __shared__ unsigned long long part[EDIT_THREADS];
  const int64_t per = (nb + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = min(nb, lo + per);
  unsigned long long s = 0;
  for (int64_t i = lo; i < hi; i++) s += bc[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (int i = 0; i < (int)blockDim.x; i++) { unsigned long long t = part[i]; part[i] = acc; acc += t; }
    cnt->n_edits = acc;
  }
  __syncthreads();
  unsigned long long acc = part[threadIdx.x];
  for (int64_t i = lo; i < hi; i++) { unsigned long long t = bc[i]; bc[i] = acc; acc += t; }
}

struct EditOut { unsigned long long v; unsigned short q; unsigned char lossless; unsigned char pad; float value; };
static_assert(sizeof(EditOut) == 16, "dmtz_edit is 16 bytes");

__global__ void k_edit_write(const uint32_t* __restrict__ state, const float* __restrict__ gf, int64_t v0, int64_t n,
                             const unsigned long long* __restrict__ boff, EditOut* __restrict__ out, int64_t cap,
                             int64_t v_global_off) {
  __shared__ unsigned int wsum[32];
  const int64_t base = v0 + (int64_t)blockIdx.x * EDIT_CHUNK;
  unsigned long long off = boff[blockIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int seg = 0; seg < EDIT_CHUNK; seg += blockDim.x) {
    const int64_t v = base + seg + threadIdx.x;
    const uint32_t st = (v < n) ? state[v] : 0u;
    const bool e = st != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, e);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    unsigned int before = 0, total = 0;
    for (int k = 0; k < nw; k++) { unsigned int c = wsum[k]; if (k < w) before += c; total += c; }
    if (e) {
      const unsigned long long pos = off + before + __popc(bal & ((1u << lane) - 1u));
      if ((int64_t)pos < cap) {
        EditOut o;
        o.v = (unsigned long long)(v + v_global_off);
        o.q = (unsigned short)(st & 0xFFFFu);
        o.lossless = (unsigned char)(st >> 16);
        o.pad = 0;
        o.value = gf[v];
        out[pos] = o;
      }
    }
    off += total;
    __syncthreads();
  }
}

}  // namespace dmtz
