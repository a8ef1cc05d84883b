// dmtz_sweep.cuh -- the round sweep of the C-loop (a3 + a4 + a5) for sm_100a.
//
// Work unit: a ROW BLOCK = UY consecutive y-rows of one z-plane (all x).  Each
// round processes an on-device list of active units (the frontier, a7): every
// unit in round 1 and in full-sweep mode, afterwards only units meeting
// v + [-2,1]^D for some target v of the previous round.
//
//  k_screen<D>  for every anchor u of an active unit: cand_g(u) from the 3^D
//               stencil of g (the local form of the gradient).
//               The dense code buffer cg keeps the previous round's codes; the
//               bit e(u) = [code changed this round] goes to a row-padded bitmap
//               (one word per 32 anchors of a row).
//  k_decode<D>  for every anchor u of an active unit with a changed code in
//               u + {0,1}^D (criticality is a function of those 8 codes) or
//               with false cells last round: crit_g(u) and the down-pair facets,
//               F(u) = crit_f(u) xor crit_g(u), and the targets of F(u) (rules
//               R1/R2/R3a/R3b) over a per-warp shared-memory work list, OR-ed
//               into a shared-memory window of the chunk, then into the round's
//               (row-padded) target bitmap with one atomic per non-empty word.
//  k_edit_rows<D> Eq. 2 edits of the marked targets and the next frontier.
#pragma once
#include <utility>

#include "dmtz_kernels.cuh"

namespace dmtz {

constexpr int UY = 4;  // rows per unit

struct RowGeom {
  int64_t wpr;     // bitmap words per row = ceil(nx / 32)
  int64_t ub;      // y-blocks per plane = ceil(ny / UY)
  int64_t units;   // ub * nz
};

__host__ __device__ inline RowGeom row_geom(const Grid& g) {
  RowGeom r;
  r.wpr = (g.nx + 31) / 32;
  r.ub = (g.ny + UY - 1) / UY;
  r.units = r.ub * g.nz;
  return r;
}

// Work decomposition of the active units: item = (unit, row, group of CG row
// chunks of 32 anchors); warps stride over items, 32-bit index arithmetic.
constexpr int CG = 4;
constexpr int DG = 16;  // k_screen / k_decode: chunks per work item (512 anchors of a row)
#define WORK_LOOP_BEGIN                                                                          \
  {                                                                                              \
    const uint32_t n_units_ = (uint32_t)*n_units_p;                                              \
    const uint32_t ncg_ = (uint32_t)((rg.wpr + CG - 1) / CG);                                    \
    const uint32_t per_unit_ = (uint32_t)UY * ncg_;                                              \
    const uint32_t total_ = n_units_ * per_unit_;                                                \
    for (uint32_t it_ = (uint32_t)warp; it_ < total_; it_ += (uint32_t)nwarps) {                 \
      const uint32_t ui_ = it_ / per_unit_, rem_ = it_ - ui_ * per_unit_;                        \
      const uint32_t unit_ = units[ui_];                                                         \
      const uint32_t ub_ = (uint32_t)rg.ub;                                                      \
      const int64_t z = unit_ / ub_;                                                             \
      const int64_t y = (int64_t)(unit_ - (uint32_t)z * ub_) * UY + rem_ / ncg_;                 \
      const int64_t c0_ = (int64_t)(rem_ % ncg_) * CG;                                           \
      if (y >= g.ny) continue;                                                                   \
      for (int64_t c = c0_; c < c0_ + CG && c < rg.wpr; c++) {
#define WORK_LOOP_END \
      }               \
    }                 \
  }

// bit word of anchor row (y, z), x-chunk c
__device__ __forceinline__ int64_t dword_index(const Grid& g, const RowGeom& rg, int64_t y, int64_t z, int64_t c) {
  return (z * g.ny + y) * rg.wpr + c;
}

// ---------------------------------------------------------------------------
// Stencil load: the 3^D neighbourhood of u, +inf outside the grid.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void load_stencil(const float* __restrict__ fld, const Grid& g, int64_t v, int64_t x,
                                             int64_t y, int64_t z, float (&s)[27]) {
  const float INF = __int_as_float(0x7f800000);
  const bool interior = x > 0 && x + 1 < g.nx && y > 0 && y + 1 < g.ny && (D == 2 || (z > 0 && z + 1 < g.nz));
  if (interior) {
#pragma unroll
    for (int dz = -1; dz <= 1; dz++)
#pragma unroll
      for (int dy = -1; dy <= 1; dy++)
#pragma unroll
        for (int dx = -1; dx <= 1; dx++) {
          const int p = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
          if (D == 2 && dz != 0) { s[p] = INF; continue; }
          s[p] = __ldg(fld + v + dx + dy * g.sy + dz * g.sz);
        }
  } else {
#pragma unroll
    for (int dz = -1; dz <= 1; dz++)
#pragma unroll
      for (int dy = -1; dy <= 1; dy++)
#pragma unroll
        for (int dx = -1; dx <= 1; dx++) {
          const int p = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
          if (D == 2 && dz != 0) { s[p] = INF; continue; }
          const bool in = (x + dx >= 0) && (x + dx < g.nx) && (y + dy >= 0) && (y + dy < g.ny) &&
                          (z + dz >= 0) && (z + dz < g.nz);
          s[p] = in ? __ldg(fld + v + dx + dy * g.sy + dz * g.sz) : INF;
        }
  }
}

// Key form of the stencil (DESIGN.md §7 "key form"): W[p] = 32 (bits(g_p) - base) + p,
// p = (dx+1) + 3 (dy+1) + 9 (dz+1) the stencil position (ascending global index).  When
// every value of the call is positive and within 2^25 bit patterns of base (keys_ok),
// W[p] < 2^30 + 32, and W[p] < W[q] <=> g_p < g_q or (g_p = g_q and p < q): the SoS
// order on the stencil.  Read as float bit patterns the keys keep that order
// (non-negative, finite), so the argmin of a type's set is one FMNMX3 tree and
// key & 31 its position.  Outside the grid: a key above every valid one.
constexpr uint32_t KEY_OUTSIDE = 0x7E000000u;
constexpr int TSEG = 64, TROW = TSEG + 8;  // k_screen's tiled dense path: anchors per segment, floats per row
constexpr int SCREEN_TILE_BYTES = (256 / 32) * 2 * 9 * TROW * 4;  // per CTA (SCREEN_THREADS = 256)
template <int D>
__device__ __forceinline__ void load_keys(const float* __restrict__ fld, const Grid& g, int64_t v, int64_t x,
                                          int64_t y, int64_t z, uint32_t base, uint32_t (&W)[27]) {
  const bool interior = x > 0 && x + 1 < g.nx && y > 0 && y + 1 < g.ny && (D == 2 || (z > 0 && z + 1 < g.nz));
  const uint32_t c0 = 0u - 32u * base;
  if (interior) {  // straight-line: 27 loads, 27 multiply-adds (FMA pipe)
#pragma unroll
    for (int dz = -1; dz <= 1; dz++)
#pragma unroll
      for (int dy = -1; dy <= 1; dy++)
#pragma unroll
        for (int dx = -1; dx <= 1; dx++) {
          const int p = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
          if (D == 2 && dz != 0) { W[p] = KEY_OUTSIDE; continue; }
          const uint32_t b = __float_as_uint(__ldg(fld + v + dx + dy * g.sy + dz * g.sz));
          asm("mad.lo.u32 %0, %1, 32, %2;" : "=r"(W[p]) : "r"(b), "r"(c0 + (uint32_t)p));
        }
  } else {
#pragma unroll
    for (int dz = -1; dz <= 1; dz++)
#pragma unroll
      for (int dy = -1; dy <= 1; dy++)
#pragma unroll
        for (int dx = -1; dx <= 1; dx++) {
          const int p = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
          if (D == 2 && dz != 0) { W[p] = KEY_OUTSIDE; continue; }
          const bool in = (x + dx >= 0) && (x + dx < g.nx) && (y + dy >= 0) && (y + dy < g.ny) && (z + dz >= 0) &&
                          (z + dz < g.nz);
          W[p] = in ? 32u * (__float_as_uint(__ldg(fld + v + dx + dy * g.sy + dz * g.sz)) - base) + (uint32_t)p
                    : KEY_OUTSIDE;
        }
  }
}

template <int D>
__device__ __forceinline__ uint64_t cand_of_keys(const uint32_t (&W)[27], const uint8_t* lut) {
  if constexpr (D == 3) return k3d::cand_code_keys(W, lut);
  else return k2d::cand_code_keys(W, lut);
}

template <int D>
__device__ __forceinline__ uint64_t cand_of(const float (&s)[27]) {
  if constexpr (D == 3) return k3d::cand_code(s);
  else return k2d::cand_code(s);
}

// ---------------------------------------------------------------------------
// k_screen: codes of g; e(u) = code changed.  Work item = (unit, row, group of DG
// 32-anchor chunks).  need(u): a vertex of u's 3^D box changed in the previous
// round -> the code may change; else it provably did not (a code is a function
// of that box) and the memoized one stays.  The anchors that need a recompute
// are compacted into full warps (lane = one anchor).
// ---------------------------------------------------------------------------
constexpr int SCREEN_THREADS = 256;
#ifndef DMTZ_SCREEN_DENSE8
#define DMTZ_SCREEN_DENSE8 5u   // frontier mode: an item is swept whole when >= 5/8 of it needs a new code
#endif
#ifndef DMTZ_SCREEN_MINB
#define DMTZ_SCREEN_MINB 4   // 4 CTAs (32 warps) per SM: <= 64 registers, the tile's shared memory fits
#endif
#define DMTZ_SCREEN_LB __launch_bounds__(SCREEN_THREADS, DMTZ_SCREEN_MINB)
// SKIP = false: the full-sweep instantiation (use_skip = 0), without the change-skip code
template <int D, bool SKIP>
__global__ void DMTZ_SCREEN_LB
k_screen(const float* __restrict__ gfld, typename Tr<D>::code_t* __restrict__ cg, uint32_t* __restrict__ ebits,
         uint32_t* __restrict__ vchg, int64_t vwords, int use_skip, const uint32_t* __restrict__ units,
         const unsigned long long* __restrict__ n_units_p, Grid g, RowGeom rg, const LoopState* __restrict__ ls,
         Counters* __restrict__ cnt, const KeyInfo* __restrict__ ki, int use_keys, uint32_t kmul) {
  // kmul = 32, a launch parameter: a multiplier the compiler cannot see stays an IMAD (FMA
  // pipe) instead of becoming a shift-add (ALU pipe, the limiting one here)
  __shared__ uint16_t s_list[SCREEN_THREADS / 32][DG * 32];
  __shared__ uint32_t s_e[SCREEN_THREADS / 32][DG];
  constexpr int NF = D == 3 ? k3d::NFIELD : k2d::NFIELD;
  __shared__ uint8_t s_lut[NF * 32];
  for (int i = threadIdx.x; i < NF * 32; i += blockDim.x)
    s_lut[i] = D == 3 ? (&k3d::KEYLUT[0][0])[i] : (&k2d::KEYLUT[0][0])[i];
  __syncthreads();
  uint32_t kbase = 0;
  const bool keys = use_keys && keys_ok(ki, &kbase);  // uniform over the launch
  // tiled dense path: 16-byte aligned rows (nx % 4 == 0); DMTZ_SCREEN_TILE=0 (use_keys & 2) disables it
  extern __shared__ __align__(16) float s_tile_dyn[];  // SCREEN_TILE_BYTES when launched tiled, else 0
  const bool tiled = keys && (use_keys & 2) && (g.nx % 4) == 0;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint16_t* list = s_list[wib];
  uint32_t* se = s_e[wib];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned long long round = ls->round;
  const bool first_round = round == 1;
  // vertices whose value changed in the previous round (its edits) / this round's (cleared here)
  const uint32_t* vprev = vchg + (int64_t)((round - 1) & 1) * vwords;
  uint32_t* vcur = vchg + (int64_t)(round & 1) * vwords;
  const bool skip = SKIP && use_skip && !first_round;
  unsigned long long swept = 0, recomputed = 0;
  const uint32_t n_units_ = (uint32_t)*n_units_p;
  const uint32_t ngr = (uint32_t)((rg.wpr + DG - 1) / DG);
  const uint32_t per_unit_ = (uint32_t)UY * ngr;
  const uint32_t total_ = n_units_ * per_unit_;
  for (uint32_t it_ = (uint32_t)warp; it_ < total_; it_ += (uint32_t)nwarps) {
    const uint32_t ui_ = it_ / per_unit_, rem_ = it_ - ui_ * per_unit_;
    const uint32_t unit_ = units[ui_];
    const uint32_t ub_ = (uint32_t)rg.ub;
    const int64_t z = unit_ / ub_;
    const int64_t y = (int64_t)(unit_ - (uint32_t)z * ub_) * UY + rem_ / ngr;
    if (y >= g.ny) continue;  // warp-uniform
    const int64_t cbase = (int64_t)(rem_ % ngr) * DG;
    const int64_t cl = cbase + lane;
    const bool inrow = lane < DG && cl < rg.wpr;
    uint32_t valid = 0, need = 0;
    if (inrow) {
      const int64_t rem = g.nx - cl * 32;
      valid = rem < 32 ? (1u << rem) - 1u : 0xffffffffu;
      need = valid;
      if (skip) {  // OR of the previous round's change words over the 3^D rows, then dilate in x
        uint32_t A = 0, B = 0, C = 0;
#pragma unroll
        for (int dz = (D == 3 ? -1 : 0); dz <= (D == 3 ? 1 : 0); dz++)
#pragma unroll
          for (int dy = -1; dy <= 1; dy++) {
            const int64_t yy = y + dy, zz = z + dz;
            if (yy < 0 || yy >= g.ny || zz < 0 || zz >= g.nz) continue;
            const int64_t wi = dword_index(g, rg, yy, zz, cl);
            B |= __ldg(vprev + wi);
            if (cl > 0) A |= __ldg(vprev + wi - 1);
            if (cl + 1 < rg.wpr) C |= __ldg(vprev + wi + 1);
          }
        need &= (A >> 31) | B | (B << 1) | (B >> 1) | (C << 31);
      }
      vcur[dword_index(g, rg, y, z, cl)] = 0u;
      swept += __popc(valid);
      se[lane] = 0u;
    }
    // dense: every anchor of the item is recomputed -- also when the change skip leaves
    // only most of them (>= 5/8): an anchor whose 3^D values did not change gets its
    // memo code back (no change bit), and the tiled full pass is cheaper than the list
    bool dense = __all_sync(0xffffffffu, need == valid);
    if (skip && !dense)   // warp-uniform
      dense = 8u * __reduce_add_sync(0xffffffffu, (unsigned)__popc(need)) >=
              DMTZ_SCREEN_DENSE8 * __reduce_add_sync(0xffffffffu, (unsigned)__popc(valid));
    int n;
    if (dense) {
      n = (int)(__shfl_sync(0xffffffffu, (int)(g.nx - cbase * 32 < DG * 32 ? g.nx - cbase * 32 : DG * 32), 0));
    } else {
      const int c = __popc(need);
      int pre = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += v;
      }
      n = __shfl_sync(0xffffffffu, pre, 31);
      pre -= c;
      uint32_t m = need;
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        list[pre++] = (uint16_t)(lane * 32 + b);
      }
    }
    __syncwarp();
    const int64_t row0 = y * g.sy + z * g.sz + cbase * 32;
    // the code's memo compare and the changed-code bits of a batch (lanes in ascending anchor order)
    auto finish = [&](bool act, int o, uint64_t code, uint64_t old) {
      bool e = false;
      if (act) {
        const int64_t v = row0 + o;
        e = first_round || code != old;
        if (e) cg[v] = (typename Tr<D>::code_t)code;
        recomputed++;
      }
      const unsigned grp = __match_any_sync(0xffffffffu, act ? (o >> 5) : -1);
      const uint32_t bits = __reduce_or_sync(grp, e ? 1u << (o & 31) : 0u);
      if (act && lane == __ffs(grp) - 1 && bits) se[o >> 5] |= bits;
      __syncwarp();
    };
    if (dense && tiled) {
      // dense item, tiled: the stencil rows of 64-anchor segments are staged in shared
      // memory with cp.async (double-buffered: segment k + 1 streams in while k is
      // computed); an anchor forms its 27 keys from shared memory
      float* tb = s_tile_dyn + wib * (2 * 9 * TROW);
      const int nseg = (n + TSEG - 1) / TSEG;
      // lane c < TROW / 4 copies 16-byte column chunk c of the 9 (3 in 2D) rows; row
      // validity and the row's global offset are per item, the column's per segment
      // rows (dy, dz) inside the grid: bit r = 3 (dz + 1) + (dy + 1)
      const unsigned ymask = (y > 0 ? 1u : 0u) | 2u | (y + 1 < g.ny ? 4u : 0u);
      const unsigned zmask = (z > 0 ? 1u : 0u) | 2u | (z + 1 < g.nz ? 4u : 0u);
      const unsigned rowok = D == 2 ? ymask << 3
                                    : ((zmask & 1u) ? ymask : 0u) | ((zmask & 2u) ? ymask << 3 : 0u) |
                                          ((zmask & 4u) ? ymask << 6 : 0u);
      const int64_t rbase = (y - 1) * g.sy + (z - 1) * g.sz;   // row (dy, dz) = (-1, -1)
      const unsigned sbase = (unsigned)__cvta_generic_to_shared(tb) + 16u * (unsigned)lane;
      const unsigned allrows = D == 3 ? 0x1FFu : 0x38u;
      auto fill = [&](int k) {
        const int64_t x0 = cbase * 32 + (int64_t)k * TSEG - 4;   // 16-byte aligned (nx % 4 == 0)
        const int64_t xx = x0 + 4 * lane;
        if (lane < TROW / 4) {
          const unsigned sb = sbase + (unsigned)((k & 1) * (9 * TROW * 4));
          const float* p0 = gfld + rbase + xx;
          if (rowok == allrows && x0 >= 0 && x0 + TROW <= g.nx) {  // warp-uniform: no checks
#pragma unroll
            for (int r = 0; r < 9; r++) {
              if (D == 2 && r / 3 != 1) continue;
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + (unsigned)(r * TROW * 4)),
                           "l"(p0 + (r / 3) * g.sz + (r % 3) * g.sy));
            }
          } else {
            const bool xin = xx >= 0 && xx < g.nx;
#pragma unroll
            for (int r = 0; r < 9; r++) {
              if (D == 2 && r / 3 != 1) continue;
              const bool in = xin && ((rowok >> r) & 1u);
              const float* src = in ? p0 + (r / 3) * g.sz + (r % 3) * g.sy : gfld;
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sb + (unsigned)(r * TROW * 4)),
                           "l"(src), "r"(in ? 16 : 0));
            }
          }
        }
        asm volatile("cp.async.commit_group;");
      };
      fill(0);
      for (int k = 0; k < nseg; k++) {
        if (k + 1 < nseg) {
          fill(k + 1);
          asm volatile("cp.async.wait_group 1;");
        } else {
          asm volatile("cp.async.wait_group 0;");
        }
        __syncwarp();
        const float* buf = tb + (k & 1) * (9 * TROW);
        const int ne = n - k * TSEG < TSEG ? n - k * TSEG : TSEG;
        for (int b0 = 0; b0 < ne; b0 += 32) {
          const int a = b0 + lane;
          const bool act = a < ne;
          const int o = k * TSEG + a;
          uint64_t code = 0, old = 0;
          if (act) {
            old = (uint64_t)cg[row0 + o];   // the memo code, loaded first: its latency overlaps the keys
            const int64_t x = cbase * 32 + o;
            const uint32_t c0 = 0u - 32u * kbase;
            uint32_t W[27];
            const bool interior = rowok == allrows && x > 0 && x + 1 < g.nx;
            const float* bp = buf + a + 3;   // column of dx = -1
#pragma unroll
            for (int r = 0; r < 9; r++)
#pragma unroll
              for (int dx = -1; dx <= 1; dx++) {
                const int p = (dx + 1) + 3 * r;
                if (D == 2 && r / 3 != 1) { W[p] = KEY_OUTSIDE; continue; }
                const uint32_t bv = __float_as_uint(bp[r * TROW + dx + 1]);
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(W[p]) : "r"(bv), "r"(kmul), "r"(c0 + (uint32_t)p));
              }
            if (!interior) {  // positions outside the grid (zero-filled in the tile)
#pragma unroll
              for (int r = 0; r < 9; r++)
#pragma unroll
                for (int dx = -1; dx <= 1; dx++) {
                  const int p = (dx + 1) + 3 * r;
                  const int dz = r / 3 - 1, dy = r % 3 - 1;
                  const bool in = (x + dx >= 0) && (x + dx < g.nx) && (y + dy >= 0) && (y + dy < g.ny) &&
                                  (z + dz >= 0) && (z + dz < g.nz) && (D == 3 || dz == 0);
                  if (!in) W[p] = KEY_OUTSIDE;
                }
            }
            code = cand_of_keys<D>(W, s_lut);
            if (!interior) code |= t_nonex_fill<D>(axes_ok(g, x, y, z));
          }
          // the batch is one 32-anchor chunk (segments of 64 from a 32-aligned group start)
          bool e = false;
          if (act) {
            e = first_round || code != old;
            if (e) cg[row0 + o] = (typename Tr<D>::code_t)code;
            recomputed++;
          }
          const uint32_t bits = __ballot_sync(0xffffffffu, e);
          if (lane == 0 && bits) se[o >> 5] |= bits;
        }
        __syncwarp();   // every lane is done with this buffer before it is refilled
      }
    } else {
      for (int b0 = 0; b0 < n; b0 += 32) {
        const bool act = b0 + lane < n;
        const int o = act ? (dense ? b0 + lane : (int)list[b0 + lane]) : 0;
        uint64_t code = 0, old = 0;
        if (act) {
          const int64_t x = cbase * 32 + o;
          const int64_t v = row0 + o;
          old = (uint64_t)cg[v];
          const int ok = axes_ok(g, x, y, z);
          if (keys) {
            uint32_t W[27];
            load_keys<D>(gfld, g, v, x, y, z, kbase, W);
            code = cand_of_keys<D>(W, s_lut) | t_nonex_fill<D>(ok);
          } else {
            float sv[27];
            load_stencil<D>(gfld, g, v, x, y, z, sv);
            code = cand_of<D>(sv) | t_nonex_fill<D>(ok);
          }
        }
        finish(act, o, code, old);
      }
    }
    if (inrow) ebits[dword_index(g, rg, y, z, cl)] = se[lane];
    __syncwarp();
  }
  warp_add(&cnt->n_swept, swept);
  warp_add(&cnt->n_recomputed, recomputed);
}

// ---------------------------------------------------------------------------
// Target rules with shared-memory tables (one copy per CTA).  The false-cell
// path is rare per anchor in late rounds but, in the first rounds of a dense
// workload, runs ~5 times per anchor: a compact loop over the set bits of the
// false mask keeps the code small.
// ---------------------------------------------------------------------------
struct TargetTables {
  uint2 tv[26];            // x: shift | none << 6 ; y: the packed delta of vertex k at 6 k (k < 4)
  uint32_t fac[26][4];     // dm | ft << 3 | k << 8 | ft's shift << 10 | ft's none << 16 | dm's delta << 20
  uint8_t ldel[26][14];    // link slot -> packed (dx+1) | (dy+1) << 2 | (dz+1) << 4
};

// delta mask (dx = bit 0, dy = bit 1, dz = bit 2) -> packed (dx+1) | (dy+1) << 2 | (dz+1) << 4
__host__ __device__ __forceinline__ uint32_t mask_del(int m) {
  return 0x15u + (m & 1) + ((m & 2) << 1) + ((m & 4) << 2);
}

template <int D>
__device__ __forceinline__ void init_target_tables(TargetTables& T, const Grid& g) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int t = 0; t < Tr<D>::NT; t++) {
      const uint32_t sh = t_dim<D>(t) < Tr<D>::TOP ? (uint32_t)t_shift<D>(t) : 0u;
      const uint32_t no = t_dim<D>(t) < Tr<D>::TOP ? (uint32_t)t_none<D>(t) : 0u;
      uint32_t md = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) md |= mask_del(t_vmask<D>(t, k)) << (6 * k);
      T.tv[t] = make_uint2(sh | (no << 6), md);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int dm = t_facet<D>(t, j, 0), ft = t_facet<D>(t, j, 1);
        const uint32_t fsh = t_dim<D>(ft) < Tr<D>::TOP ? (uint32_t)t_shift<D>(ft) : 0u;
        const uint32_t fno = t_dim<D>(ft) < Tr<D>::TOP ? (uint32_t)t_none<D>(ft) : 0u;
        T.fac[t][j] = (uint32_t)dm | ((uint32_t)ft << 3) | ((uint32_t)t_facet<D>(t, j, 3) << 8) | (fsh << 10) |
                      (fno << 16) | ((mask_del(dm) - 0x15u) << 20);
      }
#pragma unroll
      for (int q = 0; q < 14; q++)
        T.ldel[t][q] = (uint8_t)((t_link<D>(t, q, 0) + 1) | ((t_link<D>(t, q, 1) + 1) << 2) |
                                 ((t_link<D>(t, q, 2) + 1) << 4));
    }
  }
  __syncthreads();
}

template <int N>
__device__ __forceinline__ uint64_t pick(const uint64_t (&c)[N], int i) {
  uint64_t r = c[0];
#pragma unroll
  for (int k = 1; k < N; k++) r = (i == k) ? c[k] : r;
  return r;
}

// field of a code held as two 32-bit halves (funnel shift: one SHF for shift < 32)
__device__ __forceinline__ uint32_t field2(uint2 c, int shift, uint32_t none) {
  const uint32_t w = shift < 32 ? __funnelshift_r(c.x, c.y, shift) : (c.y >> (shift - 32));
  return w & none;
}

// Rules R1 / R2 / R3a / R3b for the false cell (anchor u, type t):
// returns the target's offset from the anchor as packed (dx+1) | (dy+1) << 2 |
// (dz+1) << 4, each component in [-1, 2].  cf0 / cg0 = the anchor's own f / g codes,
// lowpos its f-lowest vertex per type, dp the down-pair facet index per type in g
// (decode_crit_dp); R3b reads the f code of the facet's anchor from global memory
// (u + its delta).  Returns 0xFFFFFFFF on an inconsistency.
//  FP (critical in g, paired in f):  paired up in f -> the cofacet's extra vertex;
//     paired down in f -> m (the vertex the facet lacks is the cell's f-lowest, m).
//  FN (critical in f, paired in g):  paired up in g -> m (R2); paired down with the
//     facet gamma omitting y: y != m -> m (R3a), else the vertex gamma is paired with
//     in f (R3b).
template <int D>
__device__ __forceinline__ uint32_t target_del(const TargetTables& T, int t, bool fn, uint64_t lowpos, uint64_t dp,
                                               uint2 cf0, uint2 cg0, const typename Tr<D>::code_t* __restrict__ cand_f,
                                               int64_t u, const Grid& g) {
  // straight-line (no divergence between the rules inside a warp): every operand is
  // read, the rule is picked with selects
  const int j = (int)(dp >> (2 * t)) & 3;
  const uint32_t fc = T.fac[t][j];
  const int dm = fc & 7;
  // R3b's operand first: its load latency overlaps the rest
  const uint64_t cfg = (uint64_t)__ldg(cand_f + u + mask_delta(g, dm));
  const uint2 tv = T.tv[t];
  const int shift = tv.x & 63;
  const uint32_t none = tv.x >> 6;
  const int mp = (int)(lowpos >> (2 * t)) & 3;
  const uint32_t m_del = (tv.y >> (6 * mp)) & 63;   // m = the cell's f-lowest vertex (SoS)
  const uint32_t a = field2(fn ? cg0 : cf0, shift, none);   // top cells: none = 0 -> a = 0 = none
  const uint32_t r1 = a != none ? (uint32_t)T.ldel[t][a < 14 ? a : 0] : m_del;
  const int ft = (fc >> 3) & 31, k = (fc >> 8) & 3;
  const uint32_t fno = (fc >> 16) & 15;
  const uint32_t s2 = field2(make_uint2((uint32_t)cfg, (uint32_t)(cfg >> 32)), (fc >> 10) & 63, fno);
  const uint32_t r3b = s2 != fno ? (fc >> 20) + T.ldel[ft][s2 < 14 ? s2 : 0] : 0xFFFFFFFFu;  // dm + slot
  const uint32_t r3 = mp != k ? m_del : r3b;      // R3a: y = the vertex gamma omits != m
  return !fn ? r1 : (a != none ? m_del : r3);     // R2: paired up in g -> m
}

// ---------------------------------------------------------------------------
// k_decode: classification.  crit_f is precomputed once per call.  Work item =
// (unit, row, group of DG 32-anchor chunks); an anchor is visited only if a code
// of u + {0,1}^D changed this round ("chg") or it had false cells last round.
//  * had false cells, no code changed: same false cells, same targets (both are
//    functions of those codes, f and fixed tables) -> replay the cached target
//    offsets (tcache) and false-cell count (ncache);
//  * code changed: decode.  The anchors to decode are compacted into full warps
//    (lane = one anchor) so that sparse rows do not pay 32 lanes per anchor.
// Targets go to a shared-memory window over the group's rows y-1..y+2, planes
// z-1..z+2 (x from the group start - 32), flushed with one atomicOr per
// non-empty word into the row-padded target bitmap.
// ---------------------------------------------------------------------------
#ifndef DMTZ_DECODE_THREADS
#define DMTZ_DECODE_THREADS 128
#endif
constexpr int DECODE_THREADS = DMTZ_DECODE_THREADS;
constexpr int TWW = DG + 2;             // window words per row
struct DecodeWarpSmem {
  uint2 cf[32];                // per slot: f code of u
  uint2 cg[32];                // per slot: g code of u
  unsigned long long lowpos[32];
  unsigned long long dp[32];
  unsigned long long tm[32];   // per slot: target offsets of its false cells (bit = packed delta)
  uint32_t tw[16 * TWW];       // target window: 16 rows (dz+1)*4+(dy+1) x TWW words
  uint32_t critf[32];
  uint32_t fm[DG];             // new false-cell marks of the group's chunks
  uint16_t sx[32];             // per slot: anchor offset in the group (chunk * 32 + lane)
  uint16_t list[DG * 32];      // compacted anchor offsets
  uint16_t items[32 * 26];
};

// anchors of the group whose bit is set in the lanes' chunk masks -> W.list (ascending); count
__device__ __forceinline__ int compact_group(uint32_t m, int lane, uint16_t* list) {
  const int n = __popc(m);
  int pre = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += v;
  }
  const int total = __shfl_sync(0xffffffffu, pre, 31);
  pre -= n;
  while (m) {
    const int b = __ffs(m) - 1;
    m &= m - 1;
    list[pre++] = (uint16_t)(lane * 32 + b);
  }
  __syncwarp();
  return total;
}

#ifndef DMTZ_DECODE_MINB
#define DMTZ_DECODE_MINB 8
#endif
template <int D>
__global__ void __launch_bounds__(DECODE_THREADS, DMTZ_DECODE_MINB)
k_decode(const float* __restrict__ f, const typename Tr<D>::code_t* __restrict__ cand_f,
         const uint32_t* __restrict__ crit_f, const typename Tr<D>::code_t* __restrict__ cg,
         const uint32_t* __restrict__ ebits, uint32_t* __restrict__ fmark,
         uint32_t* __restrict__ tbits, const uint32_t* __restrict__ units,
         const unsigned long long* __restrict__ n_units_p, Grid g, RowGeom rg, uint32_t tier_mask,
         const unsigned long long* __restrict__ lowpos_f, unsigned long long* __restrict__ tcache,
         uint8_t* __restrict__ ncache, const LoopState* __restrict__ ls, int64_t own_z0,
         int64_t own_z1, int64_t count_z0, int64_t count_z1, int64_t anchor_z0, int64_t anchor_z1,
         uint32_t* __restrict__ mark_units, Counters* __restrict__ cnt) {
  const bool count_kinds = ls->round == 1;  // kinds are reported for round 1 only
  __shared__ TargetTables T;
  __shared__ DecodeWarpSmem WS[DECODE_THREADS / 32];
  init_target_tables<D>(T, g);
  const int lane = threadIdx.x & 31;
  DecodeWarpSmem& W = WS[threadIdx.x >> 5];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long nfalse = 0, nint = 0, c_dec = 0, c_items = 0, c_rep = 0;
  unsigned int kacc = 0;  // round 1: lane k < 8 counts false cells of kind k
  const uint32_t n_units_ = (uint32_t)*n_units_p;
  const uint32_t ngr = (uint32_t)((rg.wpr + DG - 1) / DG);
  const uint32_t per_unit_ = (uint32_t)UY * ngr;
  const uint32_t total_ = n_units_ * per_unit_;
  for (uint32_t it_ = (uint32_t)warp; it_ < total_; it_ += (uint32_t)nwarps) {
    const uint32_t ui_ = it_ / per_unit_, rem_ = it_ - ui_ * per_unit_;
    const uint32_t unit_ = units[ui_];
    const uint32_t ub_ = (uint32_t)rg.ub;
    const int64_t z = unit_ / ub_;
    const int64_t y = (int64_t)(unit_ - (uint32_t)z * ub_) * UY + rem_ / ngr;
    if (y >= g.ny || z < anchor_z0 || z >= anchor_z1) continue;  // warp-uniform (slab: classified planes)
    const int64_t cbase = (int64_t)(rem_ % ngr) * DG;
    // lane j < DG scans chunk cbase + j: changed-code words of u + {0,1}^D and the false-cell mark
    uint32_t chg_l = 0, had_l = 0;
    const int64_t cl = cbase + lane;
    if (lane < DG && cl < rg.wpr) {
#pragma unroll
      for (int r = 0; r < (D == 3 ? 4 : 2); r++) {
        const int64_t yy = y + (r & 1), zz = z + (r >> 1);
        if (yy >= g.ny || zz >= g.nz) continue;
        const int64_t wi = dword_index(g, rg, yy, zz, cl);
        const uint32_t w0 = __ldg(ebits + wi);
        const uint32_t w1 = (cl + 1 < rg.wpr) ? __ldg(ebits + wi + 1) : 0u;
        chg_l |= w0 | (w0 >> 1) | (w1 << 31);
      }
      had_l = fmark[dword_index(g, rg, y, z, cl)];
      const int64_t rem = g.nx - cl * 32;
      if (rem < 32) chg_l &= (1u << rem) - 1u;
    }
    if (!__any_sync(0xffffffffu, (chg_l | had_l) != 0)) continue;  // warp-uniform
    const bool counted = z >= count_z0 && z < count_z1;  // slab mode: each anchor counted by its owner
    const int64_t row0 = y * g.sy + z * g.sz + cbase * 32;  // anchor index of the group's first x
    for (int i = lane; i < 16 * TWW; i += 32) W.tw[i] = 0u;
    const uint32_t cached_l = had_l & ~chg_l;
    if (lane < DG) W.fm[lane] = cached_l;
    // (1) replay: false cells and targets unchanged since the last evaluation
    {
      const int n = compact_group(cached_l, lane, W.list);
      for (int b0 = 0; b0 < n; b0 += 32) {
        if (b0 + lane < n) {
          const int o = W.list[b0 + lane];
          const int64_t u = row0 + o;
          c_rep++;
          unsigned long long tmc = tcache[u];
          if (counted) nfalse += ncache[u];
          while (tmc) {
            const int del = __ffsll((long long)tmc) - 1;
            tmc &= tmc - 1ull;
            const int X = 32 + o + (del & 3) - 1;
            const int row = ((del >> 4) & 3) * 4 + ((del >> 2) & 3);
            atomicOr(&W.tw[row * TWW + (X >> 5)], 1u << (X & 31));
          }
        }
      }
    }
    // (2) decode the anchors whose codes changed, 32 per pass
    const int ndec = compact_group(chg_l, lane, W.list);
    for (int b0 = 0; b0 < ndec; b0 += 32) {
      const bool act = b0 + lane < ndec;
      const int o = act ? W.list[b0 + lane] : 0;
      const int64_t x = cbase * 32 + o;
      const int64_t u = row0 + o;
      uint32_t diff = 0, critf = 0;
      uint64_t dp = 0, cg0 = 0;
      int ok = 0;
      if (act) {
        uint64_t cgv[Tr<D>::NDELTA];
        ok = axes_ok(g, x, y, z);
#pragma unroll
        for (int dm = 0; dm < Tr<D>::NDELTA; dm++)
          cgv[dm] = (dm & ~ok) == 0 ? (uint64_t)__ldg(cg + u + mask_delta(g, dm)) : Tr<D>::ALL_NONE;
        cg0 = cgv[0];
        const uint32_t cgm = decode_crit_dp<D>(cgv, ok, &dp);
        critf = __ldg(crit_f + u);
        diff = (critf ^ cgm) & tier_mask;
        c_dec++;
      }
      if (!__any_sync(0xffffffffu, diff != 0)) continue;  // warp-uniform
      if (diff) atomicOr(&W.fm[o >> 5], 1u << (o & 31));
      if (count_kinds && counted) {  // round 1: false cells by (dim class, FP / FN)
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const uint32_t cls = (uint32_t)t_dimclass_mask<D>(k >> 1);
          const uint32_t n = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(diff & cls & ((k & 1) ? critf : ~critf)));
          if (lane == k) kacc += n;
        }
      }
      // work list of the false cells (slot, type): all lanes then share them
      const int nmine = __popc(diff);
      if (counted) nfalse += nmine;
      c_items += nmine;
      int pre = nmine;
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, k);
        if (lane >= k) pre += v;
      }
      const int total = __shfl_sync(0xffffffffu, pre, 31);
      pre -= nmine;
      W.tm[lane] = 0ull;
      if (diff) {  // the f code is read only for anchors with false cells
        const uint64_t cfv = (uint64_t)__ldg(cand_f + u);
        W.cf[lane] = make_uint2((uint32_t)cfv, (uint32_t)(cfv >> 32));
        W.cg[lane] = make_uint2((uint32_t)cg0, (uint32_t)(cg0 >> 32));
        W.critf[lane] = critf;
        W.dp[lane] = dp;
        W.lowpos[lane] = __ldg(lowpos_f + u);
        W.sx[lane] = (uint16_t)o;
        uint32_t dd = diff;
        for (int k = 0; dd; k++) {
          const int t = __ffs(dd) - 1;
          dd &= dd - 1;
          W.items[pre + k] = (uint16_t)(lane | (t << 5));
        }
      }
      __syncwarp();
      // targets -> window (x relative to the group start - 32)
      for (int i0 = 0; i0 < total; i0 += 32) {
        const int i = i0 + lane;
        const bool live = i < total;
        const int item = live ? W.items[i] : 0;
        const int src = item & 31, t = item >> 5;
        const bool fn = (W.critf[src] >> t) & 1u;
        if (!live) continue;
        const uint32_t del = target_del<D>(T, t, fn, W.lowpos[src], W.dp[src], W.cf[src], W.cg[src], cand_f,
                                           row0 + W.sx[src], g);
        if (del == 0xFFFFFFFFu) { nint++; continue; }
        const int X = 32 + W.sx[src] + (int)(del & 3) - 1;
        const int row = (int)((del >> 4) & 3) * 4 + (int)((del >> 2) & 3);   // (dz+1) * 4 + (dy+1)
        atomicOr(&W.tw[row * TWW + (X >> 5)], 1u << (X & 31));
        atomicOr((uint32_t*)&W.tm[src] + ((del >> 5) & 1), 1u << (del & 31));   // native 32-bit smem atomic
      }
      __syncwarp();
      if (diff) {  // evaluated anchors refresh their cache entry
        tcache[u] = W.tm[lane];
        ncache[u] = (uint8_t)nmine;
      }
      __syncwarp();
    }
    __syncwarp();
    if (lane < DG && cl < rg.wpr && W.fm[lane] != had_l) fmark[dword_index(g, rg, y, z, cl)] = W.fm[lane];
    // slab mode: a unit with false cells stays in the frontier (its targets may be another rank's)
    if (mark_units && __any_sync(0xffffffffu, lane < DG && W.fm[lane & (DG - 1)] != 0u) && lane == 0) {
      const int64_t unit = z * rg.ub + y / UY;
      atomicOr(mark_units + (unit >> 5), 1u << (unit & 31));
    }
    // flush the window: one aligned atomicOr per non-empty word (row-padded target bitmap)
    for (int i = lane; i < 16 * TWW; i += 32) {
      const uint32_t wv = W.tw[i];
      if (!wv) continue;
      const int row = i / TWW, wd = i - row * TWW;
      const int64_t ty = y + (row & 3) - 1, tz = z + (row >> 2) - 1, tc = cbase + wd - 1;
      if (tz < own_z0 || tz >= own_z1) continue;   // slab mode: only the owned vertices
      atomicOr(tbits + dword_index(g, rg, ty, tz, tc), wv);
    }
    __syncwarp();
  }
  warp_add(&cnt->n_false, nfalse);
  warp_add(&cnt->n_internal, nint);
  warp_add(&cnt->n_decoded, c_dec);
  warp_add(&cnt->n_items, c_items);
  warp_add(&cnt->n_replayed, c_rep);
  if (count_kinds && lane < 8 && kacc) atomicAdd(&cnt->kinds[lane], (unsigned long long)kacc);
}

// ---------------------------------------------------------------------------
// Slab halo refresh: new values of planes [z0, z1) from a neighbour rank; changed
// vertices go to the change bitmap the next screen reads and mark the frontier
// units meeting v + [-2,1]^3, exactly as this rank's own edits do.  One warp per
// 32-vertex row chunk.
// ---------------------------------------------------------------------------
// (ctl != nullptr: batched multi-GPU mode -- nothing to do once halted (ctl[0]) or when
// the neighbour's face flag ctl[gate] says its planes did not change)
__global__ void k_halo(float* __restrict__ gf, const float* __restrict__ planes, int64_t z0, int64_t z1, Grid g,
                       RowGeom rg, uint32_t* __restrict__ vchg_round, uint32_t* __restrict__ frontier,
                       const long long* __restrict__ ctl = nullptr, int gate = 0) {
  if (ctl && (ctl[0] || !ctl[gate])) return;
  const int lane = threadIdx.x & 31;
  const int64_t nitems = (z1 - z0) * g.ny * rg.wpr;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nitems;
       it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t c = it % rg.wpr, row = it / rg.wpr;
    const int64_t y = row % g.ny, z = z0 + row / g.ny;
    const int64_t x = c * 32 + lane;
    bool ch = false;
    if (x < g.nx) {
      const int64_t v = x + y * g.sy + z * g.sz;
      const float nv = planes[v - z0 * g.sz];
      if (__float_as_uint(nv) != __float_as_uint(gf[v])) { gf[v] = nv; ch = true; }
    }
    const unsigned b = __ballot_sync(0xffffffffu, ch);
    if (!b) continue;  // warp-uniform
    if (lane == 0) atomicOr(vchg_round + dword_index(g, rg, y, z, c), b);
    if (lane < 8) {
      const int64_t y0 = y >= 2 ? y - 2 : 0, y1 = y + 1 < g.ny ? y + 1 : g.ny - 1;
      const int64_t zz = (z >= 2 ? z - 2 : 0) + (lane >> 1), zt = z + 1 < g.nz ? z + 1 : g.nz - 1;
      const int64_t bb = y0 / UY + (lane & 1);
      if (zz <= zt && bb <= y1 / UY) {
        const int64_t unit = zz * rg.ub + bb;
        atomicOr(frontier + (unit >> 5), 1u << (unit & 31));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Edits (a6) + next frontier.  One warp per 32 target-bitmap words; lanes take
// the 32 bits of each non-empty word in parallel.  The frontier (a7) marks the
// units meeting v + [-2,1]^D for every target v (a value change at v can alter
// only cells anchored there, and every false cell is anchored there relative
// to its own target), aggregated in shared memory when it fits.
// ---------------------------------------------------------------------------
#ifndef DMTZ_EDIT_NW
#define DMTZ_EDIT_NW 2
#endif
constexpr int EDIT_NW = DMTZ_EDIT_NW;
template <int D>
__global__ void k_edit_rows(uint32_t* __restrict__ tbits, int64_t nwords, const float* __restrict__ fhat,
                            const float* __restrict__ lb, float* __restrict__ gf, uint32_t* __restrict__ state,
                            Counters* __restrict__ cnt, float step, int q_cap, uint32_t* __restrict__ next_frontier,
                            Grid g, RowGeom rg, int fwords_smem, uint32_t* __restrict__ vchg, int64_t vwords,
                            const LoopState* __restrict__ ls, FastDiv div_wpr, FastDiv div_ny) {
  uint32_t* vcur = vchg ? vchg + (int64_t)(ls->round & 1) * vwords : nullptr;
  // each block takes a contiguous word range, so its frontier units span a few planes
  const int64_t per_block = ((nwords + gridDim.x - 1) / gridDim.x + 31) / 32 * 32;
  const int64_t w_begin = (int64_t)blockIdx.x * per_block;
  const int64_t w_end = w_begin + per_block < nwords ? w_begin + per_block : nwords;
  if (w_begin >= w_end) return;  // block-uniform
  // frontier words this block can touch: units of planes z_first - 2 .. z_last + 1
  const int64_t z_first = (w_begin / rg.wpr) / g.ny, z_last = ((w_end - 1) / rg.wpr) / g.ny;
  const int64_t fz0 = z_first >= 2 ? z_first - 2 : 0, fz1 = z_last + 1 < g.nz ? z_last + 1 : g.nz - 1;
  const int64_t fw0 = (fz0 * rg.ub) >> 5, fw1 = (((fz1 + 1) * rg.ub - 1) >> 5) + 1;
  extern __shared__ uint32_t sfr[];
  const bool use_smem = fwords_smem && fw1 - fw0 <= fwords_smem;
  if (use_smem)
    for (int64_t i = threadIdx.x; i < fw1 - fw0; i += blockDim.x) sfr[i] = 0;
  __syncthreads();
  unsigned long long changed = 0, targets = 0;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  for (int64_t base = w_begin + (int64_t)wib * 32; base < w_end; base += (int64_t)nwb * 32) {
    const int64_t wi = base + lane;
    uint32_t word = wi < w_end ? tbits[wi] : 0u;
    if (word) tbits[wi] = 0;
    unsigned nz = __ballot_sync(0xffffffffu, word != 0);
    if (next_frontier && nz) {
      // the units meeting (y, z) + [-2, 1] depend on the row only: marked once per row of
      // this pass that has a target word (its first such lane), 8 lanes per row
      const uint32_t wr = div_wpr.div((uint32_t)wi);             // word indices < 2^32 (host check)
      const int l0 = lane - (int)((uint32_t)wi - wr * (uint32_t)rg.wpr);   // the row's first lane
      const unsigned below = (1u << lane) - 1u, rowlanes = l0 > 0 ? below & ~((1u << l0) - 1u) : below;
      unsigned firsts = __ballot_sync(0xffffffffu, word != 0 && !(nz & rowlanes));
      while (firsts) {
        const int fl = __ffs(firsts) - 1;
        firsts &= firsts - 1;
        const uint32_t wrow32 = __shfl_sync(0xffffffffu, wr, fl);
        if (lane < 8) {  // <= 4 planes x 2 row blocks
          const uint32_t vz32 = div_ny.div(wrow32);
          const int64_t vz = vz32, vy = (int64_t)(wrow32 - vz32 * (uint32_t)g.ny);
          const int64_t y0 = vy >= 2 ? vy - 2 : 0, y1 = vy + 1 < g.ny ? vy + 1 : g.ny - 1;
          const int64_t zz = (vz >= 2 ? vz - 2 : 0) + (lane >> 1), z1 = vz + 1 < g.nz ? vz + 1 : g.nz - 1;
          const int64_t b = y0 / UY + (lane & 1);
          if (zz <= z1 && b <= y1 / UY) {
            const int64_t unit = zz * rg.ub + b;
            if (use_smem) atomicOr(sfr + ((unit >> 5) - fw0), 1u << (unit & 31));
            else atomicOr(next_frontier + (unit >> 5), 1u << (unit & 31));
          }
        }
      }
    }
    // EDIT_NW target words per pass: their loads are independent, one memory round trip
    while (nz) {
      int src[EDIT_NW];
#pragma unroll
      for (int h = 0; h < EDIT_NW; h++) {
        src[h] = nz ? __ffs(nz) - 1 : -1;
        if (nz) nz &= nz - 1;
      }
      uint32_t st[EDIT_NW];
      float fh[EDIT_NW], lbv[EDIT_NW];
      int64_t v[EDIT_NW];
      bool mine[EDIT_NW];
#pragma unroll
      for (int h = 0; h < EDIT_NW; h++) { st[h] = 0u; fh[h] = 0.f; lbv[h] = 0.f; v[h] = 0; }
#pragma unroll
      for (int h = 0; h < EDIT_NW; h++) {
        const int sw = src[h] < 0 ? src[0] : src[h];
        const uint32_t wv = __shfl_sync(0xffffffffu, word, sw);
        mine[h] = src[h] >= 0 && ((wv >> lane) & 1u);
        if (src[h] < 0) continue;  // warp-uniform
        // row-padded target bitmap: word = (z * ny + y) * wpr + x / 32; all its targets share (y, z)
        const uint32_t wrow32 = div_wpr.div((uint32_t)(base + sw));   // word indices < 2^32 (host check)
        const uint32_t vz32 = div_ny.div(wrow32);
        const int64_t wrow = wrow32, vz = vz32, vy = (int64_t)(wrow32 - vz32 * (uint32_t)g.ny);
        if (mine[h]) {
          v[h] = ((base + sw) - wrow * rg.wpr) * 32 + lane + vy * g.sy + vz * g.sz;
          st[h] = state[v[h]];
          fh[h] = __ldg(fhat + v[h]);
          lbv[h] = __ldg(lb + v[h]);
        }
      }
#pragma unroll
      for (int h = 0; h < EDIT_NW; h++) {
        bool ch = false;
        if (mine[h]) {
          targets++;
          if (!(st[h] >> 16)) {  // lossless targets are no-ops, but their cells stay in the frontier
            ch = true;
            changed++;
            const uint32_t q = st[h] & 0xFFFFu;
            // g' = RN(fhat - RN((q+1) * step)): two roundings, never fused
            const float gp = __fsub_rn(fh[h], __fmul_rn((float)(q + 1), step));
            if ((int)q + 1 <= q_cap && gp >= lbv[h]) {
              state[v[h]] = q + 1;
              gf[v[h]] = gp;
            } else {
              gf[v[h]] = lbv[h];        // clamp to the lower bound, stored losslessly
              state[v[h]] = q | (1u << 16);
            }
          }
        }
        const unsigned cb = __ballot_sync(0xffffffffu, ch);
        if (vcur && lane == 0 && cb) atomicOr(vcur + base + src[h], cb);   // same row-padded word index
      }
    }
  }
  warp_add(&cnt->n_changed, changed);
  warp_add(&cnt->n_targets, targets);
  if (use_smem) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < fw1 - fw0; i += blockDim.x)
      if (sfr[i]) atomicOr(next_frontier + fw0 + i, sfr[i]);
  }
}

// Per anchor and cell type: position (in the type's vertex list) of the cell's
// lowest vertex under f in the SoS order -- 2 bits per type.  Computed
// once per call; the target rules read it instead of re-sorting f.
template <int D>
__global__ void k_lowpos(const float* __restrict__ f, unsigned long long* __restrict__ out, Grid g) {
  const float INF = __int_as_float(0x7f800000);
  DMTZ_FOR_ANCHORS(g, 0, g.nz) {
    const int64_t v = x + y * g.sy + z * g.sz;
    const int ok = axes_ok(g, x, y, z);
    float c[8];
#pragma unroll
    for (int dm = 0; dm < 8; dm++) {
      if (D == 2 && dm >= 4) { c[dm] = INF; continue; }
      c[dm] = ((dm & ~ok) == 0) ? __ldg(f + v + mask_delta(g, dm)) : INF;
    }
    uint64_t w = 0;
#pragma unroll
    for (int t = 0; t < Tr<D>::NT; t++) {
      int best = 0;
      float fb = c[t_vmask<D>(t, 0)];
#pragma unroll
      for (int k = 1; k < 4; k++) {
        if (k < t_nv<D>(t)) {
          // vertices are listed in ascending index order: ties keep the earlier one
          const float fv = c[t_vmask<D>(t, k)];
          if (fv < fb) { fb = fv; best = k; }
        }
      }
      w |= (uint64_t)best << (2 * t);
    }
    out[v] = w;
  }
}

// active unit list from the frontier bitmap (ordered compaction), count -> *n_out
__global__ void k_units_from_bits(uint32_t* __restrict__ fbits, int64_t n_units, uint32_t* __restrict__ list,
                                  unsigned long long* __restrict__ n_out, const long long* __restrict__ halt = nullptr) {
  if (halt && *halt) return;  // batched multi-GPU rounds after the stop: empty list
  // single pass with one atomic per warp; order inside the list does not matter
  const int lane = threadIdx.x & 31;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane; base < n_units;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = base + lane;
    const uint32_t word = u < n_units ? fbits[u >> 5] : 0u;
    const bool on = (word >> (u & 31)) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0 && u < n_units) fbits[u >> 5] = 0u;  // cleared for the next round
    unsigned long long pos = 0;
    if (lane == 0 && bal) pos = atomicAdd(n_out, (unsigned long long)__popc(bal));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (on) list[pos + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)u;
  }
}

// units of the z-planes [z0, z1) (all units: z0 = 0, z1 = nz); unit = z * ub + y-block
__global__ void k_units_all(int64_t ub, int64_t z0, int64_t z1, uint32_t* __restrict__ list,
                            unsigned long long* __restrict__ n_out, const long long* __restrict__ halt = nullptr) {
  if (halt && *halt) return;
  const int64_t n = (z1 - z0) * ub;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    list[i] = (uint32_t)(z0 * ub + i);
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = (unsigned long long)(n > 0 ? n : 0);
}

}  // namespace dmtz
