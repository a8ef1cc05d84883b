// dmtz_sweep3d.cuh -- the fused 3D round sweep (a3 + a4 + a5) for sm_100a.
//
// One CTA owns a BRICK of anchors: 31 (x) x 16 (y) x 32 (z).  Warp w computes
// gradient codes of g for code row y0 + w (w = 0..16, row 16 is the +y halo),
// lanes 0..31 for x0 .. x0+31 (lane 31 is the +x halo), marching up the brick's
// z planes with a 4-plane ring of g values in shared memory (values carry a
// one-vertex halo on every side; +inf outside the grid).  Codes of planes z and
// z+1 stay in shared memory, so every anchor's code is computed once per brick
// and the critical-cell decode (codes at u + {0,1}^3) reads shared memory only.
//
// Screening: crit_g(u) = crit_f(u) whenever cand_g = cand_f at all of u+{0,1}^3
// (a cell's criticality is a function of those 8 codes, include/dmtz.h).  A
// warp ballot of cand_g != cand_f per code row gives the anchors that need the
// full decode; the rest cost one 64-bit compare.
//
// False cells: targets by rules R1/R2/R3a/R3b, unrolled over
// the 26 cell types so every table entry is an immediate; target bits are
// OR-ed into the round's target bitmap.
#pragma once
#include "dmtz_kernels.cuh"

namespace dmtz {
namespace sw3 {
constexpr int TXC = 32;          // code columns per row (31 useful + 1 halo)
constexpr int TXU = 31;          // useful anchors per row
constexpr int TY = 16;           // useful rows
constexpr int TYC = TY + 1;      // code rows = warps
constexpr int TZ = 32;           // useful planes per brick
constexpr int VX = TXC + 2;      // value columns x0-1 .. x0+32
constexpr int VY = TYC + 2;      // value rows    y0-1 .. y0+17
constexpr int VPLANE = VX * VY;
constexpr int THREADS = TYC * 32;
}  // namespace sw3

struct BrickGeom {
  int64_t bx, by, bz;  // bricks per axis
};

__host__ __device__ inline BrickGeom brick_geom3(const Grid& g) {
  BrickGeom b;
  b.bx = (g.nx + sw3::TXU - 1) / sw3::TXU;
  b.by = (g.ny + sw3::TY - 1) / sw3::TY;
  b.bz = (g.nz + sw3::TZ - 1) / sw3::TZ;
  return b;
}

struct SweepSmem3 {
  float val[4][sw3::VPLANE];
  unsigned long long cg[2][sw3::TYC][sw3::TXC];
  unsigned long long cf[2][sw3::TYC][sw3::TXC];
  unsigned int dm[2][sw3::TYC];
  unsigned long long cnt[12];
};

// stencil accessor used by the generated k3d::cand_code (positions p = dx+1 + 3(dy+1) + 9(dz+1))
struct Stencil3 {
  float v[27];
};

__device__ __forceinline__ void load_plane3(float* dst, const float* __restrict__ fld, const Grid& g, int64_t x0,
                                            int64_t y0, int64_t z) {
  const float INF = __int_as_float(0x7f800000);
  const bool zin = z >= 0 && z < g.nz;
  for (int i = threadIdx.x; i < sw3::VPLANE; i += blockDim.x) {
    const int r = i / sw3::VX, c = i - r * sw3::VX;
    const int64_t x = x0 - 1 + c, y = y0 - 1 + r;
    float v = INF;
    if (zin && x >= 0 && x < g.nx && y >= 0 && y < g.ny) v = __ldg(fld + x + y * g.sy + z * g.sz);
    dst[i] = v;
  }
}

template <int T>
__device__ __forceinline__ uint32_t fld3(uint64_t code) {
  return (uint32_t)(code >> k3d::SHIFT[T]) & (uint32_t)k3d::NONE[T];
}

// Static target rule for type T (see target_of in dmtz_kernels.cuh for the dynamic twin).
template <int T>
__device__ __forceinline__ int64_t target_static3(const float* __restrict__ f, const Grid& g, int64_t u,
                                                  const uint64_t (&cf)[8], const uint64_t (&cg)[8], bool fn) {
  constexpr int nv = k3d::NV[T];
  int64_t vid[4];
  int64_t m = -1;
  float fm = 0.f;
#pragma unroll
  for (int k = 0; k < nv; k++) {
    vid[k] = u + mask_delta(g, k3d::VMASK[T][k]);
    const float fv = __ldg(f + vid[k]);
    if (k == 0 || sos_less(fv, vid[k], fm, m)) { m = vid[k]; fm = fv; }
  }
  if (!fn) {
    if constexpr (k3d::DIM[T] < 3) {
      const uint32_t s = fld3<T>(cf[0]);
      if (s != (uint32_t)k3d::NONE[T]) {
        // dynamic slot -> link offset: small unrolled select
        int64_t off = 0;
#pragma unroll
        for (int j = 0; j < k3d::NLINK[T]; j++)
          if (s == (uint32_t)j) off = k3d::LINK[T][j][0] + k3d::LINK[T][j][1] * g.sy + k3d::LINK[T][j][2] * g.sz;
        return u + off;
      }
    }
    return m;
  }
  if constexpr (k3d::DIM[T] < 3) {
    if (fld3<T>(cg[0]) != (uint32_t)k3d::NONE[T]) return m;
  }
#pragma unroll
  for (int j = 0; j < k3d::NFACET[T]; j++) {
    const int dm = k3d::FACET[T][j][0], ft = k3d::FACET[T][j][1], sl = k3d::FACET[T][j][2], k = k3d::FACET[T][j][3];
    if (((uint32_t)(cg[dm] >> k3d::SHIFT[ft]) & (uint32_t)k3d::NONE[ft]) != (uint32_t)sl) continue;
    if (m != vid[k]) return m;
    const uint32_t s2 = (uint32_t)(cf[dm] >> k3d::SHIFT[ft]) & (uint32_t)k3d::NONE[ft];
    if (s2 == (uint32_t)k3d::NONE[ft]) return -1;
    int64_t off = 0;
#pragma unroll
    for (int q = 0; q < 6; q++)
      if (q < k3d::NLINK[ft] && s2 == (uint32_t)q)
        off = k3d::LINK[ft][q][0] + k3d::LINK[ft][q][1] * g.sy + k3d::LINK[ft][q][2] * g.sz;
    return u + mask_delta(g, dm) + off;
  }
  return -1;
}

template <int T>
__device__ __forceinline__ void handle_type3(uint32_t diff, uint32_t critf, const float* __restrict__ f,
                                             const Grid& g, int64_t u, const uint64_t (&cf)[8],
                                             const uint64_t (&cg)[8], uint32_t* __restrict__ tbits,
                                             unsigned long long (&k)[8], unsigned long long& nint) {
  if (!((diff >> T) & 1u)) return;
  const bool fn = (critf >> T) & 1u;
  constexpr int d = k3d::DIM[T];
  constexpr int cls = d;  // 3D: min, 1-saddle, 2-saddle, max = dims 0..3
  if (fn) k[2 * cls + 1]++; else k[2 * cls]++;
  const int64_t tv = target_static3<T>(f, g, u, cf, cg, fn);
  if (tv < 0) { nint++; return; }
  atomicOr(tbits + (tv >> 5), 1u << (tv & 31));
}

template <int... Ts>
struct TypeList {};

template <int... Ts>
__device__ __forceinline__ void handle_all3(TypeList<Ts...>, uint32_t diff, uint32_t critf, const float* __restrict__ f,
                                            const Grid& g, int64_t u, const uint64_t (&cf)[8], const uint64_t (&cg)[8],
                                            uint32_t* __restrict__ tbits, unsigned long long (&k)[8],
                                            unsigned long long& nint) {
  (handle_type3<Ts>(diff, critf, f, g, u, cf, cg, tbits, k, nint), ...);
}

using AllTypes3 = TypeList<0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23,
                           24, 25>;

// frontier: bit per brick; nullptr = sweep everything
__global__ void __launch_bounds__(sw3::THREADS, 1)
k_sweep3(const float* __restrict__ f, const float* __restrict__ gfld, const unsigned long long* __restrict__ cand_f,
         uint32_t* __restrict__ tbits, const uint32_t* __restrict__ frontier, Counters* __restrict__ cnt, Grid g,
         BrickGeom bg, uint32_t tier_mask) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SweepSmem3& S = *reinterpret_cast<SweepSmem3*>(smem_raw);
  const int64_t bid = blockIdx.x;
  if (frontier && !((frontier[bid >> 5] >> (bid & 31)) & 1u)) return;
  const int64_t bxi = bid % bg.bx, byi = (bid / bg.bx) % bg.by, bzi = bid / (bg.bx * bg.by);
  const int64_t x0 = bxi * sw3::TXU, y0 = byi * sw3::TY, z0 = bzi * sw3::TZ;
  const int64_t z1 = min(z0 + sw3::TZ, g.nz);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t x = x0 + lane, y = y0 + w;
  const bool anchor_in = x < g.nx && y < g.ny;
  const int ok_xy = (x + 1 < g.nx ? 1 : 0) | (y + 1 < g.ny ? 2 : 0);

  unsigned long long kinds[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long nfalse = 0, nint = 0, nswept = 0;

  // codes of plane z for this thread's anchor -> smem slot (z & 1); returns nothing
  auto code_plane = [&](int64_t z) {
    const int slot = (int)(z & 1);
    uint64_t cgv = Tr<3>::ALL_NONE, cfv = Tr<3>::ALL_NONE;
    if (anchor_in && z < g.nz) {
      const float* p0 = S.val[(z + 3) & 3];  // plane z-1
      const float* p1 = S.val[z & 3];
      const float* p2 = S.val[(z + 1) & 3];
      Stencil3 st;
      const int c = (w + 1) * sw3::VX + (lane + 1);
#pragma unroll
      for (int dz = -1; dz <= 1; dz++)
#pragma unroll
        for (int dy = -1; dy <= 1; dy++)
#pragma unroll
          for (int dx = -1; dx <= 1; dx++) {
            const float* pl = dz < 0 ? p0 : (dz == 0 ? p1 : p2);
            st.v[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] = pl[c + dy * sw3::VX + dx];
          }
      const int ok = ok_xy | (z + 1 < g.nz ? 4 : 0);
      cgv = k3d::cand_code(st.v) | k3d::NONEX_FILL[ok];
      cfv = __ldg(cand_f + x + y * g.sy + z * g.sz);
    }
    S.cg[slot][w][lane] = cgv;
    S.cf[slot][w][lane] = cfv;
    const unsigned bal = __ballot_sync(0xffffffffu, cgv != cfv);
    if (lane == 0) S.dm[slot][w] = bal;
  };

  // prologue: planes z0-1, z0, z0+1 -> codes of plane z0
  load_plane3(S.val[(z0 + 3) & 3], gfld, g, x0, y0, z0 - 1);
  load_plane3(S.val[z0 & 3], gfld, g, x0, y0, z0);
  load_plane3(S.val[(z0 + 1) & 3], gfld, g, x0, y0, z0 + 1);
  __syncthreads();
  code_plane(z0);
  for (int64_t z = z0; z < z1; z++) {
    load_plane3(S.val[(z + 2) & 3], gfld, g, x0, y0, z + 2);
    __syncthreads();
    code_plane(z + 1);
    __syncthreads();
    // decode plane z: useful anchors are lanes 0..30, warps 0..15
    if (w < sw3::TY && lane < sw3::TXU && anchor_in) {
      nswept++;
      const int s0 = (int)(z & 1), s1 = s0 ^ 1;
      const unsigned need = S.dm[s0][w] | S.dm[s0][w + 1] | S.dm[s1][w] | S.dm[s1][w + 1];
      if ((need >> lane) & 3u) {
        uint64_t cf[8], cg[8];
#pragma unroll
        for (int dm = 0; dm < 8; dm++) {
          const int sl = (dm & 4) ? s1 : s0;
          const int yy = w + ((dm >> 1) & 1), xx = lane + (dm & 1);
          cg[dm] = S.cg[sl][yy][xx];
          cf[dm] = S.cf[sl][yy][xx];
        }
        const int ok = ok_xy | (z + 1 < g.nz ? 4 : 0);
        const uint32_t critf = decode_crit<3>(cf, ok), critg = decode_crit<3>(cg, ok);
        const uint32_t diff = (critf ^ critg) & tier_mask;
        if (diff) {
          nfalse += __popc(diff);
          handle_all3(AllTypes3{}, diff, critf, f, g, x + y * g.sy + z * g.sz, cf, cg, tbits, kinds, nint);
        }
      }
    }
  }
  warp_add(&cnt->n_false, nfalse);
  warp_add(&cnt->n_internal, nint);
  warp_add(&cnt->n_swept, nswept);
#pragma unroll
  for (int k = 0; k < 8; k++) warp_add(&cnt->kinds[k], kinds[k]);
}

// Eq. 2 edits on the marked targets + next-round frontier (bricks meeting v + [-2,1]^3).
// One warp per 32-word chunk; lanes take the 32 bits of each non-empty word in parallel.
__global__ void k_edit3(uint32_t* __restrict__ tbits, int64_t nwords, const float* __restrict__ fhat,
                        const float* __restrict__ lb, float* __restrict__ gf, uint32_t* __restrict__ state,
                        Counters* __restrict__ cnt, float step, int q_cap, uint32_t* __restrict__ next_frontier,
                        Grid g, BrickGeom bg, int fwords_smem) {
  extern __shared__ uint32_t sfr[];  // block-local copy of the next frontier (fwords_smem words, 0 = global atomics)
  for (int i = threadIdx.x; i < fwords_smem; i += blockDim.x) sfr[i] = 0;
  __syncthreads();
  uint32_t* fr = fwords_smem ? sfr : next_frontier;
  unsigned long long changed = 0, targets = 0;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp0 * 32; base < nwords; base += nwarps * 32) {
    const int64_t wi = base + lane;
    uint32_t word = wi < nwords ? tbits[wi] : 0u;
    if (word) tbits[wi] = 0;
    unsigned nz = __ballot_sync(0xffffffffu, word != 0);
    while (nz) {
      const int src = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t wv = __shfl_sync(0xffffffffu, word, src);
      if (!((wv >> lane) & 1u)) continue;
      const int64_t v = (base + src) * 32 + lane;
      targets++;
      if (next_frontier) {
        const int64_t vx = v % g.nx, vy = (v / g.nx) % g.ny, vz = v / (g.nx * g.ny);
        const int64_t ax0 = (vx >= 2 ? vx - 2 : 0) / sw3::TXU, ax1 = (vx + 1 < g.nx ? vx + 1 : g.nx - 1) / sw3::TXU;
        const int64_t ay0 = (vy >= 2 ? vy - 2 : 0) / sw3::TY, ay1 = (vy + 1 < g.ny ? vy + 1 : g.ny - 1) / sw3::TY;
        const int64_t az0 = (vz >= 2 ? vz - 2 : 0) / sw3::TZ, az1 = (vz + 1 < g.nz ? vz + 1 : g.nz - 1) / sw3::TZ;
        for (int64_t bz = az0; bz <= az1; bz++)
          for (int64_t by = ay0; by <= ay1; by++)
            for (int64_t bx = ax0; bx <= ax1; bx++) {
              const int64_t b = bx + bg.bx * (by + bg.by * bz);
              atomicOr(fr + (b >> 5), 1u << (b & 31));
            }
      }
      const uint32_t st = state[v];
      if (st >> 16) continue;  // lossless: no-op (still keeps its bricks in the frontier)
      changed++;
      const uint32_t q = st & 0xFFFFu;
      if ((int)q + 1 <= q_cap) {
        const float gp = __fsub_rn(fhat[v], __fmul_rn((float)(q + 1), step));
        if (gp >= lb[v]) { state[v] = q + 1; gf[v] = gp; continue; }
      }
      gf[v] = lb[v];
      state[v] = q | (1u << 16);
    }
  }
  warp_add(&cnt->n_changed, changed);
  warp_add(&cnt->n_targets, targets);
  if (fwords_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < fwords_smem; i += blockDim.x)
      if (sfr[i]) atomicOr(next_frontier + i, sfr[i]);
  }
}

}  // namespace dmtz
