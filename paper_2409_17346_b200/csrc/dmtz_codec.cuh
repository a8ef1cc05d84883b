// dmtz_codec.cuh -- the edit list as a storable artifact:
// the quantized representation of edits ("store only the integer count
// of edits q for each vertex"; lossless entries keep their value bits) as a
// byte stream, and the decompression-side application of the edits (Fig. 2: "the
// edits are applied to the decompressed data").
//
// Stream layout (little-endian, include/dmtz.h documents it for users):
//   0   char[4]  "DMTE"
//   4   uint32   version (1: lossless values as raw bits; 2: relative to fhat)
//   8   uint64   n_edits
//   16  uint32   edits per block (EC_BLOCK)
//   20  int32    q_max
//   24  float    xi
//   28  uint32   n_blocks = ceil(n_edits / EC_BLOCK)
//   32  uint64   block_offset[n_blocks]   byte offset of each block's first record in the payload
//   32 + 8 n_blocks: payload, one record per edit in ascending vertex order:
//        varint(delta) varint(q << 1 | lossless) [lossless only: v1 uint32 value bits;
//        v2 varint(zigzag(int(fhat bits) - int(value bits))), int = the bits as int32,
//        the difference in int64 -- small because |value - fhat| <= 2 xi]
//        delta = v for the first edit of a block, else v - v_prev - 1
//   varint = unsigned LEB128 (7 bits per byte, low groups first, bit 7 = more).
// Blocks make the decoder parallel (version 2: one warp per block, k_ec_decode_v2w;
// version 1: one thread per block); the encoder is a per-edit length pass, an
// exclusive scan and a per-edit write.
#pragma once

#include "dmtz_kernels.cuh"
#include "dmtz_trace.cuh"

namespace dmtz {

constexpr int EC_BLOCK = 4096;
constexpr size_t EC_HEADER = 32;

struct EditRec { unsigned long long v; unsigned short q; unsigned char lossless; unsigned char pad; float value; };
static_assert(sizeof(EditRec) == 16, "dmtz_edit is 16 bytes");

__host__ __device__ inline int varint_len(unsigned long long x) {
  int n = 1;
  while (x >= 128ull) { x >>= 7; n++; }
  return n;
}

__device__ __forceinline__ unsigned long long zz_rel(float fhat, float value) {
  const long long d = (long long)__float_as_int(fhat) - (long long)__float_as_int(value);
  return ((unsigned long long)d << 1) ^ (unsigned long long)(d >> 63);
}
__device__ __forceinline__ float unzz_rel(float fhat, unsigned long long z) {
  const long long d = (long long)(z >> 1) ^ -(long long)(z & 1ull);
  return __int_as_float((int)((long long)__float_as_int(fhat) - d));
}

__device__ __forceinline__ unsigned long long rec_delta(const EditRec* __restrict__ e, int64_t i) {
  return (i % EC_BLOCK) == 0 ? e[i].v : e[i].v - e[i - 1].v - 1ull;
}

// len[i] = bytes of record i; len[n] = 0 (the exclusive scan then leaves the total there).
// Edits must be sorted strictly ascending and carry q < 2^15: violations count into *bad.
__global__ void k_ec_len(const EditRec* __restrict__ e, int64_t n, const float* __restrict__ fhat,
                         long long* __restrict__ len, unsigned long long* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { len[n] = 0; continue; }
    const EditRec r = e[i];
    if ((i > 0 && r.v <= e[i - 1].v) || r.lossless > 1) atomicAdd(bad, 1ull);
    const unsigned long long code = ((unsigned long long)r.q << 1) | r.lossless;
    len[i] = varint_len(rec_delta(e, i)) + varint_len(code) +
             (r.lossless ? (fhat ? varint_len(zz_rel(fhat[r.v], r.value)) : 4) : 0);
  }
}

__device__ __forceinline__ int put_varint(uint8_t* p, unsigned long long x) {
  int k = 0;
  while (x >= 128ull) { p[k++] = (uint8_t)(x | 128u); x >>= 7; }
  p[k++] = (uint8_t)x;
  return k;
}

__global__ void k_ec_write(const EditRec* __restrict__ e, int64_t n, const long long* __restrict__ off, float xi,
                           int q_max, const float* __restrict__ fhat, uint8_t* __restrict__ out) {
  const int64_t nblocks = (n + EC_BLOCK - 1) / EC_BLOCK;
  uint8_t* payload = out + EC_HEADER + 8 * nblocks;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const EditRec r = e[i];
    uint8_t* p = payload + off[i];
    p += put_varint(p, rec_delta(e, i));
    p += put_varint(p, ((unsigned long long)r.q << 1) | r.lossless);
    if (r.lossless) {
      if (fhat) {
        put_varint(p, zz_rel(fhat[r.v], r.value));
      } else {
        const uint32_t b = __float_as_uint(r.value);
        p[0] = (uint8_t)b; p[1] = (uint8_t)(b >> 8); p[2] = (uint8_t)(b >> 16); p[3] = (uint8_t)(b >> 24);
      }
    }
    if (i % EC_BLOCK == 0) {
      const unsigned long long o = (unsigned long long)off[i];
      uint8_t* t = out + EC_HEADER + 8 * (i / EC_BLOCK);
      for (int k = 0; k < 8; k++) t[k] = (uint8_t)(o >> (8 * k));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint8_t* h = out;
    h[0] = 'D'; h[1] = 'M'; h[2] = 'T'; h[3] = 'E';
    const uint32_t ver = fhat ? 2u : 1u, blk = EC_BLOCK, nb32 = (uint32_t)nblocks, xib = __float_as_uint(xi);
    const uint32_t qm = (uint32_t)q_max;
    for (int k = 0; k < 4; k++) {
      h[4 + k] = (uint8_t)(ver >> (8 * k));
      h[16 + k] = (uint8_t)(blk >> (8 * k));
      h[20 + k] = (uint8_t)(qm >> (8 * k));
      h[24 + k] = (uint8_t)(xib >> (8 * k));
      h[28 + k] = (uint8_t)(nb32 >> (8 * k));
    }
    for (int k = 0; k < 8; k++) h[8 + k] = (uint8_t)((unsigned long long)n >> (8 * k));
  }
}

__device__ __forceinline__ unsigned long long get_varint(const uint8_t* __restrict__ p, size_t& pos, size_t end,
                                                         bool& ok) {
  unsigned long long x = 0;
  for (int sh = 0; sh < 64; sh += 7) {
    if (pos >= end) { ok = false; return 0; }
    const uint8_t b = p[pos++];
    x |= (unsigned long long)(b & 127u) << sh;
    if (!(b & 128u)) return x;
  }
  ok = false;
  return 0;
}

// One thread per block of EC_BLOCK records.
__global__ void k_ec_decode(const uint8_t* __restrict__ in, size_t nbytes, int64_t n, int64_t nblocks, int64_t N,
                            const float* __restrict__ fhat, EditRec* __restrict__ e, unsigned long long* __restrict__ bad) {
  const uint8_t* table = in + EC_HEADER;
  const uint8_t* payload = table + 8 * nblocks;
  const size_t plen = nbytes - EC_HEADER - 8 * (size_t)nblocks;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long o = 0, o1 = plen;
    for (int k = 0; k < 8; k++) o |= (unsigned long long)table[8 * b + k] << (8 * k);
    if (b + 1 < nblocks) {
      o1 = 0;
      for (int k = 0; k < 8; k++) o1 |= (unsigned long long)table[8 * (b + 1) + k] << (8 * k);
    }
    bool ok = o <= o1 && o1 <= plen;
    size_t pos = o;
    unsigned long long v = 0;
    const int64_t i0 = b * EC_BLOCK, i1 = i0 + EC_BLOCK < n ? i0 + EC_BLOCK : n;
    for (int64_t i = i0; i < i1 && ok; i++) {
      const unsigned long long d = get_varint(payload, pos, o1, ok);
      const unsigned long long code = get_varint(payload, pos, o1, ok);
      v = i == i0 ? d : v + d + 1ull;
      EditRec r;
      r.v = v;
      r.q = (unsigned short)(code >> 1);
      r.lossless = (unsigned char)(code & 1u);
      r.pad = 0;
      r.value = 0.f;
      if ((code >> 1) > 65535ull || v >= (unsigned long long)N) ok = false;
      if (r.lossless && ok) {
        if (fhat) {  // version 2: relative to fhat
          const unsigned long long z = get_varint(payload, pos, o1, ok);
          if (!ok || v >= (unsigned long long)N) { ok = false; break; }
          r.value = unzz_rel(fhat[v], z);
        } else {
          if (pos + 4 > o1) { ok = false; break; }
          const uint32_t bits = (uint32_t)payload[pos] | ((uint32_t)payload[pos + 1] << 8) |
                                ((uint32_t)payload[pos + 2] << 16) | ((uint32_t)payload[pos + 3] << 24);
          pos += 4;
          r.value = __uint_as_float(bits);
        }
      }
      e[i] = r;
    }
    if (ok && pos != o1) ok = false;  // a block's records end where the next block starts
    if (!ok) atomicAdd(bad, 1ull);
  }
}

// Version-2 decode, one WARP per block of EC_BLOCK records.  In version 2 every
// field is a varint, so the block's bytes split into varints without parsing (a
// byte with bit 7 clear ends one); only the role of each varint -- delta (0), code
// (1), zigzag value (2) -- follows from the sequence: 0 -> 1 -> (lossless ? 2 : 0),
// 2 -> 0.  Lane l owns the varints whose LAST byte lies in its 1/32 of the block's
// bytes.  Pass 1 runs the role machine over them from each of the 3 possible start
// roles (end role, records started, sum of delta + 1); the 32 results are chained
// in lane order; pass 2 re-walks with the known start role, record index and
// vertex (v = -1 + sum of delta + 1 over the block's records so far) and writes
// the fields of each record (a record's fields may be written by two lanes).
// Same checks as k_ec_decode: varints of <= 10 bytes, the block ends on a record
// boundary with exactly its record count, q <= 65535, v < N.
// Sequential byte reader of one lane: one aligned 16-byte load per 16 bytes instead of
// a load per byte.  A 16-byte aligned chunk that holds a valid byte never crosses a
// page.  (Tried: prefetching the next chunk, and gathering fhat for the lossless values
// in a separate record-parallel pass -- both slower, 3.7 -> 4.4 ms on C4.)
struct EcReader {
  uintptr_t cur = ~(uintptr_t)0;
  uint4 w;
  __device__ __forceinline__ uint32_t get(const uint8_t* p) {
    const uintptr_t a = (uintptr_t)p, c = a & ~(uintptr_t)15;
    if (c != cur) { w = __ldg((const uint4*)c); cur = c; }
    const uint32_t i = (uint32_t)(a & 15);
    const uint32_t word = i < 8 ? (i < 4 ? w.x : w.y) : (i < 12 ? w.z : w.w);
    return (word >> (8 * (i & 3))) & 255u;
  }
};

__device__ __forceinline__ bool ec_next_varint(EcReader& rd, const uint8_t* __restrict__ p, size_t pos, size_t end,
                                               unsigned long long& x, size_t& next, bool& ok) {
  x = 0;
  int nb = 0;
  while (pos < end) {
    const uint32_t by = rd.get(p + pos);
    pos++;
    if (nb < 10) x |= (unsigned long long)(by & 127u) << (7 * nb);
    nb++;
    if (!(by & 128u)) {
      next = pos;
      if (nb > 10) ok = false;
      return true;
    }
  }
  ok = false;  // runs past the block's end
  return false;
}

__global__ void __launch_bounds__(128) k_ec_decode_v2w(const uint8_t* __restrict__ in, size_t nbytes, int64_t n,
                                                       int64_t nblocks, int64_t N, const float* __restrict__ fhat,
                                                       EditRec* __restrict__ e, unsigned long long* __restrict__ bad) {
  const uint8_t* table = in + EC_HEADER;
  const uint8_t* payload = table + 8 * nblocks;
  const size_t plen = nbytes - EC_HEADER - 8 * (size_t)nblocks;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nblocks; b += nw) {
    unsigned long long o = 0, o1 = plen;
    if (lane == 0) {
      for (int k = 0; k < 8; k++) o |= (unsigned long long)__ldg(table + 8 * b + k) << (8 * k);
      if (b + 1 < nblocks) {
        o1 = 0;
        for (int k = 0; k < 8; k++) o1 |= (unsigned long long)__ldg(table + 8 * (b + 1) + k) << (8 * k);
      }
    }
    o = __shfl_sync(0xffffffffu, o, 0);
    o1 = __shfl_sync(0xffffffffu, o1, 0);
    const int64_t i0 = b * EC_BLOCK, nrec = n - i0 < EC_BLOCK ? n - i0 : EC_BLOCK;
    if (!(o <= o1 && o1 <= plen)) {  // warp-uniform
      if (lane == 0) atomicAdd(bad, 1ull);
      continue;
    }
    const size_t L = o1 - o, seg = (L + 31) / 32;
    const size_t s = o + ((size_t)lane * seg < L ? (size_t)lane * seg : L);
    const size_t t = o + ((size_t)(lane + 1) * seg < L ? (size_t)(lane + 1) * seg : L);
    bool ok = true;
    // first byte of the varint that contains byte s (it may start in the previous lane's bytes)
    size_t start = s;
    if (s < t) {
      int k = 0;
      while (start > o && (__ldg(payload + start - 1) & 128u)) {   // <= 10 bytes back
        start--;
        if (++k >= 10) { ok = false; break; }  // >= 11-byte varint
      }
    }
    // pass 1: role machine from the start roles 0, 1, 2
    int h0 = 0, h1 = 1, h2 = 2;
    uint32_t r0 = 0, r1 = 0, r2 = 0;
    unsigned long long S0 = 0, S1 = 0, S2 = 0;
    EcReader rd;
    for (size_t pos = start; ok && pos < t;) {
      unsigned long long x;
      size_t nx;
      if (!ec_next_varint(rd, payload, pos, o1, x, nx, ok)) break;
      if (nx - 1 >= t) break;  // ends in the next lane's bytes
      const int nxt1 = (x & 1ull) ? 2 : 0;
#define EC_STEP(h, r, S) \
  if (h == 0) { r++; S += x + 1ull; h = 1; } else if (h == 1) { h = nxt1; } else { h = 0; }
      EC_STEP(h0, r0, S0) EC_STEP(h1, r1, S1) EC_STEP(h2, r2, S2)
#undef EC_STEP
      pos = nx;
    }
    // chain the lanes in order (warp-uniform loop)
    int st = 0, my_st = 0;
    uint32_t rec = 0, my_rec = 0;
    unsigned long long vacc = 0, my_v = 0;
    for (int k = 0; k < 32; k++) {
      if (lane == k) { my_st = st; my_rec = rec; my_v = vacc; }
      const int hk = __shfl_sync(0xffffffffu, st == 0 ? h0 : (st == 1 ? h1 : h2), k);
      const uint32_t rk = __shfl_sync(0xffffffffu, st == 0 ? r0 : (st == 1 ? r1 : r2), k);
      const unsigned long long Sk = __shfl_sync(0xffffffffu, st == 0 ? S0 : (st == 1 ? S1 : S2), k);
      st = hk;
      rec += rk;
      vacc += Sk;
    }
    if (!__all_sync(0xffffffffu, ok) || st != 0 || (int64_t)rec != nrec) {  // warp-uniform
      if (lane == 0) atomicAdd(bad, 1ull);
      continue;
    }
    // pass 2: write the fields
    st = my_st;
    rec = my_rec;
    unsigned long long v = my_v - 1ull;  // vertex of the last record started before this lane's varints
    bool rok = true;
    for (size_t pos = start; pos < t;) {
      unsigned long long x;
      size_t nx;
      bool dummy = true;
      if (!ec_next_varint(rd, payload, pos, o1, x, nx, dummy)) break;
      if (nx - 1 >= t) break;
      EditRec* r = e + i0 + rec - (st == 0 ? 0 : 1);
      if (st == 0) {
        v += x + 1ull;
        r->v = v;
        rec++;
        st = 1;
        if (v >= (unsigned long long)N) rok = false;
      } else if (st == 1) {
        const unsigned long long q = x >> 1;
        const uint32_t ll = (uint32_t)(x & 1ull);
        if (q > 65535ull) rok = false;
        *(uint32_t*)((char*)r + 8) = (uint32_t)(q & 0xFFFFull) | (ll << 16);
        if (!ll) r->value = 0.f;
        st = ll ? 2 : 0;
      } else {
        if (v < (unsigned long long)N) r->value = unzz_rel(__ldg(fhat + v), x);
        st = 0;
      }
      pos = nx;
    }
    if (!__all_sync(0xffffffffu, rok) && lane == 0) atomicAdd(bad, 1ull);
  }
}

// Decompression side: g = fhat, then every edit: quantized -> RN(fhat - RN(q * step))
// (Eq. 2 replayed from fhat), lossless -> its stored bits.  For quantized
// entries the stored value is not read.  Out-of-range vertices count into *bad.
__global__ void k_apply_edits(const float* __restrict__ fhat, const EditRec* __restrict__ e, int64_t n, int64_t N,
                              float step, float* __restrict__ g, unsigned long long* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const EditRec r = e[i];
    if (r.v >= (unsigned long long)N) { atomicAdd(bad, 1ull); continue; }
    g[r.v] = r.lossless ? r.value : __fsub_rn(fhat[r.v], __fmul_rn((float)r.q, step));
  }
}

}  // namespace dmtz
