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
// Blocks make the decoder parallel (one thread per block); the encoder is a
// per-edit length pass, an exclusive scan and a per-edit write.
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
