// dmtz_metrics.cuh -- evaluation metrics of §5.1:
// critical-cell and separatrix recall / precision between the original and the
// edited (or decompressed) field, as match counts on the device.
//   critical: a cell matches when it is critical in both (same anchor, same type);
//   separatrix: the unit is one branch, identified by (kind, origin cell, its
//   ordinal among that origin's branches); it matches when the other trace has the
//   branch with that identity and the same terminal and cell sequence.
#pragma once

#include "dmtz_kernels.cuh"

namespace dmtz {

// out[0] += critical cells in a, out[1] += in b, out[2] += in both
__global__ void k_crit_prf(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, int64_t n,
                           unsigned long long* __restrict__ out) {
  unsigned long long na = 0, nb = 0, nm = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = a[i], y = b[i];
    na += __popc(x);
    nb += __popc(y);
    nm += __popc(x & y);
  }
  warp_add(out + 0, na);
  warp_add(out + 1, nb);
  warp_add(out + 2, nm);
}

// first index in [0, n) whose (kind, origin) is not below (k, o); lists are sorted by (kind, origin)
__device__ __forceinline__ int64_t lower_bound_ko(const uint8_t* __restrict__ kind, const uint64_t* __restrict__ origin,
                                                  int64_t n, int k, uint64_t o) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int km = kind[mid];
    const bool below = km < k || (km == k && origin[mid] < o);
    if (below) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// out[0] += branches of a that have an identical branch in b (one thread per branch of a)
__global__ void k_sep_match(const long long* __restrict__ aoff, const uint64_t* __restrict__ acells,
                            const uint64_t* __restrict__ aorigin, const uint64_t* __restrict__ aterm,
                            const uint8_t* __restrict__ akind, int64_t na, const long long* __restrict__ boff,
                            const uint64_t* __restrict__ bcells, const uint64_t* __restrict__ borigin,
                            const uint64_t* __restrict__ bterm, const uint8_t* __restrict__ bkind, int64_t nb,
                            unsigned long long* __restrict__ out) {
  unsigned long long nm = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = akind[i];
    const uint64_t o = aorigin[i];
    const int64_t ord = i - lower_bound_ko(akind, aorigin, na, k, o);
    const int64_t j = lower_bound_ko(bkind, borigin, nb, k, o) + ord;
    if (j >= nb || bkind[j] != k || borigin[j] != o || bterm[j] != aterm[i]) continue;
    const int64_t a0 = aoff[i], a1 = aoff[i + 1], b0 = boff[j], b1 = boff[j + 1];
    if (a1 - a0 != b1 - b0) continue;
    bool same = true;
    for (int64_t t = 0; t < a1 - a0 && same; t++) same = acells[a0 + t] == bcells[b0 + t];
    nm += same ? 1 : 0;
  }
  warp_add(out, nm);
}

}  // namespace dmtz
