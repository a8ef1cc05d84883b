// dmtz_trace.cuh -- V-path separatrix traces (a9-a11), see include/dmtz.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dmtz_kernels.cuh"

namespace dmtz {

struct TraceArgs {
  Grid g;
  const void* codes;
  uint32_t kinds;
  char* scratch;
  Counters* cnt;
  Counters* host_cnt;
  int64_t* out_offsets;
  uint64_t* out_cells;
  uint64_t* out_origin;
  uint64_t* out_terminal;
  uint8_t* out_kind;
  int64_t cap_b, cap_c;
  int64_t n_branches = 0, n_cells = 0, n_internal = 0;
};

inline size_t trace_scratch_bytes(const Grid&, int) { return 0; }

template <int D>
cudaError_t run_trace(TraceArgs&, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace dmtz
