// dmtz_dist.cuh -- the multi-GPU C-loop inside the library.
//
// A world > 1 context holds one rank's z-slab: owned planes [z0, z1) and a local grid
// [lz0, lz1) with up to 3 halo planes per face (dmtz_local_slab).  dmtz_correct on it
// (correct_dist) runs the same synchronous rounds as the one-GPU loop:
//   once:      owned f / fhat -> the local arrays, halo planes of f and fhat from the
//              neighbours (transport exchange), setup on the local grid;
//   per round: the halo planes of g a neighbour changed in the last round (a face is
//              skipped when the reduction of the last round says no edit touched the
//              3 planes it covers), one round on the local grid (screen, classify the
//              cells anchored in [z0 - 2, z1 + 1), edit the owned targets), the round
//              counters + every rank's two face flags summed over the ranks; every
//              rank takes the same stop decision on the sums;
//   at the end: the owned edits (global vertex indices) and the owned planes of g.
// The transport is NCCL (libnccl.so.2 loaded at run time, a communicator per context)
// or caller callbacks (dmtz_ctx_set_transport; the tests use torch.distributed gloo).
#pragma once
#include <dlfcn.h>

#include <algorithm>
#include <nccl.h>  // types only: every NCCL call goes through the dlopen'ed table below

namespace dmtz {

inline dmtz_status local_slab(int64_t nz, int world, int rank, int64_t* z0, int64_t* z1, int64_t* lz0,
                              int64_t* lz1) {
  if (world < 1 || rank < 0 || rank >= world || nz < 3 * (int64_t)world) return DMTZ_E_ARG;
  const int64_t base = nz / world, extra = nz % world;
  const int64_t a = rank * base + (rank < extra ? rank : extra);
  const int64_t b = a + base + (rank < extra ? 1 : 0);
  *z0 = a;
  *z1 = b;
  *lz0 = a - 3 > 0 ? a - 3 : 0;
  *lz1 = b + 3 < nz ? b + 3 : nz;
  return DMTZ_OK;
}

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// NCCL is loaded on first use (the process's already-loaded libnccl.so.2 -- e.g.
// torch's -- is reused by the dynamic linker); NULL if it cannot be loaded
inline NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.h ? &api : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
#define DMTZ_SYM(n) api.n = (decltype(api.n))dlsym(h, "nccl" #n)
  DMTZ_SYM(GetUniqueId);
  DMTZ_SYM(CommInitRank);
  DMTZ_SYM(CommDestroy);
  DMTZ_SYM(GroupStart);
  DMTZ_SYM(GroupEnd);
  DMTZ_SYM(Send);
  DMTZ_SYM(Recv);
  DMTZ_SYM(AllReduce);
  DMTZ_SYM(GetErrorString);
#undef DMTZ_SYM
  if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.GroupStart || !api.GroupEnd || !api.Send ||
      !api.Recv || !api.AllReduce)
    return nullptr;
  api.h = h;
  return &api;
}

// the NCCL transport: user = the ncclComm_t
inline int nccl_exchange(void* user, int n, const int* peers, const void* const* send, const size_t* sb,
                         void* const* recv, const size_t* rb, dmtz_stream_t stream) {
  NcclApi* A = nccl_api();
  if (!A) return 1;
  ncclComm_t comm = (ncclComm_t)user;
  cudaStream_t s = (cudaStream_t)stream;
  if (A->GroupStart() != ncclSuccess) return 1;
  int bad = 0;
  for (int i = 0; i < n; i++) {
    if (sb[i]) bad |= A->Send(send[i], sb[i], ncclInt8, peers[i], comm, s) != ncclSuccess;
    if (rb[i]) bad |= A->Recv(recv[i], rb[i], ncclInt8, peers[i], comm, s) != ncclSuccess;
  }
  bad |= A->GroupEnd() != ncclSuccess;
  return bad;
}
inline int nccl_allreduce(void* user, int64_t* buf, int n, dmtz_stream_t stream) {
  NcclApi* A = nccl_api();
  if (!A) return 1;
  return A->AllReduce(buf, buf, (size_t)n, ncclInt64, ncclSum, (ncclComm_t)user, (cudaStream_t)stream) != ncclSuccess;
}

// The device control block of the batched mode (dmtz_ctx_set_dist_sync > 1): rounds are
// enqueued rounds_per_sync at a time with no host synchronisation between them; the stop
// rule runs on the device (k_dist_stop) on the all-reduced counters and sets HALT, after
// which every kernel of the remaining enqueued rounds returns at once (their unit lists
// stay empty, their halo updates and counters are no-ops).
enum : int {
  DCTL_HALT = 0,      // 1 once the stop rule fired
  DCTL_STATUS = 1,    // its dmtz_status
  DCTL_ROUND = 2,     // the round running (device count; frozen at the stop)
  DCTL_ROUNDS = 3,    // dmtz_stats.rounds
  DCTL_FALSE0 = 4,    // n_false_round0, kinds at 5 .. 12
  DCTL_GATE_LO = 13,  // the lower neighbour changed its upper face planes last round
  DCTL_GATE_HI = 14,  // the upper neighbour changed its lower face planes last round
  DCTL_SWEEPS = 15,
  DCTL_N = 16
};

// start of a batched round: the device round count and the loop state's round
__global__ void k_dist_begin(long long* __restrict__ ctl, LoopState* __restrict__ ls) {
  if (threadIdx.x == 0 && !ctl[DCTL_HALT]) ls->round = (unsigned long long)++ctl[DCTL_ROUND];
}

// the stop rule (as dist_stop below) on the summed counters, on the device; also the
// halo gates of the next round from the neighbours' face flags
__global__ void k_dist_stop(const long long* __restrict__ tot, long long* __restrict__ ctl, long long max_rounds,
                            int rank, int world) {
  if (threadIdx.x != 0 || ctl[DCTL_HALT]) return;
  const long long r = ctl[DCTL_ROUND];
  ctl[DCTL_SWEEPS]++;
  if (r == 1) {
    ctl[DCTL_FALSE0] = tot[0];
    for (int k = 0; k < 8; k++) ctl[DCTL_FALSE0 + 1 + k] = tot[4 + k];
  }
  long long st = -1;
  if (tot[3]) st = DMTZ_E_INTERNAL;
  else if (tot[0] == 0) st = DMTZ_OK;
  else if (tot[1] == 0) st = DMTZ_E_STUCK;
  else if (r == max_rounds) st = DMTZ_E_ITER_CAP;
  if (st != DMTZ_OK) ctl[DCTL_ROUNDS] = r;  // rounds that found false cells
  if (st >= 0) {
    ctl[DCTL_STATUS] = st;
    ctl[DCTL_HALT] = 1;
  }
  ctl[DCTL_GATE_LO] = rank > 0 ? tot[13 + 2 * (rank - 1)] : 0;
  ctl[DCTL_GATE_HI] = rank < world - 1 ? tot[12 + 2 * (rank + 1)] : 0;
}

// round counters for the distributed reduction: out[0..11] as k_counters_out, then two
// face flags per rank at 12 + 2 rank (+1): "an owned vertex of the 3 planes next to the
// lower (upper) face changed this round" -- from the round's change bitmap, whose rows
// of those planes are cleared before the round (k_face_clear)
// the face flags of the round: any changed vertex in the rows of planes [lo0, lo1) /
// [hi0, hi1) of the change bitmap, OR-ed into flags[0] / flags[1] (zeroed by the
// counters kernel after it reads them); a grid of blocks, one atomic per warp that saw one
__global__ void k_face_flags(const uint32_t* __restrict__ vround, int64_t per_plane, int64_t lo0, int64_t lo1,
                             int64_t hi0, int64_t hi1, unsigned* __restrict__ flags, const long long* ctl) {
  if (ctl && ctl[DCTL_HALT]) return;
  const int lane = threadIdx.x & 31;
  for (int f = 0; f < 2; f++) {
    const int64_t a = (f ? hi0 : lo0) * per_plane, b = (f ? hi1 : lo1) * per_plane;
    for (int64_t base = a + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane; base < b;
         base += (int64_t)gridDim.x * blockDim.x) {
      const unsigned w = base + lane < b ? vround[base + lane] : 0u;
      if (__any_sync(0xffffffffu, w != 0u) && lane == 0) atomicOr(flags + f, 1u);
    }
  }
}

// (ctl: the device stop flag of the batched mode -- once set, this writes zeros)
__global__ void k_dist_counters(const Counters* __restrict__ cnt, long long round, long long* __restrict__ out,
                                int nout, unsigned* __restrict__ flags, int rank, const long long* ctl) {
  if (ctl && ctl[DCTL_HALT]) {
    for (int i = threadIdx.x; i < nout; i += blockDim.x) out[i] = 0;
    return;
  }
  __shared__ unsigned s_flag[2];
  if (threadIdx.x < 2) s_flag[threadIdx.x] = flags[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 2) flags[threadIdx.x] = 0u;
  for (int i = threadIdx.x; i < nout; i += blockDim.x) {
    long long v = 0;
    if (i == 0) v = (long long)cnt->n_false;
    else if (i == 1) v = (long long)cnt->n_changed;
    else if (i == 2) v = (long long)cnt->n_targets;
    else if (i == 3) v = (long long)cnt->n_internal;
    else if (i < 12) v = round == 1 ? (long long)cnt->kinds[i - 4] : 0ll;
    else if (i == 12 + 2 * rank) v = (long long)s_flag[0];
    else if (i == 13 + 2 * rank) v = (long long)s_flag[1];
    out[i] = v;
  }
}

// one-time / per-round halo exchange with the neighbours: my owned boundary planes of
// `arr` (those the peer keeps as halo) out, the peer's into my halo planes (staged in
// `recv` when `stage`, else received in place).  faces: bit 0 = lower, bit 1 = upper.
struct HaloPlan {
  int n = 0;
  int peers[2];
  const void* send[2];
  size_t sbytes[2];
  void* recv[2];
  size_t rbytes[2];
  int64_t rz0[2], rz1[2];  // local planes received
};

inline HaloPlan halo_plan(const dmtz_ctx* c, const Grid& g, const float* arr, float* dst, int lower_send,
                          int lower_recv, int upper_send, int upper_recv) {
  HaloPlan h;
  const int64_t oz0 = c->z0 - c->lz0, oz1 = c->z1 - c->lz0;  // owned, local
  const size_t plane = (size_t)g.sz * sizeof(float);
  if (c->rank > 0) {  // lower neighbour: it keeps my planes [z0, z0 + nb) as its upper halo
    const int64_t nb = oz0;                   // my lower halo planes = its planes below z0
    const int64_t ns = std::min<int64_t>(3, oz1 - oz0);  // planes it keeps from me
    h.peers[h.n] = c->rank - 1;
    h.send[h.n] = arr + oz0 * g.sz;
    h.sbytes[h.n] = lower_send ? (size_t)ns * plane : 0;
    h.recv[h.n] = dst;                        // local planes [0, oz0)
    h.rbytes[h.n] = lower_recv ? (size_t)nb * plane : 0;
    h.rz0[h.n] = 0;
    h.rz1[h.n] = lower_recv ? nb : 0;
    h.n++;
  }
  if (c->rank < c->world - 1) {
    const int64_t na = g.nz - oz1;            // my upper halo planes
    const int64_t ns = std::min<int64_t>(3, oz1 - oz0);
    h.peers[h.n] = c->rank + 1;
    h.send[h.n] = arr + (oz1 - ns) * g.sz;
    h.sbytes[h.n] = upper_send ? (size_t)ns * plane : 0;
    h.recv[h.n] = dst + oz1 * g.sz;           // relative to dst's plane 0
    h.rbytes[h.n] = upper_recv ? (size_t)na * plane : 0;
    h.rz0[h.n] = oz1;
    h.rz1[h.n] = upper_recv ? g.nz : oz1;
    h.n++;
  }
  return h;
}

inline int run_exchange(dmtz_ctx* c, HaloPlan& h, cudaStream_t s) {
  int n = 0;
  for (int i = 0; i < h.n; i++) n += (h.sbytes[i] || h.rbytes[i]) ? 1 : 0;
  if (!n) return 0;
  return c->tr.exchange(c->tr.user, h.n, h.peers, h.send, h.sbytes, h.recv, h.rbytes, (dmtz_stream_t)s);
}

// the stop rule of dmtz_correct on the summed counters (k_loop_check)
inline int dist_stop(int64_t round, const long long* t, int64_t max_rounds) {
  if (t[3]) return DMTZ_E_INTERNAL;
  if (t[0] == 0) return DMTZ_OK;
  if (t[1] == 0) return DMTZ_E_STUCK;
  if (round == max_rounds) return DMTZ_E_ITER_CAP;
  return -1;
}

}  // namespace dmtz
