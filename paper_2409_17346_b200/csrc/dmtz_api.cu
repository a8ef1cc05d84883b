// dmtz_api.cu -- the C ABI of include/dmtz.h on top of dmtz_kernels.cuh.
//
// Host side of the hot path: workspace carving, the fixed-point driver of the
// C-loop (repeat gradient -> classify -> fix until no false
// critical cell), status/error plumbing.  No device allocation happens here:
// every buffer is the caller's.
#include <chrono>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <algorithm>
#include <vector>
#include <utility>

#include "../../include/dmtz.h"
#include "dmtz_kernels.cuh"
#include "dmtz_sweep.cuh"
#include "dmtz_trace.cuh"
#include "dmtz_sloop.cuh"
#include "dmtz_codec.cuh"
#include "dmtz_metrics.cuh"

using namespace dmtz;

// The CUDA graph of the round loop: a conditional WHILE node whose body is one
// captured round (enqueue_round); k_loop_check sets the condition on the device.
struct LoopGraph {
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  // key: everything the captured body depends on
  const void *f = nullptr, *fhat = nullptr, *g = nullptr, *ws = nullptr, *sdirty = nullptr;
  float xi = 0.f;
  int q_max = -1, q_cap = -1, tier = -1, frontier = -1;
  long long max_rounds = -1;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
  }
};

struct dmtz_ctx {
  dmtz_dims dims;
  Grid g;
  int D;
  int device;
  int rank, world;
  Counters* host_cnt = nullptr;  // pinned
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // sweep timing (opts.profile): screen | decode | edit
  int verbose;         // DMTZ_VERBOSE=1: per-round counters on stderr (host-driven rounds)
  int no_graph;        // DMTZ_NO_GRAPH=1: host-driven rounds instead of the CUDA-graph loop
  cudaStream_t aux_stream = nullptr;   // dmtz_correct_host: f's gradient while fhat is uploaded
  cudaEvent_t ev_aux[2] = {nullptr, nullptr};
  int pre_codes = 0;   // set by dmtz_correct_host: f's codes / crit / lowest vertex already enqueued on aux_stream
  int no_keys;         // DMTZ_NO_KEYS=1: k_screen always uses the compare/select form of the gradient
  int no_tile;         // DMTZ_SCREEN_TILE=0: no shared-memory tile in k_screen's dense path
  LoopState* host_ls = nullptr;  // pinned
  struct LoopGraph* graph = nullptr;
  cudaStream_t cap_stream = nullptr;  // private stream the loop body is captured on (the caller's may be the legacy stream)
  uint32_t* sdirty = nullptr;  // dmtz_preserve: per-anchor "code changed since the last S-round" bits
  // multi-GPU (dist): this rank's z-slab of the global grid (g above is the LOCAL grid)
  int dist = 0;
  int64_t gnz = 0, z0 = 0, z1 = 0, lz0 = 0, lz1 = 0;
  dmtz_transport tr = {nullptr, nullptr, nullptr};
  int has_tr = 0;
  void* nccl_comm = nullptr;
  int dist_sync = 8;         // rounds per host check of the device stop flag (1: host-synchronous rounds)
  int dist_graph = 0;        // dmtz_ctx_set_dist_graph: batches as a captured CUDA graph (NCCL transport)
  int dist_graph_used = 0;   // the last dmtz_correct ran its batches from the graph
  int t3_log = 0;            // DMTZ_T3_LOG=1: per S-round candidate counts and phase times of tier 3 on stderr
  int t3_unordered = 1;      // tier-3 candidate traces fill connectors in any order (DMTZ_T3_ORDERED=1: FIFO)
};

#include "dmtz_dist.cuh"  // needs the context above

// Every entry point runs on the context's device and restores the caller's current
// device on return (the caller's thread may have another device current).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const dmtz_ctx* c) {
    if (c && cudaGetDevice(&prev) == cudaSuccess && prev != c->device) cudaSetDevice(c->device);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

namespace {

thread_local char g_err[512] = "";
thread_local int64_t g_trace_levels[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};

void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      set_err("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));       \
      return DMTZ_E_CUDA;                                                               \
    }                                                                                   \
  } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Workspace layout (offsets from the base, each 256-B aligned)
struct Layout {
  size_t cand_f, cand_g, crit_f, crit_g, lowpos, lb, state, tcache, ncache, tbits, counters, edit_bc, ebits, fmark, vchg, units,
      units2, frontier, keyinfo, dist, trace, total;
  int64_t fwords;  // frontier bitmap words (one bit per row-block unit)
};

Layout layout_for(const dmtz_ctx* c) {
  const size_t N = (size_t)c->g.N;
  const size_t cs = c->D == 3 ? 8 : 2;
  Layout L;
  size_t o = 0;
  // u64 even in 2D: the trace reuses it as int64 scratch (>= 1 MiB for small grids)
  L.cand_g = o; o += align_up(N * 8 > (size_t)(1 << 20) ? N * 8 : (size_t)(1 << 20));
  L.crit_g = o; o += align_up(N * 4);
  // [cand_f, tbits] is the trace's connector-BFS scratch (lowpos: at least 128 slots of 3 x 1024 words)
  L.cand_f = o; o += align_up(N * cs);
  L.crit_f = o; o += align_up(N * 4);
  L.lowpos = o; o += align_up(N * 8 > (size_t)128 * 3072 * 8 ? N * 8 : (size_t)128 * 3072 * 8);
  L.lb = o; o += align_up(N * 4);
  L.state = o; o += align_up(N * 4);
  L.tcache = o; o += align_up(N * 8);  // per anchor: target offsets of its false cells (last evaluation)
  L.ncache = o; o += align_up(N);      // per anchor: number of those false cells
  L.tbits = o; o += align_up((size_t)(c->g.nz * c->g.ny * ((c->g.nx + 31) / 32)) * 4 + 64);  // row-padded
  L.counters = o; o += align_up(sizeof(Counters) * 2);
  // edit-list block counts, and the trace's scan state over <= 64 N branch offsets
  L.edit_bc = o; o += align_up((64 * (N + EDIT_CHUNK - 1) / EDIT_CHUNK + 2) * 8);
  const RowGeom rg = row_geom(c->g);
  L.fwords = (rg.units + 31) / 32;
  L.ebits = o; o += align_up((size_t)(c->g.nz * c->g.ny * rg.wpr) * 4 + 64);
  L.fmark = o; o += align_up((size_t)(c->g.nz * c->g.ny * rg.wpr) * 4 + 64);
  L.vchg = o; o += align_up(2 * (size_t)(c->g.nz * c->g.ny * rg.wpr) * 4 + 64);
  L.units = o; o += align_up((size_t)rg.units * 4);
  L.units2 = o; o += align_up((size_t)rg.units * 4);
  L.frontier = o; o += align_up(L.fwords * 4 + 64);
  L.keyinfo = o; o += align_up(sizeof(KeyInfo));
  L.dist = 0;
  if (c->dist) {  // local f, fhat, g, halo staging (f32 each) + the reduced counters
    L.dist = o;
    o += align_up(4 * N * sizeof(float) + (size_t)(64 + DCTL_N + 1) * 8);   // + the 2 face flags
  }
  L.trace = o; o += align_up(trace_scratch_bytes(c->g, c->D));
  L.total = o;
  return L;
}

dim3 anchor_grid(const Grid& g, int64_t z0, int64_t z1, int threads) {
  int64_t bx = (g.nx + threads - 1) / threads;
  int64_t by = g.ny < 65535 ? g.ny : 65535;
  int64_t nzr = z1 - z0;
  int64_t bz = nzr < 65535 ? nzr : 65535;
  if (bz < 1) bz = 1;
  return dim3((unsigned)(bx < 2147483647 ? bx : 2147483647), (unsigned)by, (unsigned)bz);
}

template <int D>
void launch_codes(const Grid& g, const float* fld, void* codes, int64_t z0, int64_t z1, cudaStream_t s) {
  if (z1 <= z0) return;
  k_codes<D><<<anchor_grid(g, z0, z1, 128), 128, 0, s>>>(fld, (typename Tr<D>::code_t*)codes, g, z0, z1);
}

template <int D>
uint32_t tier_mask(int tier) {
  if (tier >= 2) return 0xFFFFFFFFu;  // tiers 3-4 build on tier 2
  // dims 0 and top only
  return D == 3 ? (1u | (0x3Fu << 20)) : (1u | (0x3u << 4));
}

// Device views of the workspace
template <int D>
struct WS {
  using code_t = typename Tr<D>::code_t;
  code_t* cand_f;
  code_t* cand_g;            // codes of g, memoized across rounds
  uint32_t *crit_f, *crit_g, *state, *tbits, *ebits, *fmark, *vchg, *units, *units2, *fbits;
  int64_t vwords;
  unsigned long long* lowpos;
  unsigned long long* tcache;
  uint8_t* ncache;
  float* lb;
  Counters* dc;
  KeyInfo* ki;               // value range of the call (key form of the gradient)
  LoopState* ls;             // second 256 B block of the counters region
  unsigned long long* bc;
  size_t rowbit_bytes;
  WS(char* ws, const Layout& L, const Grid& g) {
    cand_f = (code_t*)(ws + L.cand_f);
    cand_g = (code_t*)(ws + L.cand_g);
    crit_f = (uint32_t*)(ws + L.crit_f);
    crit_g = (uint32_t*)(ws + L.crit_g);
    lowpos = (unsigned long long*)(ws + L.lowpos);
    lb = (float*)(ws + L.lb);
    tcache = (unsigned long long*)(ws + L.tcache);
    ncache = (uint8_t*)(ws + L.ncache);
    state = (uint32_t*)(ws + L.state);
    tbits = (uint32_t*)(ws + L.tbits);
    dc = (Counters*)(ws + L.counters);
    ki = (KeyInfo*)(ws + L.keyinfo);
    ls = (LoopState*)(ws + L.counters + sizeof(Counters));
    bc = (unsigned long long*)(ws + L.edit_bc);
    ebits = (uint32_t*)(ws + L.ebits);
    fmark = (uint32_t*)(ws + L.fmark);
    vchg = (uint32_t*)(ws + L.vchg);
    units = (uint32_t*)(ws + L.units);
    units2 = (uint32_t*)(ws + L.units2);
    fbits = (uint32_t*)(ws + L.frontier);
    const RowGeom rg = row_geom(g);
    rowbit_bytes = (size_t)(g.nz * g.ny * rg.wpr) * 4;
    vwords = g.nz * g.ny * rg.wpr;
  }
};

inline int clamp_blocks(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t b = (n + threads - 1) / threads;
  return (int)(b < 1 ? 1 : b < cap ? b : cap);
}

// a2: codes, critical masks and f-lowest vertices of f (reads f only)
template <int D>
void enqueue_f_codes(const Grid& g, const float* f, WS<D>& W, cudaStream_t s) {
  launch_codes<D>(g, f, W.cand_f, 0, g.nz, s);
  k_critmask<D><<<anchor_grid(g, 0, g.nz, 128), 128, 0, s>>>(W.cand_f, W.crit_f, g);
  k_lowpos<D><<<anchor_grid(g, 0, g.nz, 128), 128, 0, s>>>(f, W.lowpos, g);
}

// a1 + a2: validate, lb, g = fhat, state = 0, codes / criticality / lowest vertex of f.
// Error messages report vertex index + v_report_off (the global index in slab mode).
template <int D>
dmtz_status setup_phase(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o, WS<D>& W,
                        float* g_out, int64_t v_report_off, int64_t* launches, cudaStream_t s) {
  const Grid& g = c->g;
  Counters* hc = c->host_cnt;
  const int64_t nwords = (int64_t)(W.rowbit_bytes / 4);
  CK(cudaMemsetAsync(W.dc, 0, sizeof(Counters), s));
  CK(cudaMemsetAsync(&W.dc->first_nonfinite, 0xFF, 16, s));
  CK(cudaMemsetAsync(W.tbits, 0, nwords * 4, s));
  CK(cudaMemsetAsync(W.fmark, 0, W.rowbit_bytes, s));
  CK(cudaMemsetAsync(W.vchg, 0, 2 * W.rowbit_bytes, s));
  CK(cudaMemsetAsync(W.ki, 0, sizeof(KeyInfo), s));
  CK(cudaMemsetAsync(&W.ki->min_bits, 0x7F, 4, s));
  k_setup<<<clamp_blocks(g.N, 256), 256, 0, s>>>(f, fhat, o->xi, g.N, W.lb, g_out, W.state, W.dc, W.ki);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hc, W.dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hc->first_nonfinite != ~0ull) {
    set_err("non-finite value at vertex %llu", hc->first_nonfinite + (unsigned long long)v_report_off);
    return DMTZ_E_NONFINITE;
  }
  if (hc->first_bound != ~0ull) {
    set_err("|fhat - f| > xi at vertex %llu", hc->first_bound + (unsigned long long)v_report_off);
    return DMTZ_E_BOUND;
  }
  if (c->pre_codes) {  // enqueued by dmtz_correct_host on the aux stream (overlapping the fhat upload)
    CK(cudaStreamWaitEvent(s, c->ev_aux[1], 0));
    *launches += 4;
    return DMTZ_OK;
  }
  enqueue_f_codes<D>(g, f, W, s);
  CK(cudaGetLastError());
  *launches += 4;
  return DMTZ_OK;
}

// unit list of the z-planes [z0, z1) into `list` (count -> *n)
inline cudaError_t units_range(const RowGeom& rg, int64_t z0, int64_t z1, uint32_t* list, unsigned long long* n,
                               cudaStream_t s, const long long* halt = nullptr) {
  const int64_t cnt = (z1 - z0) * rg.ub;
  k_units_all<<<clamp_blocks(cnt > 0 ? cnt : 1, 256, 4096), 256, 0, s>>>(rg.ub, z0, z1, list, n, halt);
  return cudaGetLastError();
}

// Enqueue one C-loop round (a3-a6, + a7 frontier when fbits != nullptr) and the
// loop check; no host synchronisation, so the same sequence is captured into the
// body of the CUDA-graph WHILE node.  The screen runs over `units`/`n_units`, the
// decode over `dunits`/`n_dunits`; targets outside [own_lo, own_hi) are dropped
// and only anchors in planes [count_z0, count_z1) are counted (slab mode).
// slab mode: classified planes, false-cell unit marks, unit list built by the caller
struct RoundExtra {
  int64_t anchor_z0 = 0, anchor_z1 = INT64_MAX;
  uint32_t* decode_marks = nullptr;
  bool list_after = true;
};

template <int D>
dmtz_status enqueue_round(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o, WS<D>& W,
                          float* g_out, const uint32_t* units, unsigned long long* n_units, const uint32_t* dunits,
                          unsigned long long* n_dunits, uint32_t* fbits, int fwords, int64_t own_z0, int64_t own_z1,
                          int64_t count_z0, int64_t count_z1, bool profile, unsigned long long max_rounds,
                          cudaGraphConditionalHandle h, int use_cond, int use_skip, int64_t* launches,
                          cudaStream_t s, const RoundExtra& X = RoundExtra()) {
  const Grid& g = c->g;
  const RowGeom rg = row_geom(g);
  const int64_t nwords = (int64_t)(W.rowbit_bytes / 4);  // row-padded target bitmap
  // grids sized by the largest possible work list (small grids: few blocks, cheap launches)
  const int64_t max_items = rg.units * UY * ((rg.wpr + CG - 1) / CG);
  const int sweep_blocks = (int)(max_items / 8 + 1 < 148 * 8 ? max_items / 8 + 1 : 148 * 8);
  const float step = ldexpf(o->xi, -o->q_max);  // xi / 2^q_max, exact
  const int fwords_smem = fbits && fwords * 4 <= 32768 ? fwords : 0;
  if (!use_cond) CK(cudaMemsetAsync(W.dc, 0, offsetof(Counters, first_nonfinite), s));  // else: k_loop_check
  if (!use_cond && c->verbose) CK(cudaMemsetAsync(&W.dc->pad[2], 0, 4 * 8, s));
  if (fbits) CK(cudaMemsetAsync(W.ebits, 0, W.rowbit_bytes, s));  // rewritten for every active unit
  if (profile) CK(cudaEventRecord(c->ev[0], s));
  const int skeys = c->no_keys ? 0 : (c->no_tile ? 1 : 3);   // the tile's smem attribute: dmtz_ctx_create
  if (use_skip)
    k_screen<D, true><<<sweep_blocks, SCREEN_THREADS, (skeys & 2) ? SCREEN_TILE_BYTES : 0, s>>>(
        g_out, W.cand_g, W.ebits, W.vchg, W.vwords, use_skip, units, n_units, g, rg, W.ls, W.dc, W.ki, skeys, 32u);
  else
    k_screen<D, false><<<sweep_blocks, SCREEN_THREADS, (skeys & 2) ? SCREEN_TILE_BYTES : 0, s>>>(
        g_out, W.cand_g, W.ebits, W.vchg, W.vwords, use_skip, units, n_units, g, rg, W.ls, W.dc, W.ki, skeys, 32u);
  if (c->sdirty) {  // dmtz_preserve: accumulate the changed codes for the next S-round
    k_sdirty_or<<<clamp_blocks(nwords, 256), 256, 0, s>>>(W.ebits, nwords, g, rg, c->sdirty);
    *launches += 1;
  }
  if (profile) CK(cudaEventRecord(c->ev[1], s));
  k_decode<D><<<sweep_blocks * 2, DECODE_THREADS, 0, s>>>(
      f, W.cand_f, W.crit_f, W.cand_g, W.ebits, W.fmark, W.tbits, dunits, n_dunits, g, rg,
      tier_mask<D>(o->tier), W.lowpos, W.tcache, W.ncache, W.ls, own_z0, own_z1, count_z0, count_z1, X.anchor_z0,
      X.anchor_z1, X.decode_marks, W.dc);
  if (profile) CK(cudaEventRecord(c->ev[2], s));
  k_edit_rows<D><<<clamp_blocks(nwords, 256), 256, fwords_smem * 4, s>>>(
      W.tbits, nwords, fhat, W.lb, g_out, W.state, W.dc, step, o->q_cap, fbits, g, rg, fwords_smem,
      (use_skip || fbits) ? W.vchg : nullptr, W.vwords, W.ls, FastDiv((uint32_t)rg.wpr), FastDiv((uint32_t)g.ny));
  if (profile) CK(cudaEventRecord(c->ev[3], s));
  k_loop_check<<<1, 32, 0, s>>>(W.dc, W.ls, max_rounds, h, use_cond, fbits && X.list_after ? n_units : nullptr);
  *launches += 4;
  if (fbits && X.list_after) {
    // next round's unit list (after the check read this round's counters); clears fbits
    if (!use_cond) CK(cudaMemsetAsync(n_units, 0, 8, s));
    k_units_from_bits<<<clamp_blocks(rg.units, 256, 4096), 256, 0, s>>>(fbits, rg.units, (uint32_t*)units, n_units);
    *launches += 1;
  }
  CK(cudaGetLastError());
  return DMTZ_OK;
}

// One round with a host synchronisation: counters -> c->host_cnt, loop state -> *hls
template <int D>
dmtz_status round_phase(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o, WS<D>& W,
                        float* g_out, const uint32_t* units, unsigned long long* n_units, const uint32_t* dunits,
                        unsigned long long* n_dunits, uint32_t* fbits, int fwords, int64_t own_z0, int64_t own_z1,
                        int64_t count_z0, int64_t count_z1, bool profile, unsigned long long max_rounds,
                        int use_skip, LoopState* hls, int64_t* launches, cudaStream_t s,
                        const RoundExtra& X = RoundExtra()) {
  dmtz_status st = enqueue_round<D>(c, f, fhat, o, W, g_out, units, n_units, dunits, n_dunits, fbits, fwords, own_z0,
                                    own_z1, count_z0, count_z1, profile, max_rounds, cudaGraphConditionalHandle(), 0,
                                    use_skip, launches, s, X);
  if (st) return st;
  CK(cudaMemcpyAsync(c->host_cnt, W.dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hls, W.ls, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return DMTZ_OK;
}

// a8: ordered edit list of the vertices [v0, v1), indices shifted by v_off
template <int D>
dmtz_status edits_phase(dmtz_ctx* c, WS<D>& W, const float* g_out, int64_t v0, int64_t v1, int64_t v_off,
                        dmtz_edit* edits, int64_t cap, int64_t* n_edits, int64_t* n_lossless, int64_t* launches,
                        cudaStream_t s) {
  Counters* hc = c->host_cnt;
  const int64_t nb = (v1 - v0 + EDIT_CHUNK - 1) / EDIT_CHUNK;
  CK(cudaMemsetAsync(&W.dc->n_lossless, 0, 8, s));
  if (nb > 0) {
    k_edit_count<<<(unsigned)nb, EDIT_THREADS, 0, s>>>(W.state, v0, v1, W.bc, W.dc);
    k_scan_counts<<<1, EDIT_THREADS, 0, s>>>(W.bc, nb, W.dc);
    k_edit_write<<<(unsigned)nb, EDIT_THREADS, 0, s>>>(W.state, g_out, v0, v1, W.bc, (EditOut*)edits, cap, v_off);
    *launches += 3;
  } else {
    CK(cudaMemsetAsync(&W.dc->n_edits, 0, 8, s));
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hc, W.dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *n_edits = (int64_t)hc->n_edits;
  *n_lossless = (int64_t)hc->n_lossless;
  return DMTZ_OK;
}

template <int D>
dmtz_status build_loop_graph(dmtz_ctx* c, LoopGraph& G, const float* f, const float* fhat,
                             const dmtz_correct_opts* o, WS<D>& W, float* g_out, char* ws, const Layout& L,
                             unsigned long long max_rounds, bool frontier_mode, cudaStream_t s) {
  G.reset();
  CK(cudaGraphCreate(&G.graph, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, G.graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, G.graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  (void)s;
  cudaStream_t cs = c->cap_stream;
  CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int64_t launches = 0;
  dmtz_status st = enqueue_round<D>(c, f, fhat, o, W, g_out, W.units, &W.dc->n_units, W.units, &W.dc->n_units,
                                    frontier_mode ? W.fbits : nullptr, (int)L.fwords, 0, c->g.nz, 0, c->g.nz, false,
                                    max_rounds, h, 1, frontier_mode ? 1 : 0, &launches, cs);
  cudaGraph_t captured;
  cudaError_t e = cudaStreamEndCapture(cs, &captured);
  if (st) return st;
  CK(e);
  CK(cudaGraphInstantiate(&G.exec, G.graph, 0));
  G.f = f; G.fhat = fhat; G.g = g_out; G.ws = ws; G.xi = o->xi; G.q_max = o->q_max; G.q_cap = o->q_cap;
  G.tier = o->tier; G.frontier = frontier_mode; G.max_rounds = (long long)max_rounds; G.sdirty = c->sdirty;
  return DMTZ_OK;
}

// Run C-loop rounds (a3-a7) until the loop check stops them.  first: start a new
// loop (round 1 over every unit); else resume at the round and unit list the caller
// prepared (after an S-round).  On return hls holds the loop state.
template <int D>
dmtz_status run_cloop(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o, WS<D>& W,
                      char* ws, const Layout& L, float* g_out, unsigned long long max_rounds, bool first,
                      dmtz_stats* st, cudaStream_t s) {
  const Grid& g = c->g;
  Counters* hc = c->host_cnt;
  LoopState* hls = c->host_ls;
  const RowGeom rg = row_geom(g);
  unsigned long long* n_units = &W.dc->n_units;
  const bool frontier_mode = !o->full_sweeps;
  dmtz_status status = DMTZ_OK;
  if (first) {
    // round 1 (and every round of a full sweep) processes every unit
    CK(units_range(rg, 0, g.nz, W.units, n_units, s));
    CK(cudaMemsetAsync(W.fbits, 0, (size_t)L.fwords * 4, s));
    CK(cudaMemsetAsync(W.dc, 0, offsetof(Counters, first_nonfinite), s));
    k_loop_reset<<<1, 32, 0, s>>>(W.ls);
    st->launches += 2;
  }
  const bool use_graph = !o->profile && !c->verbose && !c->no_graph && c->cap_stream && c->graph;
  if (use_graph) {
    // a3-a7 on the device: one graph launch runs every round
    LoopGraph& G = *c->graph;
    if (!G.exec || G.f != f || G.fhat != fhat || G.g != g_out || G.ws != ws || G.xi != o->xi ||
        G.q_max != o->q_max || G.q_cap != o->q_cap || G.tier != o->tier || G.frontier != (int)frontier_mode ||
        G.max_rounds != (long long)max_rounds || G.sdirty != (const void*)c->sdirty) {
      status = build_loop_graph<D>(c, G, f, fhat, o, W, g_out, ws, L, max_rounds, frontier_mode, s);
      if (status != DMTZ_OK) return status;
    }
    const unsigned long long sw0 = first ? 0ull : hls->sweeps;
    CK(cudaGraphLaunch(G.exec, s));
    CK(cudaMemcpyAsync(hls, W.ls, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    st->launches += 5 * (int64_t)(hls->sweeps - sw0);
  } else {
    for (;;) {
      status = round_phase<D>(c, f, fhat, o, W, g_out, W.units, n_units, W.units, n_units,
                              frontier_mode ? W.fbits : nullptr, (int)L.fwords, 0, g.nz, 0, g.nz, o->profile != 0,
                              max_rounds, frontier_mode ? 1 : 0, hls, &st->launches, s);
      if (status != DMTZ_OK) break;
      float ms0 = 0.f, ms1 = 0.f;
      if (o->profile) {
        float ms2 = 0.f;
        CK(cudaEventElapsedTime(&ms0, c->ev[0], c->ev[1]));
        CK(cudaEventElapsedTime(&ms1, c->ev[1], c->ev[2]));
        CK(cudaEventElapsedTime(&ms2, c->ev[2], c->ev[3]));
        st->sweep_ms += ms0 + ms1;
        st->edit_ms += ms2;
        st->screen_ms += ms0;
        st->decode_ms += ms1;
        if (ms0 > 0 && (int64_t)hc->n_recomputed == g.N) { st->screen_ms_full += ms0; st->n_screen_full++; }
      }
      if (c->verbose)
        fprintf(stderr, "dmtz round %llu: units %llu recomputed %llu swept %llu false %llu targets %llu changed %llu"
                " decoded %llu items %llu replayed %llu | screen %.3f ms decode %.3f ms\n",
                hls->sweeps, hc->n_units, hc->n_recomputed, hc->n_swept, hc->n_false, hc->n_targets, hc->n_changed,
                hc->n_decoded, hc->n_items, hc->n_replayed, ms0, ms1);
      const bool go = hls->status == 0 && hls->last_false != 0;  // the check advanced the round
      if (!go) break;
    }
  }
  return status;
}

template <int D>
void loop_stats(dmtz_ctx* c, dmtz_stats* st) {
  LoopState* hls = c->host_ls;
  st->sweeps = (int64_t)hls->sweeps;
  st->anchors_swept = (int64_t)hls->anchors_swept;
  st->anchors_recomputed = (int64_t)hls->recomputed;
  st->anchors_decoded = (int64_t)hls->decoded;
  st->cells_evaluated = (int64_t)hls->items;
  st->anchors_replayed = (int64_t)hls->replayed;
  st->rounds = (int64_t)hls->rounds;
  st->n_false_round0 = (int64_t)hls->n_false0;
  for (int k = 0; k < 8; k++) st->false_by_kind_round0[k] = (int64_t)hls->kinds0[k];
  const dmtz_status status = (dmtz_status)hls->status;
  if (status == DMTZ_E_INTERNAL) set_err("gradient invariant violated (round %llu)", hls->round);
  else if (status == DMTZ_E_STUCK) set_err("no target could move (round %llu)", hls->round);
  else if (status == DMTZ_E_ITER_CAP) set_err("round cap %llu reached", hls->round);
}

template <int D>
dmtz_status finish_edits(dmtz_ctx* c, WS<D>& W, float* g_out, dmtz_status status, dmtz_edit* edits, int64_t cap,
                         int64_t* n_edits, dmtz_stats* st, cudaStream_t s) {
  // a8: edit list
  int64_t nl = 0;
  dmtz_status es = edits_phase<D>(c, W, g_out, 0, c->g.N, 0, edits, cap, n_edits, &nl, &st->launches, s);
  if (es != DMTZ_OK) { st->status = es; return es; }
  st->n_edited = *n_edits;
  st->n_lossless = nl;
  st->n_quantized = st->n_edited - st->n_lossless;
  if (status == DMTZ_OK && *n_edits > cap) { status = DMTZ_E_CAPACITY; set_err("edit list needs %lld entries", (long long)*n_edits); }
  st->status = status;
  return status;
}

template <int D>
dmtz_status correct_impl(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                         char* ws, const Layout& L, float* g_out, dmtz_edit* edits, int64_t cap,
                         int64_t* n_edits, dmtz_stats* st, cudaStream_t s) {
  const Grid& g = c->g;
  WS<D> W(ws, L, g);
  dmtz_status status = setup_phase<D>(c, f, fhat, o, W, g_out, 0, &st->launches, s);
  if (status != DMTZ_OK) { st->status = status; return status; }
  const unsigned long long max_rounds =
      o->max_rounds > 0 ? (unsigned long long)o->max_rounds : (unsigned long long)g.N * (unsigned long long)(o->q_cap + 1);
  status = run_cloop<D>(c, f, fhat, o, W, ws, L, g_out, max_rounds, true, st, s);
  if (status == DMTZ_E_CUDA) { st->status = status; return status; }
  if (status == DMTZ_OK) {
    loop_stats<D>(c, st);
    status = (dmtz_status)c->host_ls->status;
  }
  return finish_edits<D>(c, W, g_out, status, edits, cap, n_edits, st, s);
}

// ----------------------------------------------------------------------------- tiers 3-4
// sep_ws layout: codes scratch (N x code), tier 3: saved lb + state (N x 8), the CSR
// of f's separatrices, a per-branch scratch, the per-cell descriptors, the per-cell
// mismatch bits, the per-anchor changed-code bits, and for tier 3 the CSR of g's
// separatrices + per-branch end flags.
struct SepLayout {
  size_t codes, save, off, cells, origin, term, kind, first, cb, canc, mbits, sdirty, sdil, goff, gcells, gorigin, gterm, gkind,
      flag, cidx, cmap, cbsum, t3box, t3st, t3psum, t3hits, fsave, fsave_bytes, total;
};

// tier 3's end cache (k_t3_valid): 16-bit box coordinates, 32-bit prefix sums; 13 B per
// branch, so it is left out above 2^28 branches (C4's 754 M: 34 S-rounds, no need), and
// the saved f-side arrays (20 B per voxel) above 2^26 voxels (recomputed instead) -- C4
// tier 3 stays within a B200's memory
inline bool t3_cache_ok(const Grid& g, int64_t cap_b) {
  return g.nx <= 65535 && g.ny <= 65535 && g.nz <= 65535 && g.N < (1ll << 31) && cap_b <= (1ll << 28);
}
inline bool t3_fsave_ok(const Grid& g) { return g.N <= (1ll << 26); }

SepLayout sep_layout(const dmtz_ctx* c, int tier, int64_t cap_b, int64_t cap_c) {
  SepLayout S = {};
  const size_t N = (size_t)c->g.N;
  const size_t cs = c->D == 3 ? 8 : 2;
  size_t o = 0;
  S.codes = o; o += align_up(N * cs);
  if (tier == 3) {
    S.save = o; o += align_up(N * 8);
    // f's codes, critical masks and lowest-vertex positions (contiguous in the workspace),
    // which the candidate traces' scratch overwrites
    if (t3_fsave_ok(c->g)) {
      const Layout L = layout_for(c);
      S.fsave_bytes = L.lb - L.cand_f;
      S.fsave = o; o += align_up(S.fsave_bytes);
    }
  }
  S.off = o; o += align_up(((size_t)cap_b + 1) * 8);
  S.cells = o; o += align_up((size_t)cap_c * 8 + 8);
  S.origin = o; o += align_up((size_t)cap_b * 8 + 8);
  S.term = o; o += align_up((size_t)cap_b * 8 + 8);
  S.kind = o; o += align_up((size_t)cap_b + 8);
  S.first = o; o += align_up((size_t)cap_b * 4 + 8);
  S.cb = o; o += align_up((size_t)cap_c + 8);  // per-cell descriptors
  S.canc = o; o += align_up((size_t)cap_c * 4 + 8);  // anchors of the examined cells
  S.mbits = o; o += align_up((size_t)cap_c / 8 + 8);
  S.sdirty = o; o += align_up(N / 8 + 8);
  S.sdil = o; o += align_up(N / 8 + 8);
  if (tier == 3) {
    S.goff = o; o += align_up(((size_t)cap_b + 1) * 8);
    S.gcells = o; o += align_up((size_t)cap_c * 8 + 8);
    S.gorigin = o; o += align_up((size_t)cap_b * 8 + 8);
    S.gterm = o; o += align_up((size_t)cap_b * 8 + 8);
    S.gkind = o; o += align_up((size_t)cap_b + 8);
    S.flag = o; o += align_up((size_t)cap_b + 8);
    S.cidx = o; o += align_up(((size_t)cap_b + 1) * 8);        // candidate flags -> indices (scan)
    S.cmap = o; o += align_up((size_t)cap_b * 4 + 8);          // candidate -> branch of f
    S.cbsum = o; o += align_up(((size_t)cap_b / 8192 + 4) * 8);
    if (t3_cache_ok(c->g, cap_b)) {
      S.t3box = o; o += align_up((size_t)cap_b * sizeof(T3Box) + 8);
      S.t3st = o; o += align_up((size_t)cap_b + 8);
      S.t3psum = o; o += align_up(N * 4);
      S.t3hits = o; o += align_up(8);
    }
  }
  S.total = o;
  return S;
}

// trace of `codes` into (off, cells, origin, term, kind) with the workspace scratch
template <int D>
dmtz_status trace_into(dmtz_ctx* c, char* ws, const Layout& L, const void* codes, char* sw, size_t off, size_t cells,
                       size_t origin, size_t term, size_t kind, int64_t cap_b, int64_t cap_c, int64_t* nb,
                       int64_t* nc, cudaStream_t s, const int64_t* given_nbk = nullptr, bool unordered = false) {
  TraceArgs a;
  a.unordered = unordered;
  if (given_nbk)
    for (int k = 0; k < 3; k++) a.given_nbk[k] = given_nbk[k];
  a.g = c->g;
  a.codes = codes;
  a.kinds = 7u;
  a.pre = (long long*)(ws + L.cand_g);
  a.pre_bytes = L.crit_g - L.cand_g;
  a.bfs = (unsigned long long*)(ws + L.cand_f);
  a.bfs_bytes = L.counters - L.cand_f;
  a.verbose = c->verbose;
  a.crit = (uint32_t*)(ws + L.crit_g);
  a.bsum = (unsigned long long*)(ws + L.edit_bc);
  a.cnt = (Counters*)(ws + L.counters);
  a.host_cnt = c->host_cnt;
  a.out_offsets = (int64_t*)(sw + off);
  a.out_cells = (uint64_t*)(sw + cells);
  a.out_origin = (uint64_t*)(sw + origin);
  a.out_terminal = (uint64_t*)(sw + term);
  a.out_kind = (uint8_t*)(sw + kind);
  a.cap_b = cap_b;
  a.cap_c = cap_c;
  cudaError_t e = run_trace<D>(a, s);
  for (int i = 0; i < 10; i++) g_trace_levels[i] = a.level_counts[i];
  if (e != cudaSuccess) { set_err("trace: %s", cudaGetErrorString(e)); return DMTZ_E_CUDA; }
  *nb = a.n_branches;
  *nc = a.n_cells;
  if (a.n_internal) { set_err("trace: cycle or inconsistent gradient"); return DMTZ_E_INTERNAL; }
  if (a.n_overflow) {
    set_err("trace: %lld connector BFS larger than the workspace scratch", (long long)a.n_overflow);
    return DMTZ_E_CAPACITY;
  }
  if (a.n_branches > cap_b || a.n_cells > cap_c) {
    set_err("separatrices need %lld branches / %lld cells", (long long)a.n_branches, (long long)a.n_cells);
    return DMTZ_E_CAPACITY;
  }
  if (a.n_branches >= (1ll << 32)) { set_err("more than 2^32 separatrix branches"); return DMTZ_E_CAPACITY; }
  return DMTZ_OK;
}

template <int D>
dmtz_status preserve_impl(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o, char* ws,
                          const Layout& L, char* sw, int64_t cap_b, int64_t cap_c, float* g_out, dmtz_edit* edits,
                          int64_t cap, int64_t* n_edits, dmtz_stats* st, dmtz_sloop_stats* ss, cudaStream_t s) {
  const Grid& g = c->g;
  WS<D> W(ws, L, g);
  const SepLayout S = sep_layout(c, o->tier, cap_b, cap_c);
  const RowGeom rg = row_geom(g);
  const size_t cs = D == 3 ? 8 : 2;
  Counters* hc = c->host_cnt;
  LoopState* hls = c->host_ls;
  cudaEvent_t e0 = c->ev[0], e1 = c->ev[1];
  int64_t nb = 0, nc = 0;
  // the separatrices of f, once (the trace borrows the loop's workspace: before setup)
  CK(cudaEventRecord(e0, s));
  launch_codes<D>(g, f, sw + S.codes, 0, g.nz, s);
  CK(cudaGetLastError());
  dmtz_status status = trace_into<D>(c, ws, L, sw + S.codes, sw, S.off, S.cells, S.origin, S.term, S.kind, cap_b,
                                     cap_c, &nb, &nc, s);
  ss->sep_branches = nb;
  ss->sep_cells = nc;
  if (status != DMTZ_OK) { st->status = status; return status; }
  const long long* off = (const long long*)(sw + S.off);
  const uint64_t* cells = (const uint64_t*)(sw + S.cells);
  const uint64_t* origin = (const uint64_t*)(sw + S.origin);
  const uint8_t* kind = (const uint8_t*)(sw + S.kind);
  uint32_t* first = (uint32_t*)(sw + S.first);  // the list of long branches, then per-branch origin mismatches
  uint32_t* mbits = (uint32_t*)(sw + S.mbits);
  uint32_t* sdirty = (uint32_t*)(sw + S.sdirty);
  uint32_t* sdil = (uint32_t*)(sw + S.sdil);
  const int64_t dwords = (g.N + 31) / 32;
  uint8_t* desc = (uint8_t*)(sw + S.cb);
  uint32_t* canc = (uint32_t*)(sw + S.canc);
  if (nb > 0) {
    CK(cudaMemsetAsync(&W.dc->pad[2], 0, 8, s));
    k_cell_desc_short<D><<<clamp_blocks(nb, 256), 256, 0, s>>>(off, kind, cells, nb, desc, canc, first,
                                                               &W.dc->pad[2]);
    k_cell_desc_long<D><<<148 * 8, 256, 0, s>>>(off, kind, cells, first, &W.dc->pad[2], desc, canc);
    CK(cudaGetLastError());
    st->launches += 2;
  }
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ss->trace_ms = ms;
  }
  status = setup_phase<D>(c, f, fhat, o, W, g_out, 0, &st->launches, s);
  if (status != DMTZ_OK) { st->status = status; return status; }
  if (o->tier == 5) {  // pre-clamp f's critical cells, then the tier-4 workflow
    k_t5_clamp<D><<<clamp_blocks(g.N, 256), 256, 0, s>>>(W.crit_f, W.lb, g_out, W.state, g);
    CK(cudaGetLastError());
    st->launches += 1;
  }
  const unsigned long long max_rounds =
      o->max_rounds > 0 ? (unsigned long long)o->max_rounds : (unsigned long long)g.N * (unsigned long long)(o->q_cap + 1);
  const bool frontier_mode = !o->full_sweeps;
  const int64_t nwords = (int64_t)(W.rowbit_bytes / 4);
  const float step = ldexpf(o->xi, -o->q_max);
  const int fwords_smem = frontier_mode && L.fwords * 4 <= 32768 ? (int)L.fwords : 0;
  int64_t c_rounds = 0;
  unsigned long long sw_before = 0;
  if (nb > 0) {
    CK(cudaMemsetAsync(sdirty, 0, (size_t)g.N / 8 + 8, s));
    c->sdirty = sdirty;
  }
  // tier 3's end cache: per branch box + end comparison of its last trace in g
  const bool t3c = o->tier == 3 && S.t3box != 0;
  uint8_t* t3st = t3c ? (uint8_t*)(sw + S.t3st) : nullptr;
  T3Box* t3box = t3c ? (T3Box*)(sw + S.t3box) : nullptr;
  unsigned long long* t3hits = t3c ? (unsigned long long*)(sw + S.t3hits) : nullptr;
  if (t3c && nb > 0) CK(cudaMemsetAsync(t3st, 0, (size_t)nb, s));
  struct Reset { dmtz_ctx* c; ~Reset() { c->sdirty = nullptr; } } reset{c};
  for (bool first_call = true;; first_call = false) {
    status = run_cloop<D>(c, f, fhat, o, W, ws, L, g_out, max_rounds, first_call, st, s);
    if (status != DMTZ_OK) { st->status = status; return status; }
    status = (dmtz_status)hls->status;
    c_rounds += (int64_t)(hls->sweeps - sw_before) - (status == DMTZ_OK ? 1 : 0);
    sw_before = hls->sweeps;
    if (status != DMTZ_OK || nb == 0) break;
    // S-round in round r: the last sweep found no false critical cell
    const unsigned long long r = hls->round;
    CK(cudaEventRecord(e0, s));
    // DMTZ_T3_LOG: the S-round's phases (host clock, synchronising after each)
    char plog[512];
    int plen = 0;
    auto p_prev = std::chrono::steady_clock::now();
    auto pmark = [&](const char* what) {
      if (!c->t3_log) return;
      cudaStreamSynchronize(s);
      const auto now = std::chrono::steady_clock::now();
      if (plen < 400)
        plen += snprintf(plog + plen, sizeof plog - plen, " %s %.2f", what,
                         std::chrono::duration<double, std::milli>(now - p_prev).count());
      p_prev = now;
    };
    plog[0] = 0;
    const uint8_t* flag = nullptr;
    CK(cudaMemsetAsync(W.dc, 0, offsetof(Counters, first_nonfinite), s));
    CK(cudaMemsetAsync(&W.dc->pad[3], 0, 5 * 8, s));
    const int full = ss->s_rounds == 0 ? 1 : 0;
    if (!full) {
      k_sdirty_dilate<<<clamp_blocks(dwords, 256), 256, 0, s>>>(sdirty, dwords, g.sy, g.sz, sdil);
      st->launches += 1;
    }
    if (nc > 0) {
      const int64_t nblk = ((nc + 31) / 32 + 8 * TM_U - 1) / (8 * TM_U);  // 8 warps x TM_U words per block
      k_tm_cells<D><<<(unsigned)nblk, 256, 0, s>>>(cells, nc, desc, canc, W.cand_f, W.cand_g, W.crit_f, g, sdil,
                                                   full, mbits, W.dc);
      st->launches += 1;
    }
    pmark("tm_cells");
    if (o->tier == 3) {
      // the candidates (branches with a troublemaker) are traced in g; the others end as in f
      long long* cidx = (long long*)(sw + S.cidx);
      uint32_t* cmap = (uint32_t*)(sw + S.cmap);
      if (t3c) {
        if (!full) {   // drop the cached ends whose box saw a changed code (sdil) since their trace
          int32_t* P = (int32_t*)(sw + S.t3psum);
          k_t3_psum_x<<<clamp_blocks(g.ny * g.nz * 32, 256), 256, 0, s>>>(sdil, g, P);
          k_t3_psum_yz<<<clamp_blocks(g.nx * g.nz, 256), 256, 0, s>>>(g, 1, P);
          k_t3_psum_yz<<<clamp_blocks(g.nx * g.ny, 256), 256, 0, s>>>(g, 2, P);
          k_t3_valid<<<clamp_blocks(nb, 256), 256, 0, s>>>(P, g, nb, t3box, t3st);
          st->launches += 4;
        }
        CK(cudaMemsetAsync(t3hits, 0, 8, s));
      }
      pmark("valid");
      CK(cudaMemsetAsync(sw + S.flag, 0, (size_t)nb, s));
      k_t3_cand<D><<<clamp_blocks(nb + 1, 256, 148 * 64), 256, 0, s>>>(cells, off, kind, origin, nb, W.cand_f,
                                                                       W.cand_g, W.crit_f, g, mbits, cidx, W.dc,
                                                                       t3st, (uint8_t*)(sw + S.flag), t3hits);
      CK(cudaGetLastError());
      CK(scan_i64(cidx, nb + 1, (unsigned long long*)(sw + S.cbsum), &W.dc->pad[0], &hc->pad[0], s));
      const int64_t ncand = (int64_t)hc->pad[0];
      CK(cudaMemcpyAsync(hc, W.dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      const int64_t nkc[3] = {(int64_t)hc->pad[4], (int64_t)hc->pad[5], (int64_t)hc->pad[6]};
      ss->cells_checked += (int64_t)hc->pad[7];
      st->launches += 4;
      if (ncand > 0) {
        k_t3_fill<D><<<clamp_blocks(nb, 256, 148 * 64), 256, 0, s>>>(
            cells, off, kind, origin, nb, cidx, g, (uint64_t*)(sw + S.gorigin), (uint8_t*)(sw + S.gkind),
            (uint64_t*)(sw + S.gterm), cmap);
        // trace g with the loop's workspace (its codes are current), then restore the loop state
        CK(cudaMemcpyAsync(sw + S.codes, W.cand_g, (size_t)g.N * cs, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(sw + S.save, W.lb, (size_t)g.N * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(sw + S.save + (size_t)g.N * 4, W.state, (size_t)g.N * 4, cudaMemcpyDeviceToDevice, s));
        if (S.fsave) CK(cudaMemcpyAsync(sw + S.fsave, ws + L.cand_f, S.fsave_bytes, cudaMemcpyDeviceToDevice, s));
        // trace the candidates in chunks whose g-paths fit the CSR (halving a chunk that does not)
        pmark("cand+save");
        const auto t3_t0 = std::chrono::steady_clock::now();
        int n_chunks = 0;
        int64_t c0 = 0, chunk = ncand;
        while (c0 < ncand) {
          const int64_t c1 = c0 + chunk < ncand ? c0 + chunk : ncand;
          int64_t knb[3];
          int64_t kb = 0;
          for (int k = 0; k < 3; k++) {   // candidates are grouped DESC, ASC, CONN
            const int64_t lo = kb > c0 ? kb : c0, hi = kb + nkc[k] < c1 ? kb + nkc[k] : c1;
            knb[k] = hi > lo ? hi - lo : 0;
            kb += nkc[k];
          }
          int64_t gnb = 0, gnc = 0;
          status = trace_into<D>(c, ws, L, sw + S.codes, sw, S.goff, S.gcells, S.gorigin + 8 * c0, S.gterm + 8 * c0,
                                 S.gkind + c0, c1 - c0, cap_c, &gnb, &gnc, s, knb, c->t3_unordered);
          if (status == DMTZ_E_CAPACITY && c1 - c0 > 1 && gnb == c1 - c0) {
            // k_t3_fill's j inputs of this chunk were consumed: refill them, retry half
            k_t3_fill<D><<<clamp_blocks(nb, 256, 148 * 64), 256, 0, s>>>(
                cells, off, kind, origin, nb, cidx, g, (uint64_t*)(sw + S.gorigin), (uint8_t*)(sw + S.gkind),
                (uint64_t*)(sw + S.gterm), cmap);
            chunk = (c1 - c0 + 1) / 2;
            status = DMTZ_OK;
            continue;
          }
          if (status == DMTZ_OK && gnb != c1 - c0) {
            set_err("tier 3: %lld candidates traced, %lld given", (long long)gnb, (long long)(c1 - c0));
            status = DMTZ_E_INTERNAL;
          }
          if (status != DMTZ_OK) { st->status = status; return status; }
          k_t3_flags_cand<D><<<clamp_blocks((c1 - c0) * 32, T3_WARPS * 32), T3_WARPS * 32, 0, s>>>(
              off, cells, (const uint64_t*)(sw + S.term), kind, (const long long*)(sw + S.goff),
              (const uint64_t*)(sw + S.gcells), (const uint64_t*)(sw + S.gterm) + c0, cmap + c0, c1 - c0,
              (uint8_t*)(sw + S.flag), (const uint64_t*)(sw + S.gorigin) + c0, g, t3box, t3st);
          CK(cudaGetLastError());
          c0 = c1;
          n_chunks++;
        }
        if (c->t3_log) {
          unsigned long long hits = 0;
          if (t3c) CK(cudaMemcpy(&hits, t3hits, 8, cudaMemcpyDeviceToHost));
          fprintf(stderr, "t3 S-round %lld: %llu cached ends reused\n", (long long)ss->s_rounds, hits);
          CK(cudaStreamSynchronize(s));
          const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t3_t0).count();
          fprintf(stderr, "t3 S-round %lld: candidates %lld (desc %lld asc %lld conn %lld), %d chunks, trace %.3f ms,"
                  " connector levels %lld %lld %lld %lld %lld %lld\n",
                  (long long)ss->s_rounds, (long long)ncand, (long long)nkc[0], (long long)nkc[1], (long long)nkc[2],
                  n_chunks, ms, (long long)g_trace_levels[0], (long long)g_trace_levels[1],
                  (long long)g_trace_levels[2], (long long)g_trace_levels[3], (long long)g_trace_levels[4],
                  (long long)g_trace_levels[5]);
        }
        pmark("trace");
        CK(cudaMemcpyAsync(W.lb, sw + S.save, (size_t)g.N * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(W.state, sw + S.save + (size_t)g.N * 4, (size_t)g.N * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(W.cand_g, sw + S.codes, (size_t)g.N * cs, cudaMemcpyDeviceToDevice, s));
        if (S.fsave) {
          CK(cudaMemcpyAsync(ws + L.cand_f, sw + S.fsave, S.fsave_bytes, cudaMemcpyDeviceToDevice, s));
        } else {
          launch_codes<D>(g, f, W.cand_f, 0, g.nz, s);
          k_critmask<D><<<anchor_grid(g, 0, g.nz, 128), 128, 0, s>>>(W.cand_f, W.crit_f, g);
          k_lowpos<D><<<anchor_grid(g, 0, g.nz, 128), 128, 0, s>>>(f, W.lowpos, g);
          st->launches += 3;
        }
        CK(cudaMemsetAsync(W.tbits, 0, nwords * 4, s));
        CK(cudaMemsetAsync(W.fmark, 0, W.rowbit_bytes, s));
        CK(cudaMemsetAsync(W.vchg, 0, 2 * W.rowbit_bytes, s));
        CK(cudaMemsetAsync(W.fbits, 0, (size_t)L.fwords * 4, s));
        // the trace cleared the counters, the full-sweep unit count among them
        if (!frontier_mode) CK(units_range(rg, 0, g.nz, W.units, &W.dc->n_units, s));
        CK(cudaGetLastError());
        st->launches += frontier_mode ? 0 : 1;
        pmark("restore");
      }
      CK(cudaMemsetAsync(W.dc, 0, offsetof(Counters, first_nonfinite), s));
      CK(cudaMemsetAsync(&W.dc->pad[3], 0, 5 * 8, s));
      flag = (const uint8_t*)(sw + S.flag);
    }
    k_tm_targets<D><<<clamp_blocks(nb, 256, 148 * 64), 256, 0, s>>>(cells, off, kind, origin, nb, W.cand_f, W.cand_g,
                                                                    W.crit_f, g, rg, mbits, flag, sdil, full,
                                                                    (uint8_t*)first,
                                                                    W.tbits, W.dc);
    CK(cudaMemsetAsync(sdirty, 0, (size_t)g.N / 8 + 8, s));
    k_edit_rows<D><<<clamp_blocks(nwords, 256), 256, fwords_smem * 4, s>>>(
        W.tbits, nwords, fhat, W.lb, g_out, W.state, W.dc, step, o->q_cap, frontier_mode ? W.fbits : nullptr, g, rg,
        fwords_smem, frontier_mode ? W.vchg : nullptr, W.vwords, W.ls, FastDiv((uint32_t)rg.wpr),
        FastDiv((uint32_t)g.ny));
    CK(cudaGetLastError());
    st->launches += 3;
    CK(cudaEventRecord(e1, s));
    CK(cudaMemcpyAsync(hc, W.dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ss->s_ms += ms;
      pmark("targets");
      if (c->t3_log) fprintf(stderr, "S-round %lld: %.3f ms:%s\n", (long long)ss->s_rounds, ms, plog);
    }
    if (hc->n_internal) { set_err("troublemaker without an original partner"); status = DMTZ_E_INTERNAL; break; }
    const int64_t ntm = (int64_t)hc->pad[3];
    if (ntm == 0) break;  // no false separatrix (and no false critical cell): done
    if (ss->s_rounds == 0) ss->tm_round1 = ntm;
    ss->s_rounds++;
    ss->troublemakers += ntm;
    for (int k = 0; k < 3; k++) ss->tm_by_kind[k] += (int64_t)hc->pad[4 + k];
    ss->cells_checked += (int64_t)hc->pad[7];
    if (hc->n_changed == 0) { set_err("no target could move (round %llu)", r); status = DMTZ_E_STUCK; break; }
    if (r == max_rounds) { set_err("round cap %llu reached", r); status = DMTZ_E_ITER_CAP; break; }
    // resume the C-loop at round r + 1 over the units the edits marked
    k_set_round<<<1, 32, 0, s>>>(W.ls, r + 1);
    if (frontier_mode) {
      CK(cudaMemsetAsync(&W.dc->n_units, 0, 8, s));
      k_units_from_bits<<<clamp_blocks(rg.units, 256, 4096), 256, 0, s>>>(W.fbits, rg.units, W.units, &W.dc->n_units);
      st->launches += 1;
    }
    CK(cudaMemsetAsync(W.dc, 0, offsetof(Counters, first_nonfinite), s));
    CK(cudaGetLastError());
    st->launches += 1;
  }
  loop_stats<D>(c, st);
  st->rounds = c_rounds;
  ss->c_rounds = c_rounds;
  return finish_edits<D>(c, W, g_out, status, edits, cap, n_edits, st, s);
}

}  // namespace

static dmtz_status slab_round_enqueue(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                                      const dmtz_slab* sl, char* ws, const Layout& L, float* g_out, int64_t round,
                                      bool full, cudaStream_t s, long long* ctl = nullptr);

// The multi-GPU C-loop (dmtz_dist.cuh): one rank's slab, its owned planes in and out.
static dmtz_status correct_dist(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                                char* ws, size_t wsb, const Layout& L, float* g_out, dmtz_edit* edits, int64_t cap,
                                int64_t* n_edits, dmtz_stats* st, cudaStream_t s) {
  if (!c->has_tr || !c->tr.exchange || !c->tr.allreduce_sum_i64) {
    set_err("multi-GPU context without a transport (NCCL id or dmtz_ctx_set_transport)");
    st->status = DMTZ_E_NCCL;
    return DMTZ_E_NCCL;
  }
  const Grid& g = c->g;  // the local grid
  const int64_t N = g.N, sz = g.sz;
  float* floc = (float*)(ws + L.dist);
  float* fhloc = floc + N;
  float* gloc = fhloc + N;
  float* stage = gloc + N;
  long long* dcnt = (long long*)(stage + N);
  const int nout = 12 + 2 * c->world;
  long long* hcnt = (long long*)c->host_cnt;  // pinned, 512 B >= 8 (14 + 2 world) for world <= 25
  if (nout > 64) { set_err("world %d too large for the pinned counter block", c->world); return DMTZ_E_ARG; }
  const int64_t oz0 = c->z0 - c->lz0, oz1 = c->z1 - c->lz0, nown = oz1 - oz0;
  auto comm_fail = [&](const char* what) {
    set_err("transport %s failed", what);
    st->status = DMTZ_E_NCCL;
    return DMTZ_E_NCCL;
  };
  // owned planes in; halo planes of f and fhat from the neighbours (once)
  CK(cudaMemcpyAsync(floc + oz0 * sz, f, (size_t)(nown * sz) * 4, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(fhloc + oz0 * sz, fhat, (size_t)(nown * sz) * 4, cudaMemcpyDeviceToDevice, s));
  for (float* a : {floc, fhloc}) {
    HaloPlan h = halo_plan(c, g, a, a, 1, 1, 1, 1);
    if (run_exchange(c, h, s)) return comm_fail("exchange");
  }
  dmtz_slab sl;
  sl.z_offset = c->lz0;
  sl.own_z0 = oz0;
  sl.own_z1 = oz1;
  sl.anchor_z0 = std::max<int64_t>(0, c->z0 - 2) - c->lz0;
  sl.anchor_z1 = std::min<int64_t>(c->gnz, c->z1 + 1) - c->lz0;
  dmtz_status bst = dmtz_slab_begin(c, floc, fhloc, o, &sl, ws, wsb, gloc, (dmtz_stream_t)s);
  // every rank learns whether any rank failed its validation (no rank may enter the
  // round loop alone: its exchanges would wait forever)
  hcnt[0] = bst != DMTZ_OK ? 1 : 0;
  CK(cudaMemcpyAsync(dcnt, hcnt, 8, cudaMemcpyHostToDevice, s));
  if (c->tr.allreduce_sum_i64(c->tr.user, (int64_t*)dcnt, 1, (dmtz_stream_t)s)) return comm_fail("allreduce");
  CK(cudaMemcpyAsync(hcnt, dcnt, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bst != DMTZ_OK) { st->status = bst; return bst; }
  if (hcnt[0]) { set_err("another rank failed its input validation"); st->status = DMTZ_E_BOUND; return DMTZ_E_BOUND; }
  WS<3> W(ws, L, g);
  const RowGeom rg = row_geom(g);
  const int64_t per_plane = g.ny * rg.wpr;
  const int64_t nface = std::min<int64_t>(3, nown);
  const int64_t max_rounds = o->max_rounds ? o->max_rounds : c->dims.nx * c->dims.ny * c->gnz * (int64_t)(o->q_cap + 1);
  std::vector<long long> tot(nout, 0);
  int status = -1;
  int64_t r = 0;
  unsigned* fflags = (unsigned*)(dcnt + 64 + DCTL_N);   // this round's two face flags (k_face_flags)
  CK(cudaMemsetAsync(fflags, 0, 8, s));
  if (c->dist_sync > 1) {
    // batched: rounds_per_sync rounds per host check; the stop rule and the halo gates
    // live on the device (k_dist_stop), every face is exchanged, and a face whose planes
    // the neighbour did not change is not applied (k_halo's gate)
    long long* ctl = dcnt + 64;
    long long* hctl = hcnt + 64 - DCTL_N;  // the pinned block's tail (nout <= 48 here)
    if (nout > 64 - DCTL_N) { set_err("world %d too large for the batched mode", c->world); return DMTZ_E_ARG; }
    CK(cudaMemsetAsync(ctl, 0, DCTL_N * 8, s));
    c->dist_graph_used = 0;
    // one round rr on stream ss: exchange, halo update, round, face flags, counters,
    // all-reduce, stop rule -- device work and transport calls only (capturable)
    int64_t launches_per_round = 0;
    auto one_round = [&](int64_t rr, cudaStream_t ss) -> dmtz_status {
      int64_t la = 0;
      if (rr > 1) {
        HaloPlan h = halo_plan(c, g, gloc, stage, 1, 1, 1, 1);
        if (run_exchange(c, h, ss)) return comm_fail("exchange");
        for (int i = 0; i < h.n; i++)
          if (h.rz1[i] > h.rz0[i]) {
            const int64_t items = (h.rz1[i] - h.rz0[i]) * g.ny * rg.wpr;
            k_halo<<<clamp_blocks(items * 32, 256), 256, 0, ss>>>(
                gloc, stage + h.rz0[i] * sz, h.rz0[i], h.rz1[i], g, rg, W.vchg + (int64_t)((rr - 1) & 1) * W.vwords,
                W.fbits, ctl, h.rz0[i] == 0 ? DCTL_GATE_LO : DCTL_GATE_HI);
            la++;
          }
      }
      uint32_t* vround = W.vchg + (int64_t)(rr & 1) * W.vwords;
      if (c->world > 1) {   // face flags (a one-rank world has no faces)
        CK(cudaMemsetAsync(vround + oz0 * per_plane, 0, (size_t)(nface * per_plane) * 4, ss));
        CK(cudaMemsetAsync(vround + (oz1 - nface) * per_plane, 0, (size_t)(nface * per_plane) * 4, ss));
      }
      const dmtz_status rs = slab_round_enqueue(c, floc, fhloc, o, &sl, ws, L, gloc, rr, o->full_sweeps != 0, ss, ctl);
      if (rs) return rs;
      if (c->world > 1)
        k_face_flags<<<clamp_blocks(2 * nface * per_plane, 256, 148 * 2), 256, 0, ss>>>(
            vround, per_plane, oz0, oz0 + nface, oz1 - nface, oz1, fflags, ctl);
      k_dist_counters<<<1, 256, 0, ss>>>(W.dc, rr, dcnt, nout, fflags, c->rank, ctl);
      CK(cudaGetLastError());
      if (c->tr.allreduce_sum_i64(c->tr.user, (int64_t*)dcnt, nout, (dmtz_stream_t)ss)) return comm_fail("allreduce");
      k_dist_stop<<<1, 32, 0, ss>>>(dcnt, ctl, max_rounds, c->rank, c->world);
      la += 8 + (rr > 1 ? 1 : 0);  // begin, [units], screen, decode, edit_rows, loop_check, flags, counters, stop
      launches_per_round = la;
      st->launches += la;
      return DMTZ_OK;
    };
    // CUDA graph of a batch (dmtz_ctx_set_dist_graph; NCCL transport; even batch): round 1
    // runs eagerly, then one captured batch of rounds 2 .. k + 1 is replayed -- its
    // round-dependent parts (change-bitmap parity, round > 1) repeat with period 2, and
    // the device counts the rounds
    cudaGraph_t dgraph = nullptr;
    cudaGraphExec_t dexec = nullptr;
    const bool try_graph = c->dist_graph && c->nccl_comm && c->cap_stream && c->ev_aux[0] && c->dist_sync % 2 == 0;
    bool graphed = false;
    for (;;) {
      if (graphed) {
        CK(cudaGraphLaunch(dexec, s));
        r += c->dist_sync;
        st->launches += launches_per_round * c->dist_sync;
      } else if (try_graph && r == 1) {
        // capture rounds 2 .. k + 1 on the private stream, after the work already on s
        CK(cudaEventRecord(c->ev_aux[0], s));
        CK(cudaStreamWaitEvent(c->cap_stream, c->ev_aux[0], 0));
        bool ok = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        const int64_t l0 = st->launches;
        for (int b = 0; ok && b < c->dist_sync; b++) ok = one_round(r + 1 + b, c->cap_stream) == DMTZ_OK;
        const cudaError_t ec = cudaStreamEndCapture(c->cap_stream, &dgraph);
        st->launches = l0;
        ok = ok && ec == cudaSuccess && dgraph && cudaGraphInstantiate(&dexec, dgraph, 0) == cudaSuccess;
        cudaGetLastError();
        if (!ok) {   // capture refused (transport or driver): eager batches from here on
          if (dexec) cudaGraphExecDestroy(dexec);
          if (dgraph) cudaGraphDestroy(dgraph);
          dexec = nullptr;
          dgraph = nullptr;
          set_err("");
          for (int b = 0; b < c->dist_sync; b++) {
            r++;
            const dmtz_status rs = one_round(r, s);
            if (rs) return rs;
          }
        } else {
          graphed = true;
          c->dist_graph_used = 1;
          continue;
        }
      } else {
        for (int b = 0; b < c->dist_sync; b++) {
          r++;
          const dmtz_status rs = one_round(r, s);
          if (rs) return rs;
          if (try_graph && r == 1) break;   // round 1 alone, then the captured batches
        }
      }
      CK(cudaMemcpyAsync(hctl, ctl, DCTL_N * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (hctl[DCTL_HALT]) break;
    }
    if (dexec) cudaGraphExecDestroy(dexec);
    if (dgraph) cudaGraphDestroy(dgraph);

    status = (int)hctl[DCTL_STATUS];
    st->rounds = hctl[DCTL_ROUNDS];
    st->sweeps = hctl[DCTL_SWEEPS];
    st->n_false_round0 = hctl[DCTL_FALSE0];
    for (int k = 0; k < 8; k++) st->false_by_kind_round0[k] = hctl[DCTL_FALSE0 + 1 + k];
    st->halo_faces_sent = (int64_t)((c->rank > 0) + (c->rank < c->world - 1)) * (st->sweeps - 1);
  }
  while (status < 0) {
    r++;
    if (r > 1) {  // halo planes of g the neighbours changed in round r - 1
      const int lo_peer = c->rank > 0 ? (int)tot[13 + 2 * (c->rank - 1)] : 0;          // its upper face
      const int hi_peer = c->rank < c->world - 1 ? (int)tot[12 + 2 * (c->rank + 1)] : 0;  // its lower face
      const int lo_me = (int)tot[12 + 2 * c->rank], hi_me = (int)tot[13 + 2 * c->rank];
      HaloPlan h = halo_plan(c, g, gloc, stage, lo_me, lo_peer, hi_me, hi_peer);
      for (int i = 0; i < h.n; i++) {
        if (h.sbytes[i]) st->halo_faces_sent++;
        else st->halo_faces_skipped++;
      }
      if (run_exchange(c, h, s)) return comm_fail("exchange");
      for (int i = 0; i < h.n; i++)
        if (h.rz1[i] > h.rz0[i]) {
          const dmtz_status hs = dmtz_slab_halo(c, &sl, ws, wsb, gloc, stage + h.rz0[i] * sz, h.rz0[i], h.rz1[i], r - 1,
                                                (dmtz_stream_t)s);
          if (hs) return hs;
        }
    }
    // this round's change bitmap rows of the owned face planes: cleared, so that after the
    // round they hold exactly this round's edits there (the face flags)
    uint32_t* vround = W.vchg + (int64_t)(r & 1) * W.vwords;
    CK(cudaMemsetAsync(vround + oz0 * per_plane, 0, (size_t)(nface * per_plane) * 4, s));
    CK(cudaMemsetAsync(vround + (oz1 - nface) * per_plane, 0, (size_t)(nface * per_plane) * 4, s));
    const dmtz_status rs = slab_round_enqueue(c, floc, fhloc, o, &sl, ws, L, gloc, r, o->full_sweeps != 0, s);
    if (rs) return rs;
    k_face_flags<<<clamp_blocks(2 * nface * per_plane, 256, 148 * 2), 256, 0, s>>>(
        vround, per_plane, oz0, oz0 + nface, oz1 - nface, oz1, fflags, nullptr);
    k_dist_counters<<<1, 256, 0, s>>>(W.dc, r, dcnt, nout, fflags, c->rank, nullptr);
    st->launches += 7 + (r > 1 ? 1 : 0);  // set_round, [units], screen, decode, edit_rows, loop_check, flags, counters
    CK(cudaGetLastError());
    if (c->tr.allreduce_sum_i64(c->tr.user, (int64_t*)dcnt, nout, (dmtz_stream_t)s)) return comm_fail("allreduce");
    CK(cudaMemcpyAsync(hcnt, dcnt, (size_t)nout * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int i = 0; i < nout; i++) tot[i] = hcnt[i];
    if (r == 1) {
      st->n_false_round0 = tot[0];
      for (int k = 0; k < 8; k++) st->false_by_kind_round0[k] = tot[4 + k];
    }
    st->sweeps++;
    status = dist_stop(r, tot.data(), max_rounds);
    if (status != DMTZ_OK && status >= 0) st->rounds = r;
    else if (status < 0) st->rounds = r;
  }
  if (status == DMTZ_E_INTERNAL) { set_err("internal invariant violated"); st->status = status; return DMTZ_E_INTERNAL; }
  int64_t nl = 0;
  const dmtz_status es = dmtz_slab_end(c, &sl, ws, wsb, gloc, edits, cap, n_edits, &nl, (dmtz_stream_t)s);
  if (es != DMTZ_OK && es != DMTZ_E_CAPACITY) return es;
  CK(cudaMemcpyAsync(g_out, gloc + oz0 * sz, (size_t)(nown * sz) * 4, cudaMemcpyDeviceToDevice, s));
  // global edit counts
  hcnt[0] = *n_edits;
  hcnt[1] = nl;
  CK(cudaMemcpyAsync(dcnt, hcnt, 16, cudaMemcpyHostToDevice, s));
  if (c->tr.allreduce_sum_i64(c->tr.user, (int64_t*)dcnt, 2, (dmtz_stream_t)s)) return comm_fail("allreduce");
  CK(cudaMemcpyAsync(hcnt, dcnt, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  st->n_edited = hcnt[0];
  st->n_lossless = hcnt[1];
  st->n_quantized = hcnt[0] - hcnt[1];
  const dmtz_status fin = es == DMTZ_E_CAPACITY && status == DMTZ_OK ? DMTZ_E_CAPACITY : (dmtz_status)status;
  st->status = fin;
  return fin;
}

extern "C" {

int dmtz_version(void) { return 1; }

const char* dmtz_last_error(void) { return g_err; }

int dmtz_last_trace_levels(int64_t* out, int n) {
  if (!out || n < 0) return DMTZ_E_ARG;
  for (int i = 0; i < n && i < 10; i++) out[i] = g_trace_levels[i];
  return DMTZ_OK;
}

const char* dmtz_status_string(dmtz_status s) {
  switch (s) {
    case DMTZ_OK: return "ok";
    case DMTZ_E_ARG: return "invalid argument";
    case DMTZ_E_DIMS: return "invalid grid dimensions";
    case DMTZ_E_NONFINITE: return "non-finite input value";
    case DMTZ_E_BOUND: return "decompressed field violates the error bound";
    case DMTZ_E_CAPACITY: return "output capacity exceeded";
    case DMTZ_E_ITER_CAP: return "round cap reached";
    case DMTZ_E_STUCK: return "stuck: every target is at its lower bound";
    case DMTZ_E_CUDA: return "CUDA error";
    case DMTZ_E_NCCL: return "NCCL error";
    case DMTZ_E_OOM: return "workspace too small";
    case DMTZ_E_INTERNAL: return "internal invariant violated";
  }
  return "unknown status";
}

dmtz_status dmtz_ctx_create(dmtz_ctx** out, const dmtz_dims* d, int rank, int world, const void* nccl_id,
                            int cuda_device) {
  if (!out || !d) { set_err("NULL argument"); return DMTZ_E_ARG; }
  *out = nullptr;
  if (d->nx < 2 || d->ny < 2 || d->nz < 1) { set_err("dims %lld x %lld x %lld", (long long)d->nx, (long long)d->ny, (long long)d->nz); return DMTZ_E_DIMS; }
  // 32-bit work indices: row-padded bitmap words and frontier units must fit in 32 bits
  if ((d->nz * d->ny) * ((d->nx + 31) / 32) >= (1ll << 31)) {
    set_err("grid %lld x %lld x %lld too large for one context (use slabs)", (long long)d->nx, (long long)d->ny,
            (long long)d->nz);
    return DMTZ_E_DIMS;
  }
  if (world < 1 || rank < 0 || rank >= world) { set_err("rank %d of world %d", rank, world); return DMTZ_E_ARG; }
  const bool dist = world > 1 || nccl_id != nullptr;
  int64_t z0 = 0, z1 = d->nz, lz0 = 0, lz1 = d->nz;
  if (dist) {
    if (d->nz == 1) { set_err("the multi-GPU C-loop needs a 3D grid"); return DMTZ_E_DIMS; }
    if (local_slab(d->nz, world, rank, &z0, &z1, &lz0, &lz1) != DMTZ_OK) {
      set_err("%lld planes cannot be split over %d ranks (>= 3 planes each)", (long long)d->nz, world);
      return DMTZ_E_DIMS;
    }
  }
  struct RestoreDevice {
    int prev = -1;
    ~RestoreDevice() { if (prev >= 0) cudaSetDevice(prev); }
  } restore_;
  if (cudaGetDevice(&restore_.prev) != cudaSuccess) restore_.prev = -1;
  CK(cudaSetDevice(cuda_device));
  dmtz_ctx* c = new (std::nothrow) dmtz_ctx();
  if (!c) return DMTZ_E_OOM;
  c->dims = *d;
  c->dist = dist ? 1 : 0;
  c->gnz = d->nz; c->z0 = z0; c->z1 = z1; c->lz0 = lz0; c->lz1 = lz1;
  c->g.nx = d->nx; c->g.ny = d->ny; c->g.nz = lz1 - lz0;   // the local grid (the whole grid unless dist)
  c->g.N = d->nx * d->ny * c->g.nz;
  c->g.sy = d->nx; c->g.sz = d->nx * d->ny;
  c->g.set_fast();
  c->D = d->nz == 1 ? 2 : 3;
  c->device = cuda_device;
  c->graph = new (std::nothrow) LoopGraph();
  if (cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) c->cap_stream = nullptr;
  if (cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking) != cudaSuccess) c->aux_stream = nullptr;
  for (int i = 0; i < 2; i++)
    if (cudaEventCreateWithFlags(&c->ev_aux[i], cudaEventDisableTiming) != cudaSuccess) c->ev_aux[i] = nullptr;
  c->rank = rank; c->world = world;
  const char* vb = getenv("DMTZ_VERBOSE");
  c->verbose = vb && vb[0] == '1';
  const char* t3l = getenv("DMTZ_T3_LOG");
  c->t3_log = t3l && t3l[0] == '1';
  const char* t3o = getenv("DMTZ_T3_ORDERED");
  c->t3_unordered = !(t3o && t3o[0] == '1');
  const char* ng = getenv("DMTZ_NO_GRAPH");
  c->no_graph = ng && ng[0] == '1';
  const char* nk = getenv("DMTZ_NO_KEYS");
  c->no_keys = nk && nk[0] == '1';
  const char* nt = getenv("DMTZ_SCREEN_TILE");
  c->no_tile = nt && nt[0] == '0';
  // k_screen's tiled dense path uses more than the default 48 KB of dynamic shared memory
  // (set here, outside any stream capture)
  CK(cudaFuncSetAttribute(k_screen<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCREEN_TILE_BYTES));
  CK(cudaFuncSetAttribute(k_screen<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCREEN_TILE_BYTES));
  CK(cudaFuncSetAttribute(k_screen<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCREEN_TILE_BYTES));
  CK(cudaFuncSetAttribute(k_screen<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCREEN_TILE_BYTES));
  cudaError_t e = cudaMallocHost((void**)&c->host_cnt, sizeof(Counters) * 2);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&c->host_ls, sizeof(LoopState));
  if (e != cudaSuccess) {
    set_err("cudaMallocHost: %s", cudaGetErrorString(e));
    dmtz_ctx_destroy(c);
    return DMTZ_E_CUDA;
  }
  for (int i = 0; i < 4; i++) {
    e = cudaEventCreate(&c->ev[i]);
    if (e != cudaSuccess) {
      set_err("cudaEventCreate: %s", cudaGetErrorString(e));
      dmtz_ctx_destroy(c);
      return DMTZ_E_CUDA;
    }
  }
  if (nccl_id) {  // the context's own NCCL communicator (a collective call over the world)
    NcclApi* A = nccl_api();
    if (!A) { set_err("libnccl.so.2 cannot be loaded"); dmtz_ctx_destroy(c); return DMTZ_E_NCCL; }
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof id);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = A->CommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) {
      set_err("ncclCommInitRank: %s", A->GetErrorString ? A->GetErrorString(r) : "error");
      dmtz_ctx_destroy(c);
      return DMTZ_E_NCCL;
    }
    c->nccl_comm = comm;
    c->tr.user = comm;
    c->tr.exchange = nccl_exchange;
    c->tr.allreduce_sum_i64 = nccl_allreduce;
    c->has_tr = 1;
  }
  *out = c;
  return DMTZ_OK;
}

void dmtz_ctx_destroy(dmtz_ctx* c) {
  if (!c) return;
  DeviceGuard dg_(c);
  if (c->nccl_comm) {
    if (NcclApi* A = nccl_api()) A->CommDestroy((ncclComm_t)c->nccl_comm);
  }
  if (c->graph) { c->graph->reset(); delete c->graph; }
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  for (int i = 0; i < 2; i++)
    if (c->ev_aux[i]) cudaEventDestroy(c->ev_aux[i]);
  if (c->host_cnt) cudaFreeHost(c->host_cnt);
  if (c->host_ls) cudaFreeHost(c->host_ls);
  for (int i = 0; i < 4; i++)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  delete c;
}

size_t dmtz_workspace_bytes(const dmtz_ctx* c, const dmtz_correct_opts*) {
  if (!c) return 0;
  return layout_for(c).total;
}

dmtz_status dmtz_compute_gradient(dmtz_ctx* c, const float* field, void* codes, void*, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !field || !codes) { set_err("NULL argument"); return DMTZ_E_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  if (c->D == 3) launch_codes<3>(c->g, field, codes, 0, c->g.nz, s);
  else launch_codes<2>(c->g, field, codes, 0, c->g.nz, s);
  CK(cudaGetLastError());
  return DMTZ_OK;
}

dmtz_status dmtz_critical_mask(dmtz_ctx* c, const void* codes, uint32_t* crit, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !codes || !crit) { set_err("NULL argument"); return DMTZ_E_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid = anchor_grid(c->g, 0, c->g.nz, 128);
  if (c->D == 3) k_critmask<3><<<grid, 128, 0, s>>>((const Tr<3>::code_t*)codes, crit, c->g);
  else k_critmask<2><<<grid, 128, 0, s>>>((const Tr<2>::code_t*)codes, crit, c->g);
  CK(cudaGetLastError());
  return DMTZ_OK;
}

dmtz_status dmtz_correct(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                         void* workspace, size_t workspace_bytes, float* g_out, dmtz_edit* edits,
                         int64_t edits_capacity, int64_t* n_edits, dmtz_stats* st, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !f || !fhat || !o || !workspace || !g_out || !n_edits || !st || (edits_capacity > 0 && !edits) ||
      edits_capacity < 0) {
    set_err("NULL argument");
    return DMTZ_E_ARG;
  }
  memset(st, 0, sizeof *st);
  *n_edits = 0;
  if (!(o->xi > 0.0f) || !isfinite(o->xi) || o->q_max < 0 || o->q_max > 30 || o->q_cap < 1 ||
      o->q_cap > 65535 || (o->tier != 1 && o->tier != 2) || o->max_rounds < 0) {
    set_err("invalid options (xi=%g q_max=%d q_cap=%d tier=%d)", (double)o->xi, o->q_max, o->q_cap, o->tier);
    st->status = DMTZ_E_ARG;
    return DMTZ_E_ARG;
  }
  Layout L = layout_for(c);
  if (workspace_bytes < L.total) {
    set_err("workspace %zu < %zu bytes", workspace_bytes, L.total);
    st->status = DMTZ_E_OOM;
    return DMTZ_E_OOM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  dmtz_status r;
  if (c->dist) return correct_dist(c, f, fhat, o, (char*)workspace, workspace_bytes, L, g_out, edits, edits_capacity,
                                   n_edits, st, s);
  if (c->D == 3) r = correct_impl<3>(c, f, fhat, o, (char*)workspace, L, g_out, edits, edits_capacity, n_edits, st, s);
  else r = correct_impl<2>(c, f, fhat, o, (char*)workspace, L, g_out, edits, edits_capacity, n_edits, st, s);
  if (r == DMTZ_E_CUDA) st->status = r;
  return r;
}

dmtz_status dmtz_correct_host(dmtz_ctx* c, const float* f_host, const float* fhat_host, const dmtz_correct_opts* o,
                              void* workspace, size_t workspace_bytes, float* f_dev, float* fhat_dev, float* g_dev,
                              dmtz_edit* edits_dev, int64_t edits_capacity, float* g_host, dmtz_edit* edits_host,
                              int64_t* n_edits, dmtz_stats* st, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !f_host || !fhat_host || !f_dev || !fhat_dev || !n_edits || !st ||
      (edits_host && edits_capacity > 0 && !edits_dev)) {
    set_err("NULL argument");
    return DMTZ_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t fb = (size_t)c->g.N * sizeof(float);
  CK(cudaMemcpyAsync(f_dev, f_host, fb, cudaMemcpyHostToDevice, s));
  // f's gradient, critical masks and lowest vertices (a2, they read f only) run on an aux
  // stream while fhat is uploaded; dmtz_correct's setup waits for them
  const bool overlap = !c->dist && c->aux_stream && c->ev_aux[0] && c->ev_aux[1] && workspace &&
                       workspace_bytes >= layout_for(c).total;
  if (overlap) {
    const Layout L = layout_for(c);
    CK(cudaEventRecord(c->ev_aux[0], s));
    CK(cudaStreamWaitEvent(c->aux_stream, c->ev_aux[0], 0));
    if (c->D == 3) { WS<3> W((char*)workspace, L, c->g); enqueue_f_codes<3>(c->g, f_dev, W, c->aux_stream); }
    else { WS<2> W((char*)workspace, L, c->g); enqueue_f_codes<2>(c->g, f_dev, W, c->aux_stream); }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_aux[1], c->aux_stream));
    c->pre_codes = 1;
  }
  CK(cudaMemcpyAsync(fhat_dev, fhat_host, fb, cudaMemcpyHostToDevice, s));
  const dmtz_status r = dmtz_correct(c, f_dev, fhat_dev, o, workspace, workspace_bytes, g_dev, edits_dev,
                                     edits_capacity, n_edits, st, stream);
  if (overlap) {
    c->pre_codes = 0;
    CK(cudaStreamWaitEvent(s, c->ev_aux[1], 0));   // (an early error return left it possibly running)
  }
  if (r != DMTZ_OK && r != DMTZ_E_STUCK && r != DMTZ_E_ITER_CAP && r != DMTZ_E_CAPACITY) return r;
  if (g_host) CK(cudaMemcpyAsync(g_host, g_dev, fb, cudaMemcpyDeviceToHost, s));
  const int64_t ne = *n_edits < edits_capacity ? *n_edits : edits_capacity;
  if (edits_host && ne > 0)
    CK(cudaMemcpyAsync(edits_host, edits_dev, (size_t)ne * sizeof(dmtz_edit), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return r;
}

dmtz_status dmtz_correct_host_stream(dmtz_ctx* c, const float* f_host, const float* fhat_host,
                                     const dmtz_correct_opts* o, void* workspace, size_t workspace_bytes,
                                     float* f_dev, float* fhat_dev, float* g_dev, dmtz_edit* edits_dev,
                                     int64_t edits_capacity, uint8_t* stream_dev, size_t stream_cap, float* g_host,
                                     uint8_t* stream_host, size_t stream_host_cap, size_t* stream_bytes,
                                     int64_t* n_edits, dmtz_stats* st, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !o || !stream_dev || !stream_host || !stream_bytes || !n_edits || !edits_dev || edits_capacity < 1) {
    set_err("NULL argument");
    return DMTZ_E_ARG;
  }
  *stream_bytes = 0;
  const dmtz_status r = dmtz_correct_host(c, f_host, fhat_host, o, workspace, workspace_bytes, f_dev, fhat_dev, g_dev,
                                          edits_dev, edits_capacity, g_host, nullptr, n_edits, st, stream);
  if (r != DMTZ_OK && r != DMTZ_E_STUCK && r != DMTZ_E_ITER_CAP) return r;   // (capacity: the list is incomplete)
  // the artifact: the edit list encoded on the device (version 2, lossless values
  // relative to fhat), and only its bytes cross to the host
  const dmtz_status e = dmtz_encode_edits(c, edits_dev, *n_edits, o->xi, o->q_max, fhat_dev, workspace,
                                          workspace_bytes, stream_dev, stream_cap, stream_bytes, stream);
  if (e != DMTZ_OK) return e;
  if (*stream_bytes > stream_host_cap) {
    set_err("edit stream needs %zu host bytes", *stream_bytes);
    return DMTZ_E_CAPACITY;
  }
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(stream_host, stream_dev, *stream_bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return r;
}

static dmtz_status slab_check(dmtz_ctx* c, const dmtz_slab* sl, void* ws, size_t wsb, Layout* L) {
  if (!c || !sl || !ws) { set_err("NULL argument"); return DMTZ_E_ARG; }
  if (c->D != 3) { set_err("slab mode needs a 3D grid"); return DMTZ_E_DIMS; }
  if (sl->own_z0 < 0 || sl->own_z1 > c->g.nz || sl->own_z0 >= sl->own_z1 || sl->anchor_z0 < 0 ||
      sl->anchor_z1 > c->g.nz || sl->anchor_z0 > sl->anchor_z1) {
    set_err("bad slab planes");
    return DMTZ_E_ARG;
  }
  *L = layout_for(c);
  if (wsb < L->total) { set_err("workspace %zu < %zu bytes", wsb, L->total); return DMTZ_E_OOM; }
  return DMTZ_OK;
}

dmtz_status dmtz_slab_begin(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                            const dmtz_slab* sl, void* workspace, size_t wsb, float* g_out, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  Layout L;
  dmtz_status st = slab_check(c, sl, workspace, wsb, &L);
  if (st) return st;
  if (!f || !fhat || !o || !g_out || !(o->xi > 0.0f) || o->q_max < 0 || o->q_max > 30 || o->q_cap < 1 ||
      o->q_cap > 65535 || (o->tier != 1 && o->tier != 2)) {
    set_err("invalid argument");
    return DMTZ_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  WS<3> W((char*)workspace, L, c->g);
  int64_t launches = 0;
  st = setup_phase<3>(c, f, fhat, o, W, g_out, sl->z_offset * c->g.sz, &launches, s);
  if (st) return st;
  const RowGeom rg = row_geom(c->g);
  // round 1 sweeps every local unit; later rounds the frontier (own edits, halo
  // changes, units with false cells)
  CK(units_range(rg, 0, c->g.nz, W.units, &W.dc->n_units, s));
  CK(cudaMemsetAsync(W.fbits, 0, (size_t)L.fwords * 4 + 64, s));
  CK(cudaStreamSynchronize(s));
  return DMTZ_OK;
}

dmtz_status dmtz_slab_round(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                            const dmtz_slab* sl, void* workspace, size_t wsb, float* g_out, int64_t round,
                            int64_t* counters, int64_t* kinds, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  Layout L;
  dmtz_status st = slab_check(c, sl, workspace, wsb, &L);
  if (st) return st;
  if (!counters || !kinds || round < 1) { set_err("invalid argument"); return DMTZ_E_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  WS<3> W((char*)workspace, L, c->g);
  int64_t launches = 0;
  k_set_round<<<1, 32, 0, s>>>(W.ls, (unsigned long long)round);
  const RowGeom rg = row_geom(c->g);
  if (round > 1) {  // this round's unit list: the frontier marked by the last round and the halo refresh
    CK(cudaMemsetAsync(&W.dc->n_units, 0, 8, s));
    k_units_from_bits<<<clamp_blocks(rg.units, 256, 4096), 256, 0, s>>>(W.fbits, rg.units, W.units, &W.dc->n_units);
  }
  RoundExtra X;
  X.anchor_z0 = sl->anchor_z0;
  X.anchor_z1 = sl->anchor_z1;
  X.decode_marks = W.fbits;
  X.list_after = false;
  st = round_phase<3>(c, f, fhat, o, W, g_out, W.units, &W.dc->n_units, W.units, &W.dc->n_units, W.fbits,
                      (int)L.fwords, sl->own_z0, sl->own_z1, sl->own_z0, sl->own_z1, false, ~0ull, 1, c->host_ls,
                      &launches, s, X);
  if (st) return st;
  Counters* hc = c->host_cnt;
  counters[0] = (int64_t)hc->n_false;
  counters[1] = (int64_t)hc->n_changed;
  counters[2] = (int64_t)hc->n_targets;
  counters[3] = (int64_t)hc->n_internal;
  for (int k = 0; k < 8; k++) kinds[k] = round == 1 ? (int64_t)hc->kinds[k] : 0;
  return DMTZ_OK;
}

}  // extern "C"

// one slab round enqueued on s (no host synchronisation); full: every local unit and
// every code recomputed (the full-sweep mode), else the frontier with change skipping
static dmtz_status slab_round_enqueue(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                                      const dmtz_slab* sl, char* ws, const Layout& L, float* g_out, int64_t round,
                                      bool full, cudaStream_t s, long long* ctl) {
  WS<3> W(ws, L, c->g);
  int64_t launches = 0;
  // batched mode (ctl): the device counts the rounds, and once its stop flag is set the
  // unit lists stay empty, so the screen / decode / edit kernels find no work
  if (ctl) k_dist_begin<<<1, 32, 0, s>>>(ctl, W.ls);
  else k_set_round<<<1, 32, 0, s>>>(W.ls, (unsigned long long)round);
  const RowGeom rg = row_geom(c->g);
  if (round > 1) {
    CK(cudaMemsetAsync(&W.dc->n_units, 0, 8, s));
    k_units_from_bits<<<clamp_blocks(rg.units, 256, 4096), 256, 0, s>>>(W.fbits, rg.units, W.units, &W.dc->n_units,
                                                                       ctl);
    if (full) CK(units_range(rg, 0, c->g.nz, W.units, &W.dc->n_units, s, ctl));  // the frontier is ignored
  }
  RoundExtra X;
  X.anchor_z0 = sl->anchor_z0;
  X.anchor_z1 = sl->anchor_z1;
  X.decode_marks = W.fbits;
  X.list_after = false;
  return enqueue_round<3>(c, f, fhat, o, W, g_out, W.units, &W.dc->n_units, W.units, &W.dc->n_units, W.fbits,
                          (int)L.fwords, sl->own_z0, sl->own_z1, sl->own_z0, sl->own_z1, false, ~0ull,
                          cudaGraphConditionalHandle(), 0, full ? 0 : 1, &launches, s, X);
}

extern "C" {

dmtz_status dmtz_slab_round_async(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                                  const dmtz_slab* sl, void* workspace, size_t wsb, float* g_out, int64_t round,
                                  int64_t* dcounters, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  Layout L;
  dmtz_status st = slab_check(c, sl, workspace, wsb, &L);
  if (st) return st;
  if (!dcounters || round < 1) { set_err("invalid argument"); return DMTZ_E_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  st = slab_round_enqueue(c, f, fhat, o, sl, (char*)workspace, L, g_out, round, false, s);
  if (st) return st;
  WS<3> W((char*)workspace, L, c->g);
  k_counters_out<<<1, 32, 0, s>>>(W.dc, round, (long long*)dcounters);
  CK(cudaGetLastError());
  return DMTZ_OK;
}

dmtz_status dmtz_slab_halo(dmtz_ctx* c, const dmtz_slab* sl, void* workspace, size_t wsb, float* g,
                           const float* planes, int64_t z_begin, int64_t z_end, int64_t round, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  Layout L;
  dmtz_status st = slab_check(c, sl, workspace, wsb, &L);
  if (st) return st;
  if (!g || !planes || z_begin < 0 || z_end > c->g.nz || z_begin > z_end || round < 1) {
    set_err("invalid argument");
    return DMTZ_E_ARG;
  }
  if (z_begin == z_end) return DMTZ_OK;
  WS<3> W((char*)workspace, L, c->g);
  const RowGeom rg = row_geom(c->g);
  const int64_t items = (z_end - z_begin) * c->g.ny * rg.wpr;
  k_halo<<<clamp_blocks(items * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      g, planes, z_begin, z_end, c->g, rg, W.vchg + (int64_t)(round & 1) * W.vwords, W.fbits);
  CK(cudaGetLastError());
  return DMTZ_OK;
}

dmtz_status dmtz_slab_end(dmtz_ctx* c, const dmtz_slab* sl, void* workspace, size_t wsb, const float* g,
                          dmtz_edit* edits, int64_t cap, int64_t* n_edits, int64_t* n_lossless,
                          dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  Layout L;
  dmtz_status st = slab_check(c, sl, workspace, wsb, &L);
  if (st) return st;
  if (!g || !n_edits || !n_lossless || cap < 0 || (cap > 0 && !edits)) { set_err("invalid argument"); return DMTZ_E_ARG; }
  WS<3> W((char*)workspace, L, c->g);
  int64_t launches = 0;
  const int64_t plane = c->g.sz;
  st = edits_phase<3>(c, W, g, sl->own_z0 * plane, sl->own_z1 * plane, sl->z_offset * plane, edits, cap, n_edits,
                      n_lossless, &launches, (cudaStream_t)stream);
  if (st) return st;
  if (*n_edits > cap) { set_err("edit list needs %lld entries", (long long)*n_edits); return DMTZ_E_CAPACITY; }
  return DMTZ_OK;
}

dmtz_status dmtz_trace_separatrices(dmtz_ctx* c, const void* codes, uint32_t kinds, void* workspace,
                                    size_t workspace_bytes, dmtz_seps* out, int64_t cap_b, int64_t cap_c,
                                    int64_t* n_b, int64_t* n_c, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c) { set_err("NULL argument"); return DMTZ_E_ARG; }
  return dmtz_trace_separatrices_range(c, codes, kinds, 0, c->g.nz, workspace, workspace_bytes, out, cap_b, cap_c,
                                       n_b, n_c, stream);
}

dmtz_status dmtz_trace_separatrices_range(dmtz_ctx* c, const void* codes, uint32_t kinds, int64_t z_begin,
                                          int64_t z_end, void* workspace, size_t workspace_bytes, dmtz_seps* out,
                                          int64_t cap_b, int64_t cap_c, int64_t* n_b, int64_t* n_c,
                                          dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !codes || !workspace || !out || !n_b || !n_c || cap_b < 0 || cap_c < 0) {
    set_err("NULL argument");
    return DMTZ_E_ARG;
  }
  if (z_begin < 0 || z_end > c->g.nz || z_begin > z_end) { set_err("bad plane range"); return DMTZ_E_ARG; }
  Layout L = layout_for(c);
  if (workspace_bytes < L.total) { set_err("workspace %zu < %zu bytes", workspace_bytes, L.total); return DMTZ_E_OOM; }
  char* ws = (char*)workspace;
  TraceArgs a;
  a.g = c->g;
  a.codes = codes;
  a.kinds = kinds;
  a.pre = (long long*)(ws + L.cand_g);
  a.pre_bytes = L.crit_g - L.cand_g;
  a.bfs = (unsigned long long*)(ws + L.cand_f);
  a.bfs_bytes = L.counters - L.cand_f;  // cand_f .. tbits: free during a trace
  a.verbose = c->verbose;
  a.crit = (uint32_t*)(ws + L.crit_g);
  a.bsum = (unsigned long long*)(ws + L.edit_bc);
  a.cnt = (Counters*)(ws + L.counters);
  a.host_cnt = c->host_cnt;
  a.out_offsets = out->branch_offsets;
  a.out_cells = out->cells;
  a.out_origin = out->origin;
  a.out_terminal = out->terminal;
  a.out_kind = out->kind;
  a.cap_b = cap_b;
  a.cap_c = cap_c;
  a.a_lo = z_begin * c->g.sz;
  a.a_hi = z_end * c->g.sz;
  cudaError_t e = c->D == 3 ? run_trace<3>(a, (cudaStream_t)stream) : run_trace<2>(a, (cudaStream_t)stream);
  for (int i = 0; i < 10; i++) g_trace_levels[i] = a.level_counts[i];
  if (e != cudaSuccess) { set_err("trace: %s", cudaGetErrorString(e)); return DMTZ_E_CUDA; }
  *n_b = a.n_branches;
  *n_c = a.n_cells;
  if (a.n_internal) { set_err("trace: cycle or inconsistent gradient"); return DMTZ_E_INTERNAL; }
  if (a.n_overflow) {
    set_err("trace: %lld connector BFS larger than the workspace scratch", (long long)a.n_overflow);
    return DMTZ_E_CAPACITY;
  }
  if (a.n_branches > cap_b || a.n_cells > cap_c) { set_err("trace needs %lld branches / %lld cells", (long long)a.n_branches, (long long)a.n_cells); return DMTZ_E_CAPACITY; }
  return DMTZ_OK;
}


size_t dmtz_preserve_sep_bytes(const dmtz_ctx* c, const dmtz_correct_opts* o, int64_t cap_b, int64_t cap_c) {
  if (!c || !o || o->tier < 3 || cap_b < 0 || cap_c < 0) return 0;
  return sep_layout(c, o->tier, cap_b, cap_c).total;
}

dmtz_status dmtz_preserve(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                          void* workspace, size_t workspace_bytes, void* sep_ws, size_t sep_ws_bytes,
                          int64_t cap_b, int64_t cap_c, float* g_out, dmtz_edit* edits, int64_t edits_capacity,
                          int64_t* n_edits, dmtz_stats* st, dmtz_sloop_stats* ss, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !f || !fhat || !o || !workspace || !g_out || !n_edits || !st || !ss ||
      (edits_capacity > 0 && !edits) || edits_capacity < 0 || cap_b < 0 || cap_c < 0) {
    set_err("NULL argument");
    return DMTZ_E_ARG;
  }
  memset(ss, 0, sizeof *ss);
  if (o->tier >= 1 && o->tier <= 2)
    return dmtz_correct(c, f, fhat, o, workspace, workspace_bytes, g_out, edits, edits_capacity, n_edits, st, stream);
  memset(st, 0, sizeof *st);
  *n_edits = 0;
  if (!(o->xi > 0.0f) || !isfinite(o->xi) || o->q_max < 0 || o->q_max > 30 || o->q_cap < 1 ||
      o->q_cap > 65535 || o->tier < 3 || o->tier > 5 || o->max_rounds < 0) {
    set_err("invalid options (xi=%g q_max=%d q_cap=%d tier=%d)", (double)o->xi, o->q_max, o->q_cap, o->tier);
    st->status = DMTZ_E_ARG;
    return DMTZ_E_ARG;
  }
  Layout L = layout_for(c);
  if (workspace_bytes < L.total) {
    set_err("workspace %zu < %zu bytes", workspace_bytes, L.total);
    st->status = DMTZ_E_OOM;
    return DMTZ_E_OOM;
  }
  if (c->g.N >= (1ll << 32)) { set_err("tiers 3-5 need fewer than 2^32 vertices per context"); return DMTZ_E_DIMS; }
  const size_t need = sep_layout(c, o->tier, cap_b, cap_c).total;
  if (!sep_ws || sep_ws_bytes < need) {
    set_err("separatrix workspace %zu < %zu bytes", sep_ws_bytes, need);
    st->status = DMTZ_E_OOM;
    return DMTZ_E_OOM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  dmtz_status r;
  if (c->D == 3)
    r = preserve_impl<3>(c, f, fhat, o, (char*)workspace, L, (char*)sep_ws, cap_b, cap_c, g_out, edits,
                         edits_capacity, n_edits, st, ss, s);
  else
    r = preserve_impl<2>(c, f, fhat, o, (char*)workspace, L, (char*)sep_ws, cap_b, cap_c, g_out, edits,
                         edits_capacity, n_edits, st, ss, s);
  if (r == DMTZ_E_CUDA) st->status = r;
  return r;
}


size_t dmtz_edit_stream_bound(int64_t n) {
  if (n < 0) return 0;
  const size_t nb = (size_t)((n + EC_BLOCK - 1) / EC_BLOCK);
  return EC_HEADER + 8 * nb + (size_t)n * (10 + 3 + 5);
}

dmtz_status dmtz_encode_edits(dmtz_ctx* c, const dmtz_edit* edits, int64_t n, float xi, int32_t q_max,
                              const float* fhat, void* ws, size_t wsb, uint8_t* out, size_t cap, size_t* nbytes,
                              dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || (n > 0 && !edits) || !ws || !out || !nbytes || n < 0) { set_err("NULL argument"); return DMTZ_E_ARG; }
  if (n > c->g.N) { set_err("%lld edits for %lld vertices", (long long)n, (long long)c->g.N); return DMTZ_E_ARG; }
  const Layout L = layout_for(c);
  if (wsb < L.total) { set_err("workspace %zu < %zu bytes", wsb, L.total); return DMTZ_E_OOM; }
  cudaStream_t s = (cudaStream_t)stream;
  char* w = (char*)ws;
  long long* len = (long long*)(w + L.cand_g);
  unsigned long long* bsum = (unsigned long long*)(w + L.edit_bc);
  Counters* dc = (Counters*)(w + L.counters);
  Counters* hc = c->host_cnt;
  CK(cudaMemsetAsync(dc, 0, sizeof(Counters), s));
  k_ec_len<<<clamp_blocks(n + 1, 256), 256, 0, s>>>((const EditRec*)edits, n, fhat, len, &dc->pad[1]);
  CK(cudaGetLastError());
  CK(scan_i64(len, n + 1, bsum, &dc->pad[0], &hc->pad[0], s));  // synchronises: hc->pad[0] = payload bytes
  CK(cudaMemcpyAsync(&hc->pad[1], &dc->pad[1], 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hc->pad[1]) { set_err("edit list not strictly ascending"); return DMTZ_E_ARG; }
  const size_t nb = (size_t)((n + EC_BLOCK - 1) / EC_BLOCK);
  *nbytes = EC_HEADER + 8 * nb + (size_t)hc->pad[0];
  if (*nbytes > cap) { set_err("edit stream needs %zu bytes", *nbytes); return DMTZ_E_CAPACITY; }
  k_ec_write<<<clamp_blocks(n > 0 ? n : 1, 256), 256, 0, s>>>((const EditRec*)edits, n, len, xi, q_max, fhat, out);
  CK(cudaGetLastError());
  return DMTZ_OK;
}

dmtz_status dmtz_decode_edits(dmtz_ctx* c, const uint8_t* in, size_t nbytes, const float* fhat, dmtz_edit* edits,
                              int64_t cap, int64_t* n_edits, float* xi, int32_t* q_max, void* ws, size_t wsb,
                              dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !in || !n_edits || !xi || !q_max || !ws || cap < 0 || (cap > 0 && !edits)) {
    set_err("NULL argument");
    return DMTZ_E_ARG;
  }
  if (nbytes < EC_HEADER) { set_err("edit stream of %zu bytes", nbytes); return DMTZ_E_ARG; }
  const Layout L = layout_for(c);
  if (wsb < L.total) { set_err("workspace %zu < %zu bytes", wsb, L.total); return DMTZ_E_OOM; }
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t h[EC_HEADER];
  CK(cudaMemcpyAsync(h, in, EC_HEADER, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  auto u32 = [&](int o) { uint32_t x = 0; for (int k = 0; k < 4; k++) x |= (uint32_t)h[o + k] << (8 * k); return x; };
  uint64_t n = 0;
  for (int k = 0; k < 8; k++) n |= (uint64_t)h[8 + k] << (8 * k);
  const uint32_t ver = u32(4), blk = u32(16), nblocks = u32(28), xib = u32(24);
  if (ver == 2 && !fhat) { set_err("a version-2 edit stream needs fhat"); return DMTZ_E_ARG; }
  if (memcmp(h, "DMTE", 4) != 0 || (ver != 1 && ver != 2) || blk != (uint32_t)EC_BLOCK ||
      (uint64_t)nblocks != (n + EC_BLOCK - 1) / EC_BLOCK || EC_HEADER + 8 * (size_t)nblocks > nbytes) {
    set_err("not a version-1/2 edit stream");
    return DMTZ_E_ARG;
  }
  *n_edits = (int64_t)n;
  memcpy(xi, &xib, 4);
  *q_max = (int32_t)u32(20);
  if ((int64_t)n > cap) { set_err("stream holds %llu edits", (unsigned long long)n); return DMTZ_E_CAPACITY; }
  Counters* dc = (Counters*)((char*)ws + L.counters);
  Counters* hc = c->host_cnt;
  CK(cudaMemsetAsync(&dc->pad[1], 0, 8, s));
  if (nblocks && ver == 2 && !getenv("DMTZ_EC_DECODE_THREAD"))   // one warp per block
    k_ec_decode_v2w<<<clamp_blocks(nblocks * 32, 128), 128, 0, s>>>(in, nbytes, (int64_t)n, nblocks, c->g.N, fhat,
                                                                    (EditRec*)edits, &dc->pad[1]);
  else if (nblocks)   // version 1 (raw value bytes): one thread per block
    k_ec_decode<<<clamp_blocks(nblocks, 128), 128, 0, s>>>(in, nbytes, (int64_t)n, nblocks, c->g.N,
                                                           ver == 2 ? fhat : nullptr, (EditRec*)edits, &dc->pad[1]);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&hc->pad[1], &dc->pad[1], 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hc->pad[1]) { set_err("malformed edit stream (%llu bad blocks)", hc->pad[1]); return DMTZ_E_ARG; }
  return DMTZ_OK;
}

dmtz_status dmtz_apply_edits(dmtz_ctx* c, const float* fhat, float xi, int32_t q_max, const dmtz_edit* edits,
                             int64_t n, float* g_out, void* ws, size_t wsb, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !fhat || !g_out || !ws || n < 0 || (n > 0 && !edits) || !(xi > 0.0f) || q_max < 0 || q_max > 30) {
    set_err("invalid argument");
    return DMTZ_E_ARG;
  }
  const Layout L = layout_for(c);
  if (wsb < L.total) { set_err("workspace %zu < %zu bytes", wsb, L.total); return DMTZ_E_OOM; }
  cudaStream_t s = (cudaStream_t)stream;
  Counters* dc = (Counters*)((char*)ws + L.counters);
  Counters* hc = c->host_cnt;
  CK(cudaMemsetAsync(&dc->pad[1], 0, 8, s));
  if (g_out != fhat) CK(cudaMemcpyAsync(g_out, fhat, (size_t)c->g.N * 4, cudaMemcpyDeviceToDevice, s));
  if (n > 0)
    k_apply_edits<<<clamp_blocks(n, 256), 256, 0, s>>>(fhat, (const EditRec*)edits, n, c->g.N, ldexpf(xi, -q_max),
                                                       g_out, &dc->pad[1]);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(&hc->pad[1], &dc->pad[1], 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hc->pad[1]) { set_err("%llu edits outside the grid", hc->pad[1]); return DMTZ_E_ARG; }
  return DMTZ_OK;
}


dmtz_status dmtz_critical_prf(dmtz_ctx* c, const uint32_t* a, const uint32_t* b, dmtz_prf* out, void* ws,
                              size_t wsb, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !a || !b || !out || !ws) { set_err("NULL argument"); return DMTZ_E_ARG; }
  const Layout L = layout_for(c);
  if (wsb < L.total) { set_err("workspace %zu < %zu bytes", wsb, L.total); return DMTZ_E_OOM; }
  cudaStream_t s = (cudaStream_t)stream;
  Counters* dc = (Counters*)((char*)ws + L.counters);
  Counters* hc = c->host_cnt;
  CK(cudaMemsetAsync(dc->pad, 0, 3 * 8, s));
  k_crit_prf<<<clamp_blocks(c->g.N, 256), 256, 0, s>>>(a, b, c->g.N, dc->pad);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hc->pad, dc->pad, 3 * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out->n_orig = (int64_t)hc->pad[0];
  out->n_rec = (int64_t)hc->pad[1];
  out->n_match = (int64_t)hc->pad[2];
  return DMTZ_OK;
}

dmtz_status dmtz_separatrix_prf(dmtz_ctx* c, const dmtz_seps* A, int64_t na, const dmtz_seps* B, int64_t nb,
                                dmtz_prf* out, void* ws, size_t wsb, dmtz_stream_t stream) {
  DeviceGuard dg_(c);
  if (!c || !A || !B || !out || !ws || na < 0 || nb < 0) { set_err("NULL argument"); return DMTZ_E_ARG; }
  const Layout L = layout_for(c);
  if (wsb < L.total) { set_err("workspace %zu < %zu bytes", wsb, L.total); return DMTZ_E_OOM; }
  cudaStream_t s = (cudaStream_t)stream;
  Counters* dc = (Counters*)((char*)ws + L.counters);
  Counters* hc = c->host_cnt;
  CK(cudaMemsetAsync(dc->pad, 0, 8, s));
  if (na > 0 && nb > 0)
    k_sep_match<<<clamp_blocks(na, 256), 256, 0, s>>>(
        (const long long*)A->branch_offsets, A->cells, A->origin, A->terminal, A->kind, na,
        (const long long*)B->branch_offsets, B->cells, B->origin, B->terminal, B->kind, nb, dc->pad);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hc->pad, dc->pad, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out->n_orig = na;
  out->n_rec = nb;
  out->n_match = (int64_t)hc->pad[0];
  return DMTZ_OK;
}

dmtz_status dmtz_local_slab(int64_t nz, int world, int rank, int64_t* z0, int64_t* z1, int64_t* lz0, int64_t* lz1) {
  if (!z0 || !z1 || !lz0 || !lz1) { set_err("NULL argument"); return DMTZ_E_ARG; }
  const dmtz_status r = local_slab(nz, world, rank, z0, z1, lz0, lz1);
  if (r) set_err("%lld planes cannot be split over %d ranks (rank %d)", (long long)nz, world, rank);
  return r;
}

dmtz_status dmtz_ctx_set_transport(dmtz_ctx* c, const dmtz_transport* t) {
  if (!c) { set_err("NULL argument"); return DMTZ_E_ARG; }
  if (c->nccl_comm) { set_err("the context owns an NCCL communicator"); return DMTZ_E_ARG; }
  if (!t) {
    c->has_tr = 0;
    return DMTZ_OK;
  }
  if (!t->exchange || !t->allreduce_sum_i64) { set_err("transport without callbacks"); return DMTZ_E_ARG; }
  c->tr = *t;
  c->has_tr = 1;
  return DMTZ_OK;
}

dmtz_status dmtz_ctx_set_dist_graph(dmtz_ctx* c, int on, int* used_last) {
  if (!c) { set_err("NULL argument"); return DMTZ_E_ARG; }
  if (used_last) *used_last = c->dist_graph_used;
  if (on >= 0) c->dist_graph = on ? 1 : 0;
  return DMTZ_OK;
}

dmtz_status dmtz_ctx_set_dist_sync(dmtz_ctx* c, int rounds_per_sync) {
  if (!c || rounds_per_sync < 1 || rounds_per_sync > 1024) { set_err("invalid argument"); return DMTZ_E_ARG; }
  c->dist_sync = rounds_per_sync;
  return DMTZ_OK;
}

dmtz_status dmtz_nccl_unique_id(void* out) {
  if (!out) { set_err("NULL argument"); return DMTZ_E_ARG; }
  NcclApi* A = nccl_api();
  if (!A) { set_err("libnccl.so.2 cannot be loaded"); return DMTZ_E_NCCL; }
  ncclUniqueId id;
  if (A->GetUniqueId(&id) != ncclSuccess) { set_err("ncclGetUniqueId failed"); return DMTZ_E_NCCL; }
  memcpy(out, &id, sizeof id);
  return DMTZ_OK;
}

}  // extern "C"
