// dmtz_api.cu -- the C ABI of include/dmtz.h on top of dmtz_kernels.cuh.
//
// Host side of the hot path: workspace carving, the fixed-point driver of the
// C-loop (repeat gradient -> classify -> fix until no false
// critical cell), status/error plumbing.  No device allocation happens here:
// every buffer is the caller's.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <utility>

#include "../../include/dmtz.h"
#include "dmtz_kernels.cuh"
#include "dmtz_sweep.cuh"
#include "dmtz_trace.cuh"

using namespace dmtz;

struct dmtz_ctx {
  dmtz_dims dims;
  Grid g;
  int D;
  int device;
  int rank, world;
  Counters* host_cnt;  // pinned
  cudaEvent_t ev[3];   // sweep timing (opts.profile): screen | decode
  int verbose;         // DMTZ_VERBOSE=1: per-round counters on stderr
};

namespace {

thread_local char g_err[512] = "";

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
  size_t cand_f, cand_g, crit_f, crit_g, lowpos, lb, state, tbits, counters, edit_bc, ebits, fmark, units, frontier, trace,
      total;
  int64_t fwords;  // frontier bitmap words (one bit per row-block unit)
};

Layout layout_for(const dmtz_ctx* c) {
  const size_t N = (size_t)c->g.N;
  const size_t cs = c->D == 3 ? 8 : 2;
  Layout L;
  size_t o = 0;
  L.cand_f = o; o += align_up(N * cs);
  // u64 even in 2D: the trace reuses it as int64 scratch (>= 1 MiB for small grids)
  L.cand_g = o; o += align_up(N * 8 > (size_t)(1 << 20) ? N * 8 : (size_t)(1 << 20));
  L.crit_f = o; o += align_up(N * 4);
  L.crit_g = o; o += align_up(N * 4);
  // lowpos doubles as the trace's connector-BFS scratch: at least 128 slots of 3 x 1024 words
  L.lowpos = o; o += align_up(N * 8 > (size_t)128 * 3072 * 8 ? N * 8 : (size_t)128 * 3072 * 8);
  L.lb = o; o += align_up(N * 4);
  L.state = o; o += align_up(N * 4);
  L.tbits = o; o += align_up((N + 31) / 32 * 4 + 64);
  L.counters = o; o += align_up(sizeof(Counters) * 2);
  L.edit_bc = o; o += align_up(((N + EDIT_CHUNK - 1) / EDIT_CHUNK + 2) * 8);
  const RowGeom rg = row_geom(c->g);
  L.fwords = (rg.units + 31) / 32;
  L.ebits = o; o += align_up((size_t)(c->g.nz * c->g.ny * rg.wpr) * 4 + 64);
  L.fmark = o; o += align_up((size_t)(c->g.nz * c->g.ny * rg.wpr) * 4 + 64);
  L.units = o; o += align_up((size_t)rg.units * 4);
  L.frontier = o; o += align_up(L.fwords * 4 + 64);
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
  if (tier == 2) return 0xFFFFFFFFu;
  // dims 0 and top only
  return D == 3 ? (1u | (0x3Fu << 20)) : (1u | (0x3u << 4));
}

template <int D>
dmtz_status correct_impl(dmtz_ctx* c, const float* f, const float* fhat, const dmtz_correct_opts* o,
                         char* ws, const Layout& L, float* g_out, dmtz_edit* edits, int64_t cap,
                         int64_t* n_edits, dmtz_stats* st, cudaStream_t s) {
  const Grid& g = c->g;
  using code_t = typename Tr<D>::code_t;
  code_t* cand_f = (code_t*)(ws + L.cand_f);
  code_t* cand_g = (code_t*)(ws + L.cand_g);  // codes of g, memoized across rounds
  float* lb = (float*)(ws + L.lb);
  uint32_t* state = (uint32_t*)(ws + L.state);
  uint32_t* tbits = (uint32_t*)(ws + L.tbits);
  Counters* dc = (Counters*)(ws + L.counters);
  unsigned long long* bc = (unsigned long long*)(ws + L.edit_bc);
  Counters* hc = c->host_cnt;
  const int64_t nwords = (g.N + 31) / 32;
  const int ethreads = 256;
  const int eblocks = (int)((g.N + ethreads - 1) / ethreads < 148 * 32 ? (g.N + ethreads - 1) / ethreads : 148 * 32);
  const int wblocks = (int)((nwords + ethreads - 1) / ethreads < 148 * 32 ? (nwords + ethreads - 1) / ethreads : 148 * 32);

  // a1: setup
  CK(cudaMemsetAsync(dc, 0, sizeof(Counters), s));
  CK(cudaMemsetAsync(&dc->first_nonfinite, 0xFF, 16, s));
  CK(cudaMemsetAsync(tbits, 0, nwords * 4, s));
  k_setup<<<eblocks, ethreads, 0, s>>>(f, fhat, o->xi, g.N, lb, g_out, state, dc);
  st->launches++;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hc->first_nonfinite != ~0ull) {
    set_err("non-finite value at vertex %llu", hc->first_nonfinite);
    st->status = DMTZ_E_NONFINITE;
    return DMTZ_E_NONFINITE;
  }
  if (hc->first_bound != ~0ull) {
    set_err("|fhat - f| > xi at vertex %llu", hc->first_bound);
    st->status = DMTZ_E_BOUND;
    return DMTZ_E_BOUND;
  }
  // a2: reference gradient of f (once)
  launch_codes<D>(g, f, cand_f, 0, g.nz, s);
  uint32_t* crit_f = (uint32_t*)(ws + L.crit_f);
  k_critmask<D><<<anchor_grid(g, 0, g.nz, 128), 128, 0, s>>>(cand_f, crit_f, g);
  unsigned long long* lowpos = (unsigned long long*)(ws + L.lowpos);
  k_lowpos<D><<<anchor_grid(g, 0, g.nz, 128), 128, 0, s>>>(f, lowpos, g);
  st->launches += 3;
  CK(cudaGetLastError());

  const float step = ldexpf(o->xi, -o->q_max);   // xi / 2^q_max, exact
  const int64_t max_rounds = o->max_rounds > 0 ? o->max_rounds : g.N * (int64_t)(o->q_cap + 1);
  const uint32_t tmask = tier_mask<D>(o->tier);
  const RowGeom rg = row_geom(g);
  uint32_t* ebits = (uint32_t*)(ws + L.ebits);
  uint32_t* fmark = (uint32_t*)(ws + L.fmark);
  uint32_t* crit_g = (uint32_t*)(ws + L.crit_g);
  const size_t rowbit_bytes = (size_t)(g.nz * g.ny * rg.wpr) * 4;
  CK(cudaMemsetAsync(fmark, 0, rowbit_bytes, s));
  uint32_t* units = (uint32_t*)(ws + L.units);
  uint32_t* fbits = (uint32_t*)(ws + L.frontier);
  unsigned long long* n_units = &dc->n_units;
  const bool frontier_mode = !o->full_sweeps;
  const int fwords_smem = L.fwords * 4 <= 32768 ? (int)L.fwords : 0;
  const int sweep_blocks = 148 * 8;
  // round 1 (and every round of a full sweep) processes every unit
  k_units_all<<<(unsigned)((rg.units + 255) / 256 < 4096 ? (rg.units + 255) / 256 : 4096), 256, 0, s>>>(
      rg.units, units, n_units);
  st->launches++;
  dmtz_status status = DMTZ_OK;
  for (int64_t round = 1;; round++) {
    // a3: gradient of g (screened);  a4/a5: classify + mark targets;  a6: edit;  a7: frontier
    CK(cudaMemsetAsync(dc, 0, offsetof(Counters, first_nonfinite), s));
    if (frontier_mode) CK(cudaMemsetAsync(fbits, 0, L.fwords * 4, s));
    if (frontier_mode && round > 1) CK(cudaMemsetAsync(ebits, 0, rowbit_bytes, s));
    if (o->profile) CK(cudaEventRecord(c->ev[0], s));
    k_screen<D><<<sweep_blocks, 256, 0, s>>>(g_out, cand_g, ebits, units, n_units, g, rg, round == 1 ? 1 : 0, dc);
    if (o->profile) CK(cudaEventRecord(c->ev[1], s));
    k_decode<D><<<sweep_blocks * 2, DECODE_THREADS, 0, s>>>(f, cand_f, crit_f, cand_g, crit_g, ebits, fmark, tbits, units, n_units,
                                             g, rg, tmask, lowpos, round == 1 ? 1 : 0, dc);
    if (o->profile) CK(cudaEventRecord(c->ev[2], s));
    k_edit_rows<D><<<wblocks, ethreads, frontier_mode ? fwords_smem * 4 : 0, s>>>(
        tbits, nwords, fhat, lb, g_out, state, dc, step, o->q_cap, frontier_mode ? fbits : nullptr, g, rg,
        frontier_mode ? fwords_smem : 0);
    st->launches += 3;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(hc, dc, offsetof(Counters, first_nonfinite), cudaMemcpyDeviceToHost, s));
    if (frontier_mode) {
      // next round's unit list (after the counters were copied: n_units is reset here)
      CK(cudaMemsetAsync(n_units, 0, 8, s));
      k_units_from_bits<<<(unsigned)((rg.units + 255) / 256 < 4096 ? (rg.units + 255) / 256 : 4096), 256, 0, s>>>(
          fbits, rg.units, units, n_units);
      st->launches++;
    }
    CK(cudaStreamSynchronize(s));
    if (o->profile) {
      float ms0 = 0.f, ms1 = 0.f;
      CK(cudaEventElapsedTime(&ms0, c->ev[0], c->ev[1]));
      CK(cudaEventElapsedTime(&ms1, c->ev[1], c->ev[2]));
      st->sweep_ms += ms0 + ms1;
      st->screen_ms += ms0;
      st->decode_ms += ms1;
      if (ms0 > 0 && (int64_t)hc->n_swept == g.N) { st->screen_ms_full += ms0; st->n_screen_full++; }
    }
    st->sweeps++;
    st->anchors_swept += (int64_t)hc->n_swept;
    if (c->verbose)
      fprintf(stderr, "dmtz round %lld: swept %llu false %llu targets %llu changed %llu\n", (long long)round,
              hc->n_swept, hc->n_false, hc->n_targets, hc->n_changed);
    if (hc->n_internal) {
      set_err("gradient invariant violated at %llu false cells (round %lld)", hc->n_internal, (long long)round);
      status = DMTZ_E_INTERNAL;
      break;
    }
    if (round == 1) {
      st->n_false_round0 = (int64_t)hc->n_false;
      for (int k = 0; k < 8; k++) st->false_by_kind_round0[k] = (int64_t)hc->kinds[k];
    }
    if (hc->n_false == 0) break;
    st->rounds = round;
    if (hc->n_changed == 0) { status = DMTZ_E_STUCK; set_err("no target could move (round %lld)", (long long)round); break; }
    if (round == max_rounds) { status = DMTZ_E_ITER_CAP; set_err("round cap %lld reached", (long long)round); break; }
  }
  // a8: edit list
  const int64_t nb = (g.N + EDIT_CHUNK - 1) / EDIT_CHUNK;
  CK(cudaMemsetAsync(&dc->n_lossless, 0, 8, s));
  k_edit_count<<<(unsigned)nb, EDIT_THREADS, 0, s>>>(state, g.N, bc, dc);
  k_scan_counts<<<1, EDIT_THREADS, 0, s>>>(bc, nb, dc);
  k_edit_write<<<(unsigned)nb, EDIT_THREADS, 0, s>>>(state, g_out, g.N, bc, (EditOut*)edits, cap);
  st->launches += 3;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *n_edits = (int64_t)hc->n_edits;
  st->n_edited = *n_edits;
  st->n_lossless = (int64_t)hc->n_lossless;
  st->n_quantized = st->n_edited - st->n_lossless;
  if (status == DMTZ_OK && *n_edits > cap) { status = DMTZ_E_CAPACITY; set_err("edit list needs %lld entries", (long long)*n_edits); }
  st->status = status;
  return status;
}

}  // namespace

extern "C" {

int dmtz_version(void) { return 1; }

const char* dmtz_last_error(void) { return g_err; }

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
  if (world != 1 || rank != 0 || nccl_id != nullptr) { set_err("world must be 1 (slab layer drives per-rank contexts)"); return DMTZ_E_ARG; }
  CK(cudaSetDevice(cuda_device));
  dmtz_ctx* c = new (std::nothrow) dmtz_ctx();
  if (!c) return DMTZ_E_OOM;
  c->dims = *d;
  c->g.nx = d->nx; c->g.ny = d->ny; c->g.nz = d->nz;
  c->g.N = d->nx * d->ny * d->nz;
  c->g.sy = d->nx; c->g.sz = d->nx * d->ny;
  c->D = d->nz == 1 ? 2 : 3;
  c->device = cuda_device;
  c->rank = rank; c->world = world;
  const char* vb = getenv("DMTZ_VERBOSE");
  c->verbose = vb && vb[0] == '1';
  cudaError_t e = cudaMallocHost((void**)&c->host_cnt, sizeof(Counters) * 2);
  if (e != cudaSuccess) { delete c; set_err("cudaMallocHost: %s", cudaGetErrorString(e)); return DMTZ_E_CUDA; }
  for (int i = 0; i < 3; i++) {
    e = cudaEventCreate(&c->ev[i]);
    if (e != cudaSuccess) { set_err("cudaEventCreate: %s", cudaGetErrorString(e)); return DMTZ_E_CUDA; }
  }
  *out = c;
  return DMTZ_OK;
}

void dmtz_ctx_destroy(dmtz_ctx* c) {
  if (!c) return;
  cudaFreeHost(c->host_cnt);
  for (int i = 0; i < 3; i++) cudaEventDestroy(c->ev[i]);
  delete c;
}

size_t dmtz_workspace_bytes(const dmtz_ctx* c, const dmtz_correct_opts*) {
  if (!c) return 0;
  return layout_for(c).total;
}

dmtz_status dmtz_compute_gradient(dmtz_ctx* c, const float* field, void* codes, void*, dmtz_stream_t stream) {
  if (!c || !field || !codes) { set_err("NULL argument"); return DMTZ_E_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  if (c->D == 3) launch_codes<3>(c->g, field, codes, 0, c->g.nz, s);
  else launch_codes<2>(c->g, field, codes, 0, c->g.nz, s);
  CK(cudaGetLastError());
  return DMTZ_OK;
}

dmtz_status dmtz_critical_mask(dmtz_ctx* c, const void* codes, uint32_t* crit, dmtz_stream_t stream) {
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
  if (c->D == 3) r = correct_impl<3>(c, f, fhat, o, (char*)workspace, L, g_out, edits, edits_capacity, n_edits, st, s);
  else r = correct_impl<2>(c, f, fhat, o, (char*)workspace, L, g_out, edits, edits_capacity, n_edits, st, s);
  if (r == DMTZ_E_CUDA) st->status = r;
  return r;
}

dmtz_status dmtz_trace_separatrices(dmtz_ctx* c, const void* codes, uint32_t kinds, void* workspace,
                                    size_t workspace_bytes, dmtz_seps* out, int64_t cap_b, int64_t cap_c,
                                    int64_t* n_b, int64_t* n_c, dmtz_stream_t stream) {
  if (!c || !codes || !workspace || !out || !n_b || !n_c || cap_b < 0 || cap_c < 0) {
    set_err("NULL argument");
    return DMTZ_E_ARG;
  }
  Layout L = layout_for(c);
  if (workspace_bytes < L.total) { set_err("workspace %zu < %zu bytes", workspace_bytes, L.total); return DMTZ_E_OOM; }
  char* ws = (char*)workspace;
  TraceArgs a;
  a.g = c->g;
  a.codes = codes;
  a.kinds = kinds;
  a.pre = (long long*)(ws + L.cand_g);
  a.pre_bytes = L.crit_f - L.cand_g;
  a.bfs = (unsigned long long*)(ws + L.lowpos);
  a.bfs_bytes = L.lb - L.lowpos;  // the lowpos region, which lb follows
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
  cudaError_t e = c->D == 3 ? run_trace<3>(a, (cudaStream_t)stream) : run_trace<2>(a, (cudaStream_t)stream);
  if (e != cudaSuccess) { set_err("trace: %s", cudaGetErrorString(e)); return DMTZ_E_CUDA; }
  *n_b = a.n_branches;
  *n_c = a.n_cells;
  if (a.n_internal) { set_err("trace: cycle or inconsistent gradient"); return DMTZ_E_INTERNAL; }
  if (a.n_branches > cap_b || a.n_cells > cap_c) { set_err("trace needs %lld branches / %lld cells", (long long)a.n_branches, (long long)a.n_cells); return DMTZ_E_CAPACITY; }
  return DMTZ_OK;
}

}  // extern "C"
