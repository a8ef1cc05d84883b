/*
 * include/dmtz.h -- C ABI of the B200-native DMTz hot path (libdmtz.so).
 *
 * DMTz (arXiv 2409.17346) preserves the discrete Morse-Smale complex of a 2D/3D
 * scalar field under error-bounded lossy compression by editing the
 * decompressed field.  This library implements its data-parallel hot path on
 * sm_100a: the discrete gradient, the
 * critical-cell correction loop "C-loop" with quantized edits, and
 * the V-path separatrix traces the S-loop checks.
 * P:<n> cites line n of the paper text; DESIGN.md §3 lists every reading taken
 * where the paper is silent or garbled.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless marked (host).  The caller owns
 *     every buffer; the library never allocates device memory (scratch comes
 *     from the caller's workspace, sized by dmtz_workspace_bytes).
 *   - Fields are float32, x fastest: v = x + nx*(y + ny*z).  nz == 1 means 2D.
 *   - Calls are asynchronous on the given stream, except dmtz_correct and
 *     dmtz_trace_separatrices, which synchronise the stream to read counters
 *     and write their host outputs before returning.
 *   - No exception crosses the ABI; every call returns a dmtz_status.  Details of
 *     the last failure on the calling thread: dmtz_last_error().
 *
 * Cell complex (reading A1): the Freudenthal/Kuhn triangulation of
 * the grid.  Every cell is identified by its anchor (its lowest-index vertex)
 * and a TYPE: the chain 0 = m0 < m1 < ... < md of nested bit masks (dx = 1,
 * dy = 2, dz = 4) of its vertex offsets.  Types are numbered by dimension, then
 * lexicographically by the mask tuple:
 *   3D (26 types): vertex 0; edges 1..7 (masks 1..7); triangles 8..19
 *     ((1,3)(1,5)(1,7)(2,3)(2,6)(2,7)(3,7)(4,5)(4,6)(4,7)(5,7)(6,7));
 *     tetrahedra 20..25 ((1,3,7)(1,5,7)(2,3,7)(2,6,7)(4,5,7)(4,6,7)).
 *   2D (6 types): vertex 0; edges 1..3 (masks 1,2,3); triangles 4,5 ((1,3),(2,3)).
 * The LINK of a cell is the set of vertices w such that cell + {w} is a cell of
 * the unbounded grid; its SLOTS are the link vertices in ascending global index
 * ((dz,dy,dx) lexicographic) order.
 *
 * Gradient codes: cell a is paired with the cofacet
 * a + {w} ("a -> w") or is not paired upward.  One code per anchor:
 *   3D uint64: bits 0-3 vertex slot (15 = none), edge type k (1..7) at
 *              4 + 3(k-1) (7 = none), triangle type k (8..19) at 25 + 2(k-8)
 *              (3 = none); bits 49-63 zero.
 *   2D uint16: bits 0-2 vertex slot (7 = none), edge type k (1..3) at
 *              3 + 2(k-1) (3 = none); bits 9-15 zero.
 * A cell is CRITICAL iff it exists (all its vertices lie in the grid), it is
 * not paired upward, and no facet is paired with it.  Critical masks are
 * uint32 per anchor, bit t = type t critical.
 *
 * Cell ids (trace output): (dim << 56) | (anchor * T_dim + index of the type
 * within its dimension), T_dim = 1/7/12/6 (3D), 1/3/2 (2D).
 */
#ifndef DMTZ_H
#define DMTZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dmtz_stream_t; /* a cudaStream_t; NULL = legacy default stream */

typedef enum {
  DMTZ_OK = 0,
  DMTZ_E_ARG = 1,       /* bad argument (NULL pointer, xi <= 0, q_max/q_cap/tier out of range) */
  DMTZ_E_DIMS = 2,      /* nx < 2 or ny < 2 or nz < 1 */
  DMTZ_E_NONFINITE = 3, /* NaN/Inf in f or fhat; dmtz_last_error names the first index */
  DMTZ_E_BOUND = 4,     /* |fhat - f| > xi somewhere; first index in dmtz_last_error */
  DMTZ_E_CAPACITY = 5,  /* output buffer too small; the needed count is still returned */
  DMTZ_E_ITER_CAP = 6,  /* max_rounds reached with false cells left */
  DMTZ_E_STUCK = 7,     /* false cells left but every target is already at its lower bound
                           (reading A10: f32 lower bounds can merge distinct values) */
  DMTZ_E_CUDA = 8,      /* a CUDA runtime error; message in dmtz_last_error */
  DMTZ_E_NCCL = 9,      /* reserved for the multi-GPU layer */
  DMTZ_E_OOM = 10,      /* workspace smaller than dmtz_workspace_bytes */
  DMTZ_E_INTERNAL = 11  /* an invariant of the gradient did not hold (never expected) */
} dmtz_status;

typedef struct { int64_t nx, ny, nz; } dmtz_dims;

typedef struct {
  float xi;            /* absolute error bound xi > 0; relative -> absolute is the caller's */
  int32_t q_max;       /* edit step xi / 2^q_max, 0..30 (default 6) */
  int32_t q_cap;       /* max quantized steps per vertex, 1..65535; the paper's literal
                          "q < q_max" is q_cap = q_max (reading A6) */
  int32_t tier;        /* 1: extrema only (dims 0 and top), 2: all critical cells */
  int64_t max_rounds;  /* 0 = N * (q_cap + 1), the bound of the progress argument */
  int32_t full_sweeps; /* 1: reference mode -- every round recomputes the code of every anchor and
                          classifies every anchor; 0 (default): only the dirty frontier, and within
                          it only codes whose 3x3x3 box changed (exact, bit-identical) */
  int32_t profile;     /* 1: time each round's sweep with CUDA events on `stream` (stats.sweep_ms) */
} dmtz_correct_opts;

/* One edited vertex: quantized (g = RN(fhat - RN(q * xi/2^q_max))) or
 * lossless (g = the lower bound, stored as its float bits in `value`). */
typedef struct {
  uint64_t v;        /* global vertex index */
  uint16_t q;        /* quantized steps taken (for lossless entries: steps before the clamp) */
  uint8_t lossless;  /* 1 = value is stored losslessly */
  uint8_t pad;
  float value;       /* final edited value g_v (bit-exact) */
} dmtz_edit;         /* 16 bytes; edit lists are sorted by v */

typedef struct {
  int64_t rounds;          /* C-loop rounds that found false cells (and edited) */
  int64_t n_edited, n_quantized, n_lossless;
  int64_t n_false_round0;  /* false critical cells before any edit */
  int64_t false_by_kind_round0[8]; /* FPmin FNmin FP1s FN1s FP2s FN2s FPmax FNmax */
  int32_t status;
  int32_t pad;
  int64_t sweeps;          /* gradient evaluations of g (rounds + 1 on success) */
  int64_t anchors_swept;   /* sum over sweeps of anchors evaluated (frontier accounting) */
  int64_t launches;        /* kernels this call launched */
  double sweep_ms;         /* opts.profile: summed device time of the round sweeps (screen + decode) */
  double screen_ms;        /* opts.profile: of which the gradient screening kernel */
  double decode_ms;        /* opts.profile: of which the classification / target kernel */
  double screen_ms_full;   /* opts.profile: screening time of the rounds that recomputed every code */
  int64_t n_screen_full;   /* number of such rounds */
  int64_t anchors_recomputed; /* sum over sweeps of anchors whose code was recomputed (the rest
                                 provably kept theirs: no vertex of their 3x3x3 box changed) */
  int64_t anchors_decoded;    /* sum over sweeps of anchors whose criticality was decoded (a code of
                                 u + {0,1}^D changed) */
  int64_t cells_evaluated;    /* sum over sweeps of false cells whose target rule was evaluated */
  int64_t anchors_replayed;   /* sum over sweeps of anchors whose unchanged targets were replayed */
  int64_t halo_faces_sent;    /* world > 1: halo faces this rank sent over the rounds */
  int64_t halo_faces_skipped; /* world > 1: faces skipped (no edit touched their 3 planes) */
  double edit_ms;             /* opts.profile: summed k_edit_rows time (Eq. 2 edits + frontier marks) */
} dmtz_stats;

typedef struct dmtz_ctx dmtz_ctx;

/* Create a context for a global grid on `cuda_device` (the device the caller's
 * buffers live on).
 *   world == 1: the whole grid; nccl_unique_id must be NULL.
 *   world > 1 (3D only, multi-GPU C-loop): rank `rank` of
 *     `world` owns the z-planes [z0, z1) of dmtz_local_slab(nz, world, rank, ...); its
 *     dmtz_correct takes and returns the OWNED planes only (f, fhat, g_out are
 *     nx * ny * (z1 - z0) floats) and exchanges halo planes with ranks rank +- 1.
 *     nccl_unique_id (128 bytes, the same on every rank, from dmtz_nccl_unique_id on one
 *     rank) makes the context own an NCCL communicator (libnccl.so.2 is loaded at run
 *     time); NULL leaves the transport to dmtz_ctx_set_transport.
 *   world == 1 with an nccl_unique_id runs the same distributed driver on a one-rank
 *     communicator (one slab, no halos): the NCCL path on one GPU.
 * Errors: DMTZ_E_DIMS (an axis < 2, world > 1 with nz < 3 world or a 2D grid),
 * DMTZ_E_ARG (rank out of range), DMTZ_E_NCCL (NCCL missing or its initialisation
 * failed), DMTZ_E_CUDA. */
dmtz_status dmtz_ctx_create(dmtz_ctx** out, const dmtz_dims* global, int rank, int world,
                            const void* nccl_unique_id, int cuda_device);
void dmtz_ctx_destroy(dmtz_ctx* ctx);

/* The z-slab partition of the multi-GPU C-loop: rank `rank` of `world`
 * owns planes [*z0, *z1) (contiguous, balanced, at least 3 planes each); its local grid
 * is [*lz0, *lz1) = the owned planes plus up to 3 halo planes below and above -- a
 * target lies within [-1, 2]^3 of its false cell's anchor, so the cells that can
 * target owned vertices are anchored in [z0 - 2, z1 + 1) and their criticality reads
 * [z0 - 3, z1 + 3).  Host only; DMTZ_E_ARG if nz < 3 world or rank is out of range. */
dmtz_status dmtz_local_slab(int64_t nz, int world, int rank, int64_t* z0, int64_t* z1, int64_t* lz0, int64_t* lz1);

/* Transport of the multi-GPU C-loop.  Each callback returns 0 on success and must
 * leave the data in place, ordered after the work already enqueued on `stream`, when
 * it returns (an NCCL implementation enqueues on `stream`; a host-staged one
 * synchronises it).  exchange: for i < n, send send_bytes[i] bytes at device pointer
 * send[i] to rank peers[i] and receive recv_bytes[i] bytes from peers[i] into recv[i]
 * (a rank appears at most once per call; both sides post matching pairs).
 * allreduce_sum_i64: sum dev_buf[0 .. n) over all ranks, in place. */
typedef struct {
  void* user;
  int (*exchange)(void* user, int n, const int* peers, const void* const* send, const size_t* send_bytes,
                  void* const* recv, const size_t* recv_bytes, dmtz_stream_t stream);
  int (*allreduce_sum_i64)(void* user, int64_t* dev_buf, int n, dmtz_stream_t stream);
} dmtz_transport;
/* Install (or, with NULL, remove) a transport for a world > 1 context that has no
 * NCCL communicator.  The struct is copied. */
dmtz_status dmtz_ctx_set_transport(dmtz_ctx* ctx, const dmtz_transport* transport);
/* How a world > 1 context's dmtz_correct synchronises with the host (default 8):
 *   rounds_per_sync == 1: every round ends on the host -- the summed counters are read
 *     back, the stop rule runs there, and the next round exchanges only the faces whose
 *     3 planes some edit touched (dmtz_stats.halo_faces_skipped counts the others);
 *   rounds_per_sync  > 1: rounds are enqueued that many at a time with no host
 *     synchronisation between them; the stop rule runs on the device on the all-reduced
 *     counters and sets a stop flag after which the rest of the batch does no work, so
 *     the per-rank round + counter all-reduce + stop decision is one stream of device
 *     work with no host hop; every face is exchanged each round and a face the neighbour
 *     did not change is not applied (halo_faces_skipped stays 0).
 * Results are identical in both modes.  DMTZ_E_ARG outside [1, 1024]. */
dmtz_status dmtz_ctx_set_dist_sync(dmtz_ctx* ctx, int rounds_per_sync);
/* Batched mode over the context's own NCCL communicator with an even rounds_per_sync:
 * on != 0 captures one batch (rounds 2 .. k + 1: exchanges, rounds, counter all-reduce,
 * device stop rule) into a CUDA graph once per dmtz_correct and replays it, one graph
 * launch per k rounds (round 1 runs eagerly; the batch's round-dependent parts repeat
 * with period 2).  If the capture is refused the batches run eagerly.  on < 0 leaves the
 * setting; *used_last (may be NULL) = whether the last dmtz_correct replayed the graph.
 * Default off. */
dmtz_status dmtz_ctx_set_dist_graph(dmtz_ctx* ctx, int on, int* used_last);
/* An NCCL unique id (128 bytes into `out`) for dmtz_ctx_create; DMTZ_E_NCCL if
 * libnccl.so.2 cannot be loaded. */
dmtz_status dmtz_nccl_unique_id(void* out);

/* Bytes of device workspace dmtz_correct / dmtz_compute_gradient / trace need. */
size_t dmtz_workspace_bytes(const dmtz_ctx* ctx, const dmtz_correct_opts* opts);

/* Discrete gradient of `field`: one code per anchor (layout
 * above) into `codes` (uint64[N] in 3D, uint16[N] in 2D).  `field` must be finite
 * (not checked here; dmtz_correct validates).  workspace may be NULL. */
dmtz_status dmtz_compute_gradient(dmtz_ctx* ctx, const float* field, void* codes,
                                  void* workspace, dmtz_stream_t stream);

/* Critical-cell masks (uint32[N], bit t = type t critical) from gradient codes. */
dmtz_status dmtz_critical_mask(dmtz_ctx* ctx, const void* codes, uint32_t* crit,
                               dmtz_stream_t stream);

/* The C-loop with quantized edits (Eq. 2):
 *   validate (finite, |fhat - f| <= xi); lb = RU32(f - xi); g = fhat; q = 0
 *   repeat: F = cells critical in exactly one of gradient(f), gradient(g)
 *           (tier 1: dims 0 and top only); F empty -> OK
 *           T = { target(a) : a in F } (one step per vertex per round, rules
 *           R1/R2/R3a/R3b of DESIGN.md §3); each non-lossless v in T takes one
 *           step g' = RN(fhat - RN((q+1) xi 2^-q_max)) if q+1 <= q_cap and
 *           g' >= lb, else g = lb (lossless); no v changed -> STUCK
 * Outputs: g_out (float[N], device), the sorted edit list (device, capacity
 * edits_capacity entries), *n_edits (host) and *stats (host).  On
 * DMTZ_E_CAPACITY g_out and *n_edits are valid and the list holds the first
 * edits_capacity entries. */
/* Multi-GPU (world > 1 context): call on every rank with its OWNED planes of f, fhat
 * and g_out; the edit list holds the rank's owned edits (global vertex indices,
 * sorted), so the ranks' lists in rank order are the one-GPU list, and g_out the
 * owned planes of the one-GPU g (bit-identical: the rounds are the same synchronous
 * rounds).  Per round: the halo planes a neighbour changed are exchanged (faces whose
 * 3 boundary planes no edit touched are skipped, both sides know it from the previous
 * round's reduction), the round runs on the local grid, and the round counters plus
 * per-face change flags are summed over the ranks; every rank applies the same stop
 * rule.  stats are global (summed over ranks). */
dmtz_status dmtz_correct(dmtz_ctx* ctx, const float* f, const float* fhat,
                         const dmtz_correct_opts* opts, void* workspace, size_t workspace_bytes,
                         float* g_out, dmtz_edit* edits, int64_t edits_capacity,
                         int64_t* n_edits /* host */, dmtz_stats* stats /* host */,
                         dmtz_stream_t stream);

/* dmtz_correct from HOST buffers (the end-to-end call): copies f_host and fhat_host
 * (float[N]; pinned for full PCIe/C2C bandwidth, pageable works) into the caller's
 * device buffers f_dev / fhat_dev, runs dmtz_correct on the device buffers, and
 * copies g (float[N]) into g_host and the n = min(*n_edits, edits_capacity) edits
 * into edits_host (dmtz_edit[edits_capacity]), all on `stream`; returns after the
 * copies completed.  g_dev / edits_dev are device outputs as in dmtz_correct.
 * g_host or edits_host may be NULL (that result is not copied back).  Same
 * statuses as dmtz_correct; the host outputs are written when it returns
 * DMTZ_OK, DMTZ_E_STUCK, DMTZ_E_ITER_CAP or DMTZ_E_CAPACITY. */
dmtz_status dmtz_correct_host(dmtz_ctx* ctx, const float* f_host, const float* fhat_host,
                              const dmtz_correct_opts* opts, void* workspace, size_t workspace_bytes,
                              float* f_dev, float* fhat_dev, float* g_dev, dmtz_edit* edits_dev,
                              int64_t edits_capacity, float* g_host, dmtz_edit* edits_host,
                              int64_t* n_edits /* host */, dmtz_stats* stats /* host */,
                              dmtz_stream_t stream);

/* Separatrix traces of a gradient (P:82 gradient paths):
 *   DESC: from each endpoint (ascending index) of each critical edge, vertex ->
 *         paired edge -> its other vertex, until a critical vertex (minimum).
 *         cells = v0, e1, v1, ..., v_min; terminal = the minimum.
 *   ASC:  from each critical (top-1)-cell, through each top cofacet in slot
 *         order: critical top cell -> maximum (terminal); else the top cell is
 *         paired down with a facet c, continue through c's other top cofacet;
 *         none -> terminal = DMTZ_BOUNDARY.  cells = t0, c1, t1, ...
 *   CONN (3D): breadth-first from each critical triangle over facet edges (in
 *         omitted-vertex order): critical edge -> recorded (each time met);
 *         edge paired up with an unvisited triangle -> recorded and enqueued.
 *         cells = the event log (triangles visited, edges reached); terminal =
 *         DMTZ_BOUNDARY.
 * Branches are grouped DESC, ASC, CONN; within a kind ordered by origin cell id,
 * then branch order.  Outputs go to caller buffers with capacities cap_branches
 * (branch_offsets holds cap_branches + 1) and cap_cells; *n_branches / *n_cells
 * (host) receive the needed sizes; DMTZ_E_CAPACITY if they exceed the caps. */
#define DMTZ_KIND_DESC 1u
#define DMTZ_KIND_ASC 2u
#define DMTZ_KIND_CONN 4u
#define DMTZ_BOUNDARY UINT64_MAX
typedef struct {
  int64_t* branch_offsets; /* [cap_branches + 1] */
  uint64_t* cells;         /* [cap_cells] */
  uint64_t* origin;        /* [cap_branches] */
  uint64_t* terminal;      /* [cap_branches] */
  uint8_t* kind;           /* [cap_branches] */
} dmtz_seps;
dmtz_status dmtz_trace_separatrices(dmtz_ctx* ctx, const void* codes, uint32_t kinds,
                                    void* workspace, size_t workspace_bytes, dmtz_seps* out,
                                    int64_t cap_branches, int64_t cap_cells,
                                    int64_t* n_branches /* host */, int64_t* n_cells /* host */,
                                    dmtz_stream_t stream);
/* The same restricted to the branches whose origin cell is anchored in the z-planes
 * [z_begin, z_end) (codes cover the whole grid): within each kind these are a
 * contiguous run of dmtz_trace_separatrices' branches, so ranks that own disjoint
 * plane ranges (with the gradient replicated, slab.trace_distributed) produce, kind by
 * kind and in rank order, exactly its output. */
dmtz_status dmtz_trace_separatrices_range(dmtz_ctx* ctx, const void* codes, uint32_t kinds, int64_t z_begin,
                                          int64_t z_end, void* workspace, size_t workspace_bytes, dmtz_seps* out,
                                          int64_t cap_branches, int64_t cap_cells, int64_t* n_branches /* host */,
                                          int64_t* n_cells /* host */, dmtz_stream_t stream);

/* ------------------------------------------------------------------------
 * Tiers 3-4: S-loops and the alternating C/S workflow.
 * P:150 / Fig. 2: "C-loops and S-loops alternate until no false critical cells
 * or separatrices exist"; an S-loop iteration (1) traces the
 * separatrices, (2) identifies the TROUBLEMAKER of each -- the first cell along it
 * whose gradient pairing differs from the original one -- and (3)
 * decreases the vertex of the original partner the troublemaker does not share
 * ("decrease j" / "k" / "l").  Rounds are synchronous (DESIGN.md
 * readings A7, A17): each round recomputes the gradient of g; false critical cells
 * (tier 2's F) make it a C-round; otherwise the separatrices of f are checked --
 * tier 4: every branch (same paths); tier 3: the branches whose traced end in
 * g differs (same extrema; connectors: the same multiset of 1-saddles) --
 * and the set of their troublemakers' targets takes one Eq. 2 step; none left ->
 * done.  Each branch is walked in the order of dmtz_trace_separatrices' cells:
 * DESC the vertices before the minimum, ASC the (top-1)-cells, CONN the facet
 * edges (facet order, f-critical ones skipped) of the triangles in queue order.
 * ------------------------------------------------------------------------ */
typedef struct {
  int64_t c_rounds;        /* rounds that fixed false critical cells */
  int64_t s_rounds;        /* rounds that fixed troublemakers */
  int64_t troublemakers;   /* summed over the S-rounds */
  int64_t tm_by_kind[3];   /* of which on DESC / ASC / CONN branches */
  int64_t sep_branches;    /* separatrices of f (branches / CSR cells) */
  int64_t sep_cells;
  int64_t tm_round1;       /* troublemakers of the first S-round */
  double trace_ms;         /* device time: trace of f + its cell -> branch map */
  double s_ms;             /* device time summed over the S-rounds (search + edit; tier 3: + trace of g) */
  int64_t cells_checked;   /* CSR cells whose pairing was re-evaluated, summed over the S-rounds (after
                              the first, only cells with a code changed since the last S-round) */
  int64_t pad[4];
} dmtz_sloop_stats;

/* Device bytes dmtz_preserve needs in `sep_ws` for separatrix CSRs of at most
 * cap_branches branches / cap_cells cells (size them with a
 * dmtz_trace_separatrices call of capacity 0 on the codes of f: it returns
 * DMTZ_E_CAPACITY with the exact counts; tier 3 also traces g, whose paths may
 * be longer: give it headroom).  0 for tiers 1-2. */
size_t dmtz_preserve_sep_bytes(const dmtz_ctx* ctx, const dmtz_correct_opts* opts, int64_t cap_branches,
                               int64_t cap_cells);

/* The workflow for opts->tier in 1..5 (tiers 1-2: exactly dmtz_correct; sep_ws may
 * be NULL; tier 5: every vertex of every critical cell of f is first
 * set to its lower bound (a lossless edit), then the tier-4 workflow runs).  Same inputs, outputs and errors as dmtz_correct, plus sstats (host);
 * DMTZ_E_CAPACITY also when a separatrix CSR exceeds the caps (sstats->sep_* hold
 * the needed counts).  ITER_CAP counts C- and S-rounds together. */
dmtz_status dmtz_preserve(dmtz_ctx* ctx, const float* f, const float* fhat, const dmtz_correct_opts* opts,
                          void* workspace, size_t workspace_bytes, void* sep_ws, size_t sep_ws_bytes,
                          int64_t cap_branches, int64_t cap_cells, float* g_out, dmtz_edit* edits,
                          int64_t edits_capacity, int64_t* n_edits /* host */, dmtz_stats* stats /* host */,
                          dmtz_sloop_stats* sstats /* host */, dmtz_stream_t stream);

/* ------------------------------------------------------------------------
 * Edits as a storable artifact.  P:276-280: the quantized
 * representation stores "only the integer count of edits q for each vertex"; the
 * rare lossless entries keep their value; Fig. 2: "the edits are applied to
 * the decompressed data ... in the decompression stage".
 *
 * Edit stream (little-endian):
 *   0  char[4] "DMTE" | 4 uint32 version (1 or 2) | 8 uint64 n_edits | 16 uint32 edits
 *   per block (4096) | 20 int32 q_max | 24 float xi | 28 uint32 n_blocks | 32 uint64
 *   block_offset[n_blocks] (byte offset of each block's first record in the payload) |
 *   payload: per edit, ascending v: varint(delta) varint(q << 1 | lossless)
 *   [lossless only -- version 1: uint32 value bits; version 2: varint(zigzag(d)),
 *   d = int64(fhat bits as int32) - int64(value bits as int32): the stored value is
 *   exact and, since fhat - 2 xi <= value <= fhat, d is a few thousand ulps at most];
 *   delta = v for a block's first edit, else v - v_prev - 1; varint = unsigned LEB128.
 * ------------------------------------------------------------------------ */
/* dmtz_correct_host that returns the storable artifact instead of the raw edit list:
 * pinned host f and fhat in (as dmtz_correct_host), the C-loop, the edit list encoded
 * on the device (version 2 below) into stream_dev (capacity stream_cap, e.g.
 * dmtz_edit_stream_bound(N)), and only the stream's *stream_bytes bytes copied to
 * stream_host (capacity stream_host_cap) -- plus g to g_host when it is not NULL (g
 * is also f_hat with the stream applied: dmtz_apply_edits).  edits_dev (capacity
 * edits_capacity) holds the raw list on return.  Synchronises the stream.  Status as
 * dmtz_correct; DMTZ_E_CAPACITY if a buffer is too small. */
dmtz_status dmtz_correct_host_stream(dmtz_ctx* ctx, const float* f_host, const float* fhat_host,
                                     const dmtz_correct_opts* opts, void* workspace, size_t workspace_bytes,
                                     float* f_dev, float* fhat_dev, float* g_dev, dmtz_edit* edits_dev,
                                     int64_t edits_capacity, uint8_t* stream_dev, size_t stream_cap, float* g_host,
                                     uint8_t* stream_host, size_t stream_host_cap, size_t* stream_bytes /* host */,
                                     int64_t* n_edits /* host */, dmtz_stats* stats /* host */, dmtz_stream_t stream);
/* Upper bound of the stream size for n_edits edits. */
size_t dmtz_edit_stream_bound(int64_t n_edits);
/* Encode a sorted edit list (device, as dmtz_correct writes it) into `out` (device,
 * capacity cap bytes); *nbytes (host) = the stream size (DMTZ_E_CAPACITY if > cap).
 * fhat (device, the decompressed field) != NULL writes version 2 (lossless values
 * relative to fhat), NULL version 1.  Uses the workspace as scratch (n_edits <= the
 * context's vertex count).  DMTZ_E_ARG if the list is not strictly ascending. */
dmtz_status dmtz_encode_edits(dmtz_ctx* ctx, const dmtz_edit* edits, int64_t n_edits, float xi, int32_t q_max,
                              const float* fhat, void* workspace, size_t workspace_bytes, uint8_t* out, size_t cap,
                              size_t* nbytes /* host */, dmtz_stream_t stream);
/* Decode a stream (device, nbytes) into edits (device, capacity cap); *n_edits, *xi,
 * *q_max (host) from its header; fhat (device) is required for version 2 (ignored for
 * version 1).  Quantized entries carry no value (apply recomputes it).  DMTZ_E_ARG on a
 * malformed stream (bad magic or version, truncated, a vertex outside the grid). */
dmtz_status dmtz_decode_edits(dmtz_ctx* ctx, const uint8_t* in, size_t nbytes, const float* fhat, dmtz_edit* edits,
                              int64_t cap, int64_t* n_edits /* host */, float* xi /* host */, int32_t* q_max /* host */,
                              void* workspace, size_t workspace_bytes, dmtz_stream_t stream);
/* Decompression side: g_out = fhat with every edit applied -- quantized:
 * RN(fhat - RN(q * xi 2^-q_max)) (Eq. 2 replayed from fhat), lossless: the
 * stored bits.  Equals dmtz_correct's g bit for bit.  DMTZ_E_ARG if a vertex is
 * outside the grid (checked on the device; the call synchronises the stream). */
dmtz_status dmtz_apply_edits(dmtz_ctx* ctx, const float* fhat, float xi, int32_t q_max, const dmtz_edit* edits,
                             int64_t n_edits, float* g_out, void* workspace, size_t workspace_bytes,
                             dmtz_stream_t stream);

/* ------------------------------------------------------------------------
 * Evaluation metrics (§5.1).  Recall = n_match /
 * n_orig, precision = n_match / n_rec (1 when the denominator is 0).
 * ------------------------------------------------------------------------ */
typedef struct { int64_t n_orig, n_rec, n_match; } dmtz_prf;
/* Critical cells: masks (uint32[N] per anchor, bit = type, as dmtz_critical_mask
 * writes them) of the original and the reconstructed field; a cell matches when it is
 * critical in both ("retained").  Synchronises the stream. */
dmtz_status dmtz_critical_prf(dmtz_ctx* ctx, const uint32_t* crit_orig, const uint32_t* crit_rec,
                              dmtz_prf* out /* host */, void* workspace, size_t workspace_bytes,
                              dmtz_stream_t stream);
/* Separatrices: two outputs of dmtz_trace_separatrices (device CSRs with nb_orig /
 * nb_rec branches).  The unit is a branch, identified by (kind, origin cell, ordinal
 * among its origin's branches); it matches when both traces hold it with the same
 * terminal and the same cell sequence.  Synchronises the stream. */
dmtz_status dmtz_separatrix_prf(dmtz_ctx* ctx, const dmtz_seps* orig, int64_t nb_orig, const dmtz_seps* rec,
                                int64_t nb_rec, dmtz_prf* out /* host */, void* workspace,
                                size_t workspace_bytes, dmtz_stream_t stream);

/* ------------------------------------------------------------------------
 * Slab mode (multi-GPU z-slab decomposition).  One context per
 * rank, created for its LOCAL grid: the owned z-planes plus up to 3 halo planes
 * below and above (nz_local = own + halos).  The caller drives the rounds and,
 * between them, refreshes the halo planes of g from the neighbouring ranks (the
 * library never communicates).  Cells are classified only when anchored in local
 * planes [anchor_z0, anchor_z1) -- own_z0 - 2 .. own_z1 + 1 clipped to the grid:
 * every cell whose target can be an owned vertex -- and only owned vertices are
 * edited, so the rounds are those of dmtz_correct on the global grid and the
 * concatenated edit lists are its edit list (bit for bit).
 * ------------------------------------------------------------------------ */
typedef struct {
  int64_t z_offset;              /* global z of local plane 0 */
  int64_t own_z0, own_z1;        /* owned local planes */
  int64_t anchor_z0, anchor_z1;  /* local planes whose anchored cells are classified */
} dmtz_slab;

/* Validate (finite, |fhat - f| <= xi), lb, g = fhat, gradient of f on the local grid. */
dmtz_status dmtz_slab_begin(dmtz_ctx* ctx, const float* f, const float* fhat, const dmtz_correct_opts* opts,
                            const dmtz_slab* slab, void* workspace, size_t workspace_bytes, float* g,
                            dmtz_stream_t stream);
/* One round (a3-a6) with g's halo planes current.  counters (host, 4): false cells
 * anchored in the classified planes, targets that moved, targets, invariant
 * violations; kinds (host, 8): false cells by kind (round 1 only, else zero).
 * The caller sums counters over ranks and stops as dmtz_correct does. */
dmtz_status dmtz_slab_round(dmtz_ctx* ctx, const float* f, const float* fhat, const dmtz_correct_opts* opts,
                            const dmtz_slab* slab, void* workspace, size_t workspace_bytes, float* g,
                            int64_t round, int64_t* counters, int64_t* kinds, dmtz_stream_t stream);
/* The same round without any host synchronisation: the 12 counters (counters[4] then
 * kinds[8]) go to dcounters (device, int64[12]) on the stream, so the caller can
 * all-reduce them on the device and decide to stop a round later (a round after the
 * fixed point or after STUCK changes nothing). */
dmtz_status dmtz_slab_round_async(dmtz_ctx* ctx, const float* f, const float* fhat, const dmtz_correct_opts* opts,
                                  const dmtz_slab* slab, void* workspace, size_t workspace_bytes, float* g,
                                  int64_t round, int64_t* dcounters /* device, 12 */, dmtz_stream_t stream);
/* Halo refresh between rounds: replace the local planes [z_begin, z_end) of g with
 * `planes` (device, (z_end - z_begin) * ny * nx f32, the neighbour's values after
 * round `round`), and record every vertex whose value changed, so that round + 1
 * re-screens exactly the anchors whose 3x3x3 box holds such a vertex and its frontier
 * contains the cells they can affect (the same rule as for this rank's own edits). */
dmtz_status dmtz_slab_halo(dmtz_ctx* ctx, const dmtz_slab* slab, void* workspace, size_t workspace_bytes, float* g,
                           const float* planes, int64_t z_begin, int64_t z_end, int64_t round, dmtz_stream_t stream);
/* The owned edits (global vertex indices, sorted). */
dmtz_status dmtz_slab_end(dmtz_ctx* ctx, const dmtz_slab* slab, void* workspace, size_t workspace_bytes,
                          const float* g, dmtz_edit* edits, int64_t edits_capacity, int64_t* n_edits /* host */,
                          int64_t* n_lossless /* host */, dmtz_stream_t stream);

const char* dmtz_status_string(dmtz_status s);
const char* dmtz_last_error(void);
int dmtz_version(void);
/* Diagnostics of the calling thread's last dmtz_trace_separatrices(_range) call: out[i]
 * (i < n, n <= 10) = connectors handled at escalation level i in its count pass --
 * [0] all connectors (one thread each, shared-memory queue), [1] those that overflowed
 * into one warp each, [2], [3], ... those that overflowed into the block-parallel BFS
 * with slots growing per level.  Host pointer; returns
 * DMTZ_E_ARG for a NULL out. */
int dmtz_last_trace_levels(int64_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* DMTZ_H */
