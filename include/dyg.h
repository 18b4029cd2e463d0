/*
 * dyg.h -- C-ABI of the B200-native dyGRASS batched update path.
 *
 * The reference (/root/reference/proj) has no C API or FFI; its seams are two
 * C++ interfaces:
 *   (1) run_batch(const DynamicGraph&, span<const WalkQuery>, const WalkConfig&)
 *       -- proj/src/walk.hpp:86-92, a pure function of the graph snapshot;
 *   (2) SparsifierState -- proj/src/sparsifier.hpp:71-112: ctor(G, H, options),
 *       graph(), sparsifier(), update_counter(), apply_insertion(),
 *       apply_deletion(), last_event_steps(), replay_batch(stream, b),
 *       replay(stream).
 * Each entry point below names the reference interface it replaces. Plain
 * pointers and sizes only; no exceptions cross the boundary. Return codes are
 * the reference's ErrorKind values (proj/src/error.hpp:8-9: "values match ...
 * the C API status codes"): 0 ok, 1 Usage, 2 Data, 3 Numeric, plus 4 for a
 * CUDA/device failure. dyg_last_error() holds the message (thread-local).
 *
 * Ownership: the caller owns every host buffer passed in or out; a session
 * owns its device memory. One session = one writer thread (sparsifier.hpp:
 * 67-70). All calls are stream-ordered on the session's CUDA stream and
 * synchronous on return unless stated otherwise.
 *
 * Struct layouts are part of the ABI (tests share numpy dtypes with them).
 */
#ifndef DYG_H
#define DYG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define DYG_OK 0
#define DYG_ERR_USAGE 1   /* ErrorKind::Usage   (error.hpp:9) */
#define DYG_ERR_DATA 2    /* ErrorKind::Data    */
#define DYG_ERR_NUMERIC 3 /* ErrorKind::Numeric */
#define DYG_ERR_DEVICE 4  /* CUDA error or missing device (no reference analogue) */

/* Per-event decisions (the optional per_event_decision outputs below), one
 * byte per event. Insertions: InsertionDecision (sparsifier.hpp:36), what
 * commit_insertion returns (sparsifier.cpp:220-241). Deletions:
 * DeletionOutcome::Kind (sparsifier.hpp:38-42) as replay_batch_deferred
 * resolves it at commit (sparsifier.cpp:489-523): not in live H -> GraphOnly,
 * a recovered path -> PathRecovered, the local fallback (or freeze) ->
 * LocalFallback. Events that did not commit (validation error, the failing
 * event and every event after it, :525-529) stay DYG_DECISION_NONE. */
#define DYG_DECISION_KEPT 0
#define DYG_DECISION_PRUNED 1
#define DYG_DECISION_GRAPH_ONLY 2
#define DYG_DECISION_PATH_RECOVERED 3
#define DYG_DECISION_LOCAL_FALLBACK 4
#define DYG_DECISION_NONE 255

/* Graph rows in reference row order: row u is DynamicGraph::neighbors(u)
 * (graph.hpp:37-38), flattened. row_ptr has n+1 entries; ids/w have
 * row_ptr[n] = 2|E| entries. Every edge appears in both endpoint rows with
 * bit-identical weights. */
typedef struct dyg_csr {
  uint32_t n;
  uint32_t pad;
  const uint64_t* row_ptr;
  const uint32_t* ids;
  const double* w;
} dyg_csr;

/* WalkConfig (walk.hpp:13-18). */
typedef struct dyg_walk_config {
  double distortion_threshold; /* K; 0 = no-filter baseline (sparsifier.hpp:32-33) */
  uint32_t step_cap;           /* T */
  uint32_t walker_count;       /* s */
  uint64_t global_seed;
} dyg_walk_config;

/* SparsifierOptions (sparsifier.hpp:25-34). */
typedef struct dyg_options {
  dyg_walk_config walk;
  int32_t batched;           /* deferred (batched) replay; 0 = immediate */
  int32_t freeze_sparsifier; /* drift baseline */
} dyg_options;

/* EdgeEvent (stream.hpp:11-18). kind: 0 insertion, 1 deletion. */
typedef struct dyg_event {
  uint32_t kind;
  uint32_t u;
  uint32_t v;
  uint32_t batch_index;
  double weight; /* insertions only */
} dyg_event;

/* WalkQuery (walk.hpp:71-78). kind: 0 Reach, 1 MinPath. */
typedef struct dyg_walk_query {
  uint32_t kind;
  uint32_t p;
  uint32_t q;
  uint32_t pad;
  double w_pq; /* Reach only */
  uint64_t update_id;
} dyg_walk_query;

/* WalkResult (walk.hpp:80-84) flattened: Reach -> reached, best_estimate;
 * MinPath -> reached (= path found), path_len, resistance and the loop-erased
 * vertices in path_buf[i*(T+1) ...]. */
typedef struct dyg_walk_result {
  uint32_t reached;
  uint32_t path_len;
  double best_estimate;
  uint64_t steps_used;
  double resistance;
} dyg_walk_result;

/* BatchReport (sparsifier.hpp:44-59). wall_ms is the batch's T_update on the
 * device: its first kernel's start to its commit's end (%globaltimer stamps
 * the kernels write), host staging excluded. */
typedef struct dyg_batch_report {
  uint32_t batch_index;
  uint32_t pad;
  uint64_t insertions_seen;
  uint64_t insertions_kept;
  uint64_t insertions_pruned;
  uint64_t deletions_seen;
  uint64_t deletions_in_sparsifier;
  uint64_t paths_recovered;
  uint64_t edges_recovered;
  uint64_t fallback_activations;
  uint64_t walker_steps;
  uint64_t max_event_steps;
  double wall_ms;
  double density_graph;
  double density_sparsifier;
} dyg_batch_report;

/* Per-session counters (no reference analogue; SURVEY.md 5 "metrics"). */
typedef struct dyg_stats {
  uint64_t batches;
  uint64_t kernel_launches;     /* kernels this library launched */
  uint64_t reach_queries;
  uint64_t minpath_queries;
  uint64_t reach_steps;         /* walker steps on H (== sum of steps_used) */
  uint64_t minpath_steps;       /* walker steps on shadow G */
  uint64_t reach_row_bytes;     /* sum over steps of 32*ceil((8+12*deg)/32) */
  uint64_t minpath_row_bytes;
  double reach_ms;              /* device time of the reach-walk kernel(s) */
  double minpath_ms;            /* device time of the min-path walk + winner kernels */
  double commit_ms;             /* device time of the commit engine */
  double total_ms;              /* device time of whole batches */
  uint64_t commit_rounds;       /* dependency rounds used by the commit engine */
  uint64_t pool_used;           /* overflow-pool entries in use (G + H) */
  uint64_t pool_capacity;
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  double commit_ms_deletion;    /* commit_ms share of batches containing deletions */
  double reach_tail_ms;         /* reach walks after the work queue drained (device clock) */
  double minpath_tail_ms;
  uint64_t commit_rounds_deletion;
  /* Dataflow deletion commit (k_del_flow) phase times, device clock:
     fallback promotion, record emission, ranks, apply, reset. */
  double flow_ms_promote;
  double flow_ms_emit;
  double flow_ms_rank;
  double flow_ms_apply;
  double flow_ms_reset;
  uint64_t graph_launches;      /* CUDA-graph replays (one per batch or per range) */
  double prep_ms;               /* batch start -> first walk warp (validation, query build) */
  double walk_commit_gap_ms;    /* last walk warp -> commit start */
  double batch_gap_ms;          /* previous batch end -> batch start, inside one replay */
  double minpath_walk_ms;       /* the min-path walk kernel alone (minpath_ms adds the winner) */
  uint64_t reach_tail_row_bytes;   /* reach_row_bytes of steps after the work queue drained */
  uint64_t minpath_tail_row_bytes;
} dyg_stats;

typedef struct dyg_session dyg_session;

/* Thread-local message for the last non-zero return on this thread. */
const char* dyg_last_error(void);
/* Library build string (arch, flags). */
const char* dyg_version(void);
/* Number of visible CUDA devices (0 when none). */
int dyg_device_count(void);
/* Page-locked host memory for event buffers (NULL on failure / no device).
   dyg_replay_events and dyg_shard_begin DMA straight from such buffers;
   other host buffers are staged through the session's pinned copy first.
   No reference counterpart: a B200 host-side addition. */
void* dyg_host_alloc(size_t bytes);
void dyg_host_free(void* p);

/* SparsifierState::SparsifierState(G, H, options) (sparsifier.cpp:183-203):
 * validates shapes and H subset of G, uploads both graphs to `device` as
 * device-resident dynamic rows. */
int dyg_session_create(const dyg_csr* g, const dyg_csr* h, const dyg_options* options,
                       int device, dyg_session** out);
void dyg_session_destroy(dyg_session* s);

/* SparsifierState::replay_batch(stream, b) (sparsifier.cpp:541-548): the
 * stream is `events[0..n_events)` with `batch_count` (UpdateStream,
 * stream.hpp:20-23); events of batch b are found by scanning, as the
 * reference does (sparsifier.cpp:401-404). Deferred or immediate mode per
 * options.batched. per_event_decision (nullable): one DYG_DECISION_* per
 * event OF THE BATCH, in stream order (k-th event of batch b at [k]). */
int dyg_replay_batch(dyg_session* s, const dyg_event* events, size_t n_events,
                     uint32_t batch_count, uint32_t batch_index, dyg_batch_report* out,
                     uint8_t* per_event_decision);

/* The same for a batch already extracted by the caller: `events` are the
 * batch's events in stream order and `positions` their stream indices (used
 * in error messages; NULL means 0..n-1). per_event_decision (nullable):
 * n entries, [k] for events[k]. */
int dyg_replay_events(dyg_session* s, const dyg_event* events, const uint64_t* positions,
                      size_t n, uint32_t batch_index, dyg_batch_report* out,
                      uint8_t* per_event_decision);

/* SparsifierState::replay(stream) (sparsifier.cpp:550-559) from a host
 * stream: out[b] for every batch b < batch_count. Events grouped by batch
 * (batch b = events[batch_offsets[b] .. batch_offsets[b+1]); batch_offsets
 * NULL = found by one pass over batch_index) replay with the upload of later
 * batches overlapping the work on earlier ones; ungrouped streams replay
 * batch by batch. On an error the batches before the failing one are
 * committed and reported, the failing one returns the reference's error and
 * later ones do not run. per_event_decision (nullable): n_events entries,
 * indexed by stream position. */
int dyg_replay_stream(dyg_session* s, const dyg_event* events, size_t n_events,
                      const uint64_t* batch_offsets, uint32_t batch_count,
                      dyg_batch_report* out, uint8_t* per_event_decision);

/* Device-resident stream: upload once, then replay batches with no per-batch
 * host->device traffic (used for the kernel-level benchmark). Events already
 * grouped by batch in page-locked memory (dyg_host_alloc) are DMA'd
 * asynchronously, stream-ordered before any later replay: keep that buffer
 * unchanged until the next replay call returns. */
int dyg_stream_upload(dyg_session* s, const dyg_event* events, size_t n_events,
                      uint32_t batch_count);
/* The same upload for a stream grouped by batch (batch b =
 * events[batch_offsets[b] .. batch_offsets[b+1]), as in dyg_replay_stream):
 * from page-locked memory it returns at once -- each batch is DMA'd and its
 * kinds counted on a copy stream, and dyg_shard_begin_uploaded(b) waits for
 * batch b alone, so the upload overlaps the earlier batches' work. `events`
 * must stay valid until the next upload or the session's destruction.
 * Pageable events fall back to dyg_stream_upload. */
int dyg_stream_upload_batches(dyg_session* s, const dyg_event* events, size_t n_events,
                              const uint64_t* batch_offsets, uint32_t batch_count);
int dyg_replay_uploaded(dyg_session* s, uint32_t batch_index, dyg_batch_report* out);
/* SparsifierState::replay over batches [first, first + count) of the
 * uploaded stream (sparsifier.cpp:550-559): all batches are enqueued back to
 * back with one host synchronisation; out[i] is batch first + i. On an error
 * the batches before the failing one are committed and reported, the
 * failing one returns the reference's error, and later ones do not run.
 * per_event_decision (nullable): indexed by position in the uploaded stream
 * (entries of batches outside the range are left untouched). */
int dyg_replay_uploaded_range(dyg_session* s, uint32_t first, uint32_t count,
                              dyg_batch_report* out, uint8_t* per_event_decision);

/* SparsifierState::apply_insertion / apply_deletion (sparsifier.cpp:243-317).
 * decision: 0 Kept, 1 Pruned (InsertionDecision). kind: 0 GraphOnly,
 * 1 PathRecovered, 2 LocalFallback (DeletionOutcome::Kind). */
int dyg_apply_insertion(dyg_session* s, uint32_t u, uint32_t v, double w, int* decision);
int dyg_apply_deletion(dyg_session* s, uint32_t u, uint32_t v, int* kind,
                       uint32_t* edges_added);
/* SparsifierState::last_event_steps (sparsifier.hpp:92-93). */
uint64_t dyg_last_event_steps(const dyg_session* s);
/* SparsifierState::update_counter (sparsifier.hpp:79). */
uint64_t dyg_update_counter(const dyg_session* s);

/* graph() / sparsifier() accessors (sparsifier.hpp:76-77). which: 0 = G,
 * 1 = H. Counters, then a row-order export: row_ptr[n+1], ids/w sized by
 * *entries (= 2|E|). */
int dyg_graph_info(const dyg_session* s, int which, uint32_t* n, uint64_t* edges,
                   double* density);
int dyg_export_rows(dyg_session* s, int which, uint64_t* row_ptr, uint32_t* ids, double* w,
                    uint64_t capacity);

/* Device-side snapshot of (G, H, update_counter) and its restore: resume /
 * parity bisection (SURVEY.md 5 checkpoint row) and benchmark resets. */
int dyg_session_snapshot(dyg_session* s);
int dyg_session_restore(dyg_session* s);

/* Cross-process checkpoint / resume (no reference counterpart --
 * the reference's SparsifierState lives in one process). Saves (options,
 * update_counter, G rows, H rows) in reference row order with a checksum;
 * a session loaded from it continues with the same walker keys
 * (sparsifier.cpp:431) and adjacency order, so replaying the rest of a
 * stream gives what the uninterrupted session would have. DYG_ERR_DATA on
 * an unreadable, truncated or corrupt file. */
int dyg_session_save(dyg_session* s, const char* path);
/* SparsifierState::options() (sparsifier.hpp:75). */
int dyg_session_options(const dyg_session* s, dyg_options* out);
int dyg_session_load(const char* path, int device, dyg_session** out);

int dyg_session_stats(const dyg_session* s, dyg_stats* out);
/* Per-step walk statistics (dyg_stats reach_steps, minpath_steps,
 * *_row_bytes, *_tail_row_bytes): counted by an instrumented variant of the
 * walk kernels, ~6 % slower than the default one; off by default (those
 * fields then stay 0; the walk durations and drain stamps are always
 * recorded). The walks themselves -- and every result -- are identical. */
int dyg_session_set_walk_counters(dyg_session* s, int on);
int dyg_session_reset_stats(dyg_session* s);

/* build_initial_sparsifier (sparsifier.cpp:105-159) on `device`, bit-identical
 * to the reference: maximum spanning tree in (weight desc, (u, v) asc) order,
 * then off-tree edges by distortion w * R_tree(u, v) descending (ties:
 * hash_mix(seed ^ (u << 32 | v)) ascending) until density >= target.
 * row_ptr_out[n + 1]; ids_out / w_out need room for g's nnz (H's rows, in
 * the order the reference's insert_edge calls build them). Usage error for a
 * negative target, Data error for a disconnected graph. */
int dyg_build_initial_sparsifier(const dyg_csr* g, double target_density, uint64_t seed,
                                 int device, uint64_t* row_ptr_out, uint32_t* ids_out,
                                 double* w_out);

/* ---- spectral evaluation ----------------------
 * ConditionOptions (spectral.hpp:78-85). method: 0 Auto (Dense when
 * n <= dense_cap), 1 Dense, 2 Iterative. Zero-initialised fields take the
 * reference defaults: tolerance 1e-6, max_iterations 400, dense_cap 5000,
 * seed 0x5eed (use dyg_condition_options_default). */
typedef struct dyg_condition_options {
  int32_t method;
  uint32_t max_iterations;
  double tolerance;
  uint32_t dense_cap;
  uint32_t pad;
  uint64_t seed;
} dyg_condition_options;

/* ConditionEstimate (spectral.hpp:69-76). method: 0 Dense, 1 Iterative.
 * inner_iterations: CG iterations of the L_H solves (no reference analogue:
 * the reference factorises L_H exactly). */
typedef struct dyg_condition_estimate {
  double kappa;
  double lambda_max;
  double lambda_min;
  int32_t method;
  uint32_t iterations_used;
  int32_t converged;
  uint32_t pad;
  uint64_t inner_iterations;
} dyg_condition_estimate;

void dyg_condition_options_default(dyg_condition_options* out);
/* condition_number(G, H, options) (spectral.cpp:278-303): extreme
 * generalized eigenvalues of the pencil (L_G, L_H) on the complement of the
 * constant vector. Dense: cuSOLVER sygvd on the grounded pencil; Iterative:
 * Lanczos in the L_H inner product (spectral.cpp:151-276) on `device`. */
int dyg_condition_number(const dyg_csr* g, const dyg_csr* h, const dyg_condition_options* options,
                         int device, dyg_condition_estimate* out);
/* calibrate_budget(G, H, probe_fraction, rho, seed) (sparsifier.cpp:561-577):
 * clamp(rho * kappa, 1, 1e6) from a coarse (tolerance 1e-3) estimate. */
int dyg_calibrate_budget(const dyg_csr* g, const dyg_csr* h, double probe_fraction, double rho,
                         uint64_t seed, int device, double* budget);
/* The same on a session's current G and H; the seed is the session's
 * walk.global_seed (sparsifier.cpp:579-583). */
int dyg_session_calibrate_budget(dyg_session* s, double probe_fraction, double rho,
                                 double* budget);
int dyg_session_condition_number(dyg_session* s, const dyg_condition_options* options,
                                 dyg_condition_estimate* out);

/* PcgResult (solver.hpp:44-49); the solution goes to the caller's buffer. */
typedef struct dyg_pcg_result {
  uint32_t iterations;
  int32_t converged;
  double relative_residual; /* recomputed from scratch */
  uint64_t inner_iterations;
  uint64_t energy_count;    /* entries written to energy_trace */
} dyg_pcg_result;

/* pcg_solve(laplacian(G), rhs, M, tolerance, max_iterations, energy_trace)
 * (solver.cpp:71-144) with M = Preconditioner::from_graph(H, factor_cap)
 * (solver.cpp:10-25), or the identity when h == NULL. rhs and x have n
 * entries; energy_trace (nullable) receives up to energy_cap values of
 * 0.5 x'L_G x - b'x, one per iteration. factor_cap 0 = the reference's
 * 2,000,000. */
int dyg_pcg_solve(const dyg_csr* g, const dyg_csr* h, uint32_t factor_cap, const double* rhs,
                  double tolerance, uint32_t max_iterations, int device, double* x,
                  dyg_pcg_result* out, double* energy_trace, size_t energy_cap);
/* random_rhs(n, seed) (solver.cpp:146-159), on the host. */
int dyg_random_rhs(uint32_t n, uint64_t seed, double* out);

/* generate_update_stream(G, {insert_fraction, delete_fraction, batches,
 * seed, locality 0}) (stream.cpp:114-200) with the insertion sampling on
 * `device`, bit-identical to the reference: attempts are drawn
 * speculatively in parallel from the counter-based SplitMix64 stream and
 * accepted up to the first rejected one per round (self-loop, edge of G,
 * repeated pair); deletions (a partial Fisher-Yates) on the host. Writes the
 * events in stream order; *n_out is set even when `capacity` is too small
 * (then DYG_ERR_USAGE: call again with a larger buffer). The locality > 0
 * mode is the host generator's (dygh_generate_stream). */
int dyg_generate_stream(const dyg_csr* g, double insert_fraction, double delete_fraction,
                        uint32_t batches, uint64_t seed, int device, dyg_event* out,
                        size_t capacity, size_t* n_out, uint32_t* batch_count);
/* Exact Laplacian solves reuse a fill-reducing ordering for an identical H
 * sparsity pattern, or one differing in at most 5 % of its nonzeros (H
 * between batches); cumulative counts of exact hits, near hits and fresh
 * orderings in this process. No reference counterpart. */
int dyg_spectral_ordering_stats(uint64_t* hits, uint64_t* near_hits, uint64_t* misses);

/* Stateless twin of run_batch (walk.hpp:86-92): uploads g, runs the queries
 * on `device`, returns results in query order. path_buf (nullable) receives
 * MinPath vertices at [i*(T+1)]. */
int dyg_run_batch(const dyg_csr* g, const dyg_walk_query* queries, size_t n_queries,
                  const dyg_walk_config* cfg, dyg_walk_result* out, uint32_t* path_buf,
                  int device);

/* ---- multi-GPU split of replay_batch -------------------
 * Every rank holds a replica of (G, H). For batch b every rank calls
 * dyg_shard_walk(rank, world), which runs the walk phase for the contiguous
 * query range [floor(nq*rank/world), floor(nq*(rank+1)/world)) and writes a
 * fixed-size record per query slot into `records` (device pointer,
 * dyg_shard_record_bytes() bytes per slot, `slots` slots = ceil(nq_max/world)
 * on every rank, unused slots zeroed). The caller all-gathers the records
 * (NCCL over NVLink) into `gathered` (world*slots slots, rank-major) and
 * calls dyg_shard_commit, which applies the identical deterministic commit on
 * every replica. dyg_shard_begin returns nq_max for both kinds -- upper
 * bounds of the query counts (the batch's insertions and deletions), so the
 * caller sizes buffers without a host round trip; the exact counts stay on
 * the device. Begin and walk only enqueue (stream order); validation errors
 * surface at dyg_shard_commit. The event and position buffers passed to dyg_shard_begin
 * must stay valid until the batch's commit is reported -- dyg_shard_commit, or
 * dyg_shard_finish after dyg_shard_commit_async (error messages read them).
 * While asynchronous commits are pending, every other entry point that reads
 * or writes the session's state fails with DYG_ERR_USAGE, and
 * dyg_update_counter / dyg_last_event_steps report the last settled state.
 * The session stream may be replaced by the caller's (dyg_set_stream) so
 * the collective is stream-ordered with the kernels. */
int dyg_set_stream(dyg_session* s, void* cuda_stream);
int dyg_shard_begin(dyg_session* s, const dyg_event* events, const uint64_t* positions,
                    size_t n, uint32_t batch_index, uint64_t* n_reach, uint64_t* n_minpath);
/* The same for batch `batch_index` of the stream given to dyg_stream_upload
 * (device-resident events: no per-batch upload). */
int dyg_shard_begin_uploaded(dyg_session* s, uint32_t batch_index, uint64_t* n_reach,
                             uint64_t* n_minpath);
size_t dyg_shard_record_bytes(const dyg_session* s, int minpath);
/* Enqueues this rank's walk and record packing on the session stream and
 * returns without waiting: consume the records in stream order (or
 * synchronise first). */
int dyg_shard_walk(dyg_session* s, int rank, int world, void* reach_records,
                   void* minpath_records);
int dyg_shard_commit(dyg_session* s, int world, const void* reach_gathered,
                     const void* minpath_gathered, dyg_batch_report* out);
/* The commit enqueued without waiting: the next dyg_shard_begin plans its
 * update counter and pool headroom past it, so a whole range of batches is
 * enqueued with no host round trip (a failed batch raises the device abort
 * flag and the later ones do nothing, as in dyg_replay_uploaded_range).
 * dyg_shard_finish waits, then returns the pending batches' reports in order
 * (up to `cap`; *n_out = reports produced) and fails at the first failing
 * batch. At most 256 commits may be pending. */
int dyg_shard_commit_async(dyg_session* s, int world, const void* reach_gathered,
                           const void* minpath_gathered);
int dyg_shard_finish(dyg_session* s, dyg_batch_report* out, size_t cap, size_t* n_out);

/* Peer-memory exchange for the split (the B200 path; NCCL not involved):
 * every rank packs its walk records into its OWN exchange area and
 * publishes them with a system-scope release of a per-batch epoch; every
 * rank then reads each peer's records straight from the peer's area (P2P
 * loads over NVLink through CUDA IPC mappings) once that peer's epoch has
 * arrived. A batch's prepare, walk, pack, publish, wait, unpack and commit
 * are all kernels, so a range of uploaded batches is one captured graph
 * with no host step between them.
 *   dyg_shard_peer_create: (re)allocates this rank's area for batches of up
 *     to max_reach insertions / max_minpath deletions split `world` ways;
 *     returns the area, its size and (ipc_handle non-null) its 64-byte CUDA
 *     IPC handle for the other ranks.
 *   dyg_ipc_open / dyg_ipc_close: map / unmap a peer's area on `device`.
 *   dyg_shard_peer_bind: areas[q] = rank q's area as this device sees it
 *     (areas[rank] = the own area). A peer that does not publish within
 *     timeout_s seconds (<= 0: 30 s) fails the batch with DYG_ERR_DEVICE.
 *   dyg_shard_peer_range_begin / _end: enqueue the uploaded batches
 *     [first, first + count) (dyg_stream_upload*) / synchronise and report
 *     them (the first failing batch's error, as dyg_replay_uploaded_range).
 * Every rank must run the same ranges in the same order. Ranks are
 * separate processes (one per GPU; several may share a GPU, whose contexts
 * then time-slice): two sessions of ONE process must not be peers, since a
 * rank's wait kernel could then hold SM resources another rank's
 * cooperative commit needs (the exchange would time out). */
int dyg_shard_peer_create(dyg_session* s, int world, uint64_t max_reach, uint64_t max_minpath,
                          void** area, size_t* bytes, void* ipc_handle);
int dyg_ipc_open(const void* ipc_handle, int device, void** ptr);
int dyg_ipc_close(void* ptr);
int dyg_shard_peer_bind(dyg_session* s, int rank, int world, void* const* areas, double timeout_s);
int dyg_shard_peer_range_begin(dyg_session* s, uint32_t first, uint32_t count);
int dyg_shard_peer_range_end(dyg_session* s, dyg_batch_report* out, size_t cap, size_t* n_out);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* DYG_H */
