// batch.cuh -- device side of replay_batch_deferred
// (proj/src/sparsifier.cpp:395-539), minus the walks (walk.cuh).
//
// Kernel map (SURVEY.md 2 kernel table):
//   k_validate        validate_event_shape (sparsifier.cpp:321-337)
//   ShadowOp rounds   shadow G = batch-start G minus the batch's deletions in
//                     event order (sparsifier.cpp:416-423)          [K5]
//   k_flags/k_scatter query build (sparsifier.cpp:429-457)           [K4]
//   CommitOp rounds   the sequential commit (sparsifier.cpp:466-533)
//                     incl. commit_insertion / set_edge_weight
//                     (:207-241) and run_local_fallback (:264-280)  [K6-K8]
//   batch_finish      BatchReport counters (sparsifier.hpp:44-59), run at
//                     the end of the commit launch                   [K9]
//
// The commit engine ("dependency rounds"): every round, each pending event
// reserves all rows it will read or write (atomicMax of a round-stamped key
// that prefers the lowest event index); an event that won all its rows
// applies, with exactly the reference's per-event operations. Events that
// touch disjoint rows commute, and an event only applies after every
// earlier event sharing a row, so the final rows equal the sequential
// event-order commit bit for bit. One cooperative launch runs all rounds.
#pragma once

#include "walk.cuh"

namespace dyg {

constexpr uint32_t kNoSlot = 0xFFFFFFFFu;

struct DevEvent {   // dyg_event / EdgeEvent (stream.hpp:11-18)
  uint32_t kind;    // 0 insertion, 1 deletion
  uint32_t u, v;
  uint32_t batch_index;
  double weight;
};

// Report counters in BatchReport order (sparsifier.hpp:46-55).
enum ReportField {
  kInsSeen = 0, kInsKept, kInsPruned, kDelSeen, kDelInH, kPaths, kEdgesRec, kFallbacks,
  kWalkerSteps, kMaxEventSteps, kReportFields
};

// Validation error codes (packed as (k << 8) | code into err keys).
enum EventError : uint32_t {
  kErrRange = 1,       // "vertex id out of range"
  kErrSelfLoop = 2,    // "self-loop"
  kErrWeight = 3,      // "non-positive weight"
  kErrAbsent = 4,      // delete_edge: "edge (u, v) does not exist"
  kErrPool = 5,        // overflow pool exhausted (device)
  kErrAborted = 6,     // an earlier batch of the same enqueued range failed
  kErrPeer = 7,        // a peer never published its walk records (multi-GPU exchange)
};

struct BatchCtl {
  unsigned long long val_err;     // min (k << 8 | code) from validation
  unsigned long long commit_err;  // min (k << 8 | code) from the commit
  unsigned int first_absent;      // min k whose deletion found no shadow edge
  unsigned int limit;             // commit only events k < limit
  unsigned int use_absent_limit;  // deletion-only batch: also k < first_absent
  unsigned int nq_reach;
  unsigned int nq_min;
  unsigned int remaining[3];
  unsigned int rounds;
  unsigned long long report[kReportFields];
  WalkCounters reach;
  WalkCounters minpath;
  unsigned long long g_edges, h_edges, g_pool_top, h_pool_top;
  unsigned int n_saved;  // rows saved for the in-place walk shadow
  unsigned long long side_top;       // side-pool entries used by saved rows
  unsigned long long scratch_edges;  // |E| sink of the shadow pass
  unsigned int fast;                 // insertion fast path attempted
  unsigned int not_simple;           // fast-path precondition violated
  unsigned long long fp_report[kReportFields];
  // Dataflow commit of deletion-only batches (k_del_flow).
  unsigned int fl_top;       // row records handed out
  unsigned int fl_next_ev;   // next event to take (in event order)
  unsigned int fl_overflow;  // record buffer too small: the round engine commits
  unsigned int flow_done;    // k_del_flow committed the batch
  unsigned int fl_changed[3];  // fallback-promotion fixpoint (rotating)
  unsigned int fl_depth;     // longest chain of row-sharing events
  unsigned int fl_blocks_done;  // k_del_flow blocks past the reset (the last one runs the epilogue)
  unsigned int fl_any_fb;       // some event may run the local fallback (else no promotion fixpoint)
  unsigned long long fl_t[6];  // %globaltimer at the phase boundaries
  unsigned long long counter_base;  // update_counter_ at batch start (:431)
  // %globaltimer stamps (ns) for the phase times in dyg_stats.
  unsigned long long t_batch0;   // k_ctl_init
  unsigned long long t_commit0;  // first commit kernel (min over blocks)
  unsigned long long t_mp_end;   // k_minpath_finish end (max over blocks)
  unsigned long long t_batch1;   // batch epilogue
  unsigned long long t_prep0, t_prep1;  // k_prep first block start / last block end
  unsigned long long epoch;      // unique per batch (single-pass scan tile states)
  unsigned int tile_ctr;         // single-pass scan: next tile
  unsigned int nq_long;        // reach queries in the low slots (walk-order split)
};

// Arguments of the batch control-block initialisation kernel: the only
// per-batch values a captured batch graph has to be re-pointed with.
struct CtlInitArgs {
  BatchCtl* ctl;
  unsigned long long* epoch_ctr;  // session counter: one epoch per batch
  uint32_t limit;
  uint32_t use_absent_limit;
  uint32_t fast;
  unsigned long long counter_base;
};

struct WalkOpts {
  double K;
  uint32_t T;
  uint32_t s;
  uint64_t seed;
  int filtering;   // K != 0 && !freeze (sparsifier.cpp:409-410)
  int freeze;
  // Engine selection (per session, from the environment at creation; the
  // alternatives are A/B and test knobs, all bit-identical):
  int fastpath;      // insertion fast path      (DYG_NO_FASTPATH disables)
  int single_pass;   // single-pass prepare      (DYG_SINGLE_PASS=0 disables)
  int shadow_lists;  // per-row shadow lists     (DYG_SHADOW_ROUNDS=1 disables)
  int flow;          // dataflow deletion commit (DYG_COMMIT_ROUNDS=1 disables)
  int keep_shadow;   // deletion-only batches keep the walk shadow as G (DYG_KEEP_SHADOW=0 disables)
  int flow_balance;  // deal the ordered events round-robin to warps (DYG_FLOW_BALANCE=0 disables)
  // Reach walk order (insertion-only, single-GPU batches): queries whose
  // w_pq <= split_wpq (the budget lets them walk longest) get the low slots and
  // are walked first, the rest take slots from the top of the buffer; 0 = off.
  double split_wpq;
  int count;  // instrumented walk kernels (per-step statistics), dyg_session_set_walk_counters
};

// Device buffers of one batch (sized by the session; grown on demand).
struct BatchDev {
  DevEvent* events;
  uint8_t* state;
  uint32_t* slot;
  unsigned long long* scan_in;
  unsigned long long* scan_out;
  ReachQuery* rq;
  MinQuery* mq;
  ReachOut rout;
  MinOut mout;
  MinScratch mscratch;
  uint32_t* dec;           // per-event outcome (kind | edges_added << 8)
  double* wpq;             // per-event insertion w_pq (batch-start G)
  // In-place walk shadow (k_sh_apply / k_save_rows save, the commit restores).
  uint32_t* mark;          // per-vertex batch stamp
  uint32_t* saved_rows;
  Slab<kCapG>* side_slab;
  unsigned long long* side_off;
  uint32_t* side_id;
  double* side_w;
  unsigned long long* side_top;       // = &ctl->side_top
  unsigned long long* scratch_edges;  // = &ctl->scratch_edges
  unsigned long long* locks;  // per-vertex row reservations
  unsigned long long* round_ctr;
  BatchCtl* ctl;
  unsigned int* abort_flag;  // session device abort flag (stops later batches)
  unsigned int* work;        // walk work counter (reset by k_scatter)
  // Single-pass (decoupled look-back) query scan: per 256-event tile,
  // {aggregate, inclusive, epoch << 2 | state}; state 1 = aggregate, 2 = inclusive.
  unsigned long long* tile_state;
  uint32_t q_cap;            // query slot capacity (reach slots are < q_cap)
  uint32_t n_vertices;
  ReachQuery* rq_sh;  // multi-GPU split: this rank's query range, moved to the front
  MinQuery* mq_sh;
  uint32_t* save_idx;        // per vertex: index of its saved batch-start G row
  void* scan_temp;
  size_t scan_temp_bytes_;
  // Insertion fast path ([0] = G, [1] = H): per-vertex append counts and
  // list heads (zero / kNoSlot between batches), per-record list links.
  uint32_t* fp_cnt[2];
  uint32_t* fp_head[2];
  uint32_t* fp_next[2];
  // Dataflow commit (k_del_flow): one record per (event, row) of the event's
  // row superset; per-event record ranges. Per-vertex list heads and done
  // counters reuse fp_head[0] / fp_cnt[0] (kNoSlot / 0 between batches).
  uint32_t* fl_row;
  uint32_t* fl_ev;
  uint32_t* fl_next;
  uint32_t* fl_rank;
  uint32_t* fl_base;
  uint32_t* fl_cnt;
  uint8_t* fl_promo;   // per event: may run the local fallback
  uint32_t* fl_heavy;  // bitmap: events the apply phase must order (0 between batches)
  uint32_t* fl_depth;  // per vertex, 0 between batches
  uint64_t fl_cap;
};

// Host launchers (batch.cu); each returns kernels launched.
int launch_ctl_init(const CtlInitArgs& a, cudaStream_t st);
int launch_set_u32x2(uint32_t* dst, uint32_t a, uint32_t b, cudaStream_t st);
// Multi-GPU split: rank's query ranges from the device counts (rng[0..3] =
// lo_r, n_r, lo_m, n_m) and the range's queries copied to rq_sh / mq_sh.
int launch_shard_range(const BatchDev& b, int rank, int world, uint32_t* rng, uint32_t max_r,
                       uint32_t max_m, cudaStream_t st);
// Graph support: is `n` a k_ctl_init kernel node (then *out = its args)?
bool ctl_init_node_args(cudaGraphNode_t n, CtlInitArgs* out);
cudaError_t ctl_init_node_update(cudaGraphExec_t ex, cudaGraphNode_t n, const CtlInitArgs& a);
int launch_count_kinds(const DevEvent* ev, uint32_t nb, uint32_t* out, cudaStream_t st);
// Per-event decisions of a committed batch in the ABI's codes
// (DYG_DECISION_*): insertions InsertionDecision (sparsifier.hpp:36),
// deletions 2 + DeletionOutcome::Kind (sparsifier.hpp:38-42).
int launch_export_decisions(const uint32_t* dec, const DevEvent* ev, uint32_t nb, uint8_t* out,
                            cudaStream_t st);
int launch_validate(const BatchDev& b, uint32_t nb, uint32_t n, const unsigned int* abort_flag,
                    cudaStream_t st);
// Validation + walk shadow + query build: single-pass kernels for
// insertion-only / deletion-only batches, else the chain below.
int launch_prepare(const DevGraph<kCapH>& H, DevGraph<kCapG> G, const BatchDev& b, uint32_t nb,
                   uint32_t n_del, uint32_t n, uint32_t stamp, const WalkOpts& o,
                   cudaStream_t st);
// Query build; with deletions in the batch it also saves the touched G
// rows and applies the walk shadow to G in place (undone at the start of
// the commit launch).
int launch_queries(const DevGraph<kCapH>& H, DevGraph<kCapG> G, const BatchDev& b,
                   uint32_t nb, uint32_t n_del, uint64_t counter, uint32_t stamp,
                   const WalkOpts& o, int coop_blocks, cudaStream_t st);
// Insertion-only fast path (ctl.fast set; the lists are built by k_prep):
// G appends (may run concurrently with the reach walk), then H appends and
// the per-event accounting after it; k_rounds only commits if a
// precondition failed on the device.
int launch_fastpath_g(const DevGraph<kCapG>& G, const BatchDev& b, uint32_t nb, cudaStream_t st);
// The whole commit in one cooperative launch, epilogue included: insertion
// batches k_rounds (fast-path appends, or rounds), deletion-only batches
// k_del_flow (shadow undo + dataflow commit), mixed batches k_rounds_warp.
// fp_h: an insertion-only fast-path batch -- the launch starts with the H
// appends (fp_write_h_pass), then the epilogue from its last block.
int launch_commit(const DevGraph<kCapG>& G, const DevGraph<kCapH>& H, const BatchDev& b,
                  uint32_t nb, uint32_t n_del, const WalkOpts& o, cudaStream_t st,
                  bool fp_h = false);
size_t scan_temp_bytes(uint32_t nb_cap);

// Multi-GPU exchange records. Reach: 16 B per query.
// MinPath: 24 B header + (T+1) u32 vertices, padded to 8 B.
struct ReachRecord {
  uint32_t reached;
  uint32_t pad;
  unsigned long long steps;
};
struct MinRecordHead {
  uint32_t has_path;
  uint32_t path_len;
  unsigned long long steps;
  double resistance;
};
__host__ __device__ inline size_t min_record_bytes(uint32_t T) {
  return (sizeof(MinRecordHead) + 4ull * (T + 1ull) + 7ull) & ~7ull;
}
// Pack this rank's queries [lo, hi) into `slots` records (rest zeroed).
int launch_pack(const BatchDev& b, const uint32_t* rng, uint32_t slots_r, uint32_t slots_m,
                uint32_t T, void* rrec, void* mrec, cudaStream_t st);
// Scatter rank-major gathered records back to query order.
int launch_unpack(const BatchDev& b, uint32_t max_r, uint32_t max_m, int world, uint32_t slots_r,
                  uint32_t slots_m, uint32_t T, const void* rrec, const void* mrec,
                  cudaStream_t st);
// Co-resident blocks for the cooperative round kernels.
int coop_grid_blocks(int device);

// ---- peer-memory exchange of the multi-GPU split ----------
// Instead of an NCCL all-gather between two host calls, every rank packs its
// walk records into its OWN exchange area, publishes them with a
// system-scope release of its `ready` epoch, and reads every peer's records
// straight from the peer's area (P2P loads over NVLink, CUDA IPC mappings)
// once that peer's `ready` reaches the batch's epoch. All of it is kernels,
// so a whole sharded batch -- prepare, walk, pack, signal, wait, unpack,
// commit -- is one captured graph with no host step in between.
// Area layout: [0, 256) the ready epoch (u64 at 0); then two parity
// buffers of `stride` bytes (reach records, then min-path records at
// min_off). Batch epoch e uses parity e & 1; a rank writes parity buffer
// e & 1 again only at epoch e + 2, after it has seen every peer's ready
// reach e + 1, and a peer publishes e + 1 only after its unpack of e
// finished (stream order): two buffers suffice.
constexpr int kMaxPeers = 16;
constexpr size_t kPeerHeader = 256;
struct PeerX {
  uint8_t* own;                    // this rank's area (device memory)
  const uint8_t* base[kMaxPeers];  // every rank's area as this device sees it
  unsigned long long* ep;          // this rank's epoch (local device counter)
  unsigned long long stride;       // bytes per parity buffer
  unsigned long long min_off;      // min-path records within a parity buffer
  int world;
  int rank;
  unsigned long long timeout_ns;   // a peer that never publishes fails the batch
};
size_t peer_area_bytes(uint32_t slots_r, uint32_t slots_m, uint32_t T, size_t* stride,
                       size_t* min_off);
// Pack into the own area's next parity buffer, then publish (signal).
int launch_pack_peer(const BatchDev& b, const uint32_t* rng, uint32_t slots_r, uint32_t slots_m,
                     uint32_t T, const PeerX& px, cudaStream_t st);
// Wait for every peer's epoch, then unpack from the peers' areas.
int launch_unpack_peer(const BatchDev& b, uint32_t max_r, uint32_t max_m, uint32_t slots_r,
                       uint32_t slots_m, uint32_t T, const PeerX& px, cudaStream_t st);

}  // namespace dyg
