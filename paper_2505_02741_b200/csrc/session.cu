// session.cu -- the C-ABI (include/dyg.h): device session lifecycle, the
// per-batch pipeline of replay_batch_deferred (sparsifier.cpp:395-539),
// immediate mode as 1-event batches, the stateless
// run_batch twin, exports and snapshots.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#include "../../include/dyg.h"
#include "batch.cuh"
#include "graph_store.cuh"
#include "spectral.cuh"
#include "stream_gen.cuh"

using namespace dyg;

namespace {

thread_local std::string g_last_error;

struct ApiError {
  int code;
  std::string message;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw ApiError{code, msg}; }

template <typename F>
int guarded(F&& f) {
  try {
    // Launch checks read cudaGetLastError(): start every entry point from a
    // clean slate so a non-sticky error left by an earlier unchecked call
    // (e.g. a free during teardown) is not misattributed.
    cudaGetLastError();
    f();
    return DYG_OK;
  } catch (const ApiError& e) {
    g_last_error = e.message;
    return e.code;
  } catch (const DeviceError& e) {
    g_last_error = e.message;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return DYG_ERR_DEVICE;
  }
}

void check(cudaError_t e, const char* what) { cuda_check(e, what); }

template <typename T>
void dev_alloc(T** p, size_t count, const char* what) {
  check(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<size_t>(count, 1)), what);
}
template <typename T>
void dev_free(T*& p) {
  cudaFree(p);
  p = nullptr;
}

// Milliseconds between two %globaltimer stamps (0 when a phase did not run).
double span_ms(unsigned long long a, unsigned long long b) {
  return (a != ~0ull && a != 0 && b > a) ? (b - a) * 1e-6 : 0.0;
}

double density_of(uint64_t edges, uint32_t n) {
  return static_cast<double>(edges) / static_cast<double>(n) - 1.0;  // graph.cpp:114-116
}


// One instantiated CUDA graph of an enqueue sequence. Its only per-launch
// input is the update counter, carried by the k_ctl_init nodes.
struct CapturedGraph {
  uint64_t key = 0;
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;        // kept: node handles refer to it
  std::vector<cudaGraphNode_t> ctl_nodes;
  std::vector<CtlInitArgs> ctl_args;  // as captured
  uint64_t cap_base = 0;              // update counter at capture
  uint64_t base = 0;                  // update counter the nodes currently hold
  int launches = 0;
  std::vector<int> per_batch;  // range graphs: kernels per batch
  uint64_t last_use = 0;
};

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  return h;
}

}  // namespace

namespace {
struct Pending;  // one batch in flight (below)
}  // namespace

struct dyg_session {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  dyg_options opt{};
  uint32_t n = 0;
  int coop_blocks = 0;

  GraphStore<kCapG> G, G_snap;
  GraphStore<kCapH> H, H_snap;
  uint64_t counter = 0, counter_snap = 0;
  uint64_t g_edges = 0, h_edges = 0, g_top = 0, h_top = 0;
  uint64_t g_edges_snap = 0, h_edges_snap = 0, g_top_snap = 0, h_top_snap = 0;
  bool have_snap = false;
  uint64_t last_event_steps = 0;

  // Batch buffers.
  BatchDev b{};
  uint32_t nb_cap = 0, nd_cap = 0;
  unsigned long long* d_locks = nullptr;
  unsigned long long* d_round = nullptr;
  unsigned int* d_work = nullptr;  // walk work counter
  uint64_t side_cap = 0;           // side-pool entries allocated
  uint32_t stamp = 0;              // batch stamp for the row-save marks
  DevEvent* d_events = nullptr;
  DevEvent* h_events_pinned = nullptr;
  BatchCtl* h_ctl = nullptr;
  BatchCtl* d_ctl = nullptr;  // the single-batch control block (b.ctl is re-pointed per batch)

  // Device-resident stream.
  DevEvent* d_stream = nullptr;
  std::vector<dyg_event> stream_events;      // sorted by batch (stable)
  std::vector<uint64_t> stream_positions;    // original stream index
  std::vector<uint64_t> batch_off, batch_cnt, batch_ins, batch_del;
  uint32_t stream_batches = 0;
  bool have_stream = false;

  // Last-batch outputs (immediate mode / apply_*).
  uint32_t last_dec = 0;
  // Per-event decisions requested by the caller (device staging and its
  // pinned host copy, one byte per event of a batch / range / stream).
  uint8_t* d_dec = nullptr;
  uint8_t* h_dec = nullptr;
  uint64_t dec_cap = 0;
  uint32_t* d_counts = nullptr;   // [2..3] batch kind counts, [4..7] shard ranges
  uint32_t* h_counts = nullptr;   // pinned: [0..1] shard counts, [2] decision, [4..5] kinds
  // Multi-GPU split state (dyg_shard_*).
  bool shard_active = false;
  const DevEvent* shard_host = nullptr;  // caller's buffers, valid until dyg_shard_commit
  const DevEvent* shard_dev = nullptr;   // the batch's events on the device
  const uint64_t* shard_pos = nullptr;
  uint64_t shard_pos_base = 0;           // stream position of event 0 when shard_pos is null
  uint32_t shard_nb = 0, shard_ins = 0, shard_del = 0, shard_batch = 0;
  uint32_t shard_nq_r = 0, shard_nq_m = 0;
  std::chrono::steady_clock::time_point shard_wall0;
  int shard_launches = 0;
  uint64_t shard_counter = 0;
  // Asynchronous shard commits (dyg_shard_commit_async) not yet finalised:
  // their control blocks land in a pinned ring; the next batch plans its
  // update counter and pool headroom past them.
  std::vector<Pending> shard_pending;
  BatchCtl* h_shard_ctls = nullptr;
  uint64_t shard_next_counter = 0;
  uint64_t shard_pend_g = 0, shard_pend_h = 0;
  // The shard batch's record unpack (enqueued with its commit) and a key of
  // everything it bakes into kernel arguments.
  std::function<int(dyg_session*)> shard_unpack;
  uint64_t shard_unpack_key = 0;
  // Peer-memory exchange (dyg_shard_peer_*, batch.cuh PeerX): this rank's
  // exchange area and epoch, the bound view of every rank's area, and the
  // batches of an enqueued peer range awaiting dyg_shard_peer_range_end.
  uint8_t* px_area = nullptr;
  size_t px_bytes = 0, px_stride = 0, px_min_off = 0;
  uint32_t px_slots_r = 0, px_slots_m = 0, px_world = 0;
  unsigned long long* px_ep = nullptr;
  PeerX px{};
  bool px_bound = false;
  std::vector<Pending> px_pending;
  uint32_t px_first = 0;

  dyg_stats stats{};
  BatchCtl* d_ctls = nullptr;      // batch-range control blocks
  BatchCtl* h_ctls = nullptr;
  uint32_t ctl_cap = 0;
  unsigned int* d_abort = nullptr; // set by a failing batch; later batches no-op
  bool debug_sync = false;
  // Captured device sequences (one batch, or a whole uploaded range), keyed
  // by a fingerprint of everything baked into their kernel arguments.
  std::vector<CapturedGraph> graphs;
  bool graphs_on = true;   // DYG_GRAPHS=0 disables; a failed capture disables
  bool capturing = false;
  uint64_t graph_clock = 0;
  unsigned long long* d_epoch = nullptr;  // batch epochs (single-pass scan tile states)
  uint64_t stream_gen = 0;  // fingerprint of the uploaded stream's batch structure
  uint64_t stream_cap = 0;  // events d_stream can hold
  // dyg_replay_stream: host stream replayed with its upload pipelined.
  cudaStream_t copy_stream = nullptr;
  cudaStream_t aux_stream = nullptr;  // fork target inside a batch
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevEvent* d_replay = nullptr;
  uint64_t replay_cap = 0;
  uint32_t* d_kinds = nullptr;
  uint32_t* h_kinds = nullptr;
  uint64_t kinds_cap = 0;
  std::vector<cudaEvent_t> ready;
  // dyg_stream_upload_batches: per-batch uploads + device kind counts on the
  // copy stream; batch_ins / batch_del are filled as each batch lands.
  std::vector<cudaEvent_t> up_ready;
  std::vector<uint8_t> up_settled;
  uint32_t* d_up_kinds = nullptr;
  uint32_t* h_up_kinds = nullptr;
  uint64_t up_kinds_cap = 0;
  bool up_pending = false;
  cudaEvent_t ev_up_fence = nullptr;
  bool no_fastpath = false;        // DYG_NO_FASTPATH: force the round engine
  bool single_pass = true;         // DYG_SINGLE_PASS=0: multi-kernel prepare chain
  bool shadow_lists = true;        // DYG_SHADOW_ROUNDS=1: dependency-round walk shadow
  bool flow = true;                // DYG_COMMIT_ROUNDS=1: round-engine deletion commit
  uint64_t flow_cap = 0;           // DYG_FLOW_CAP: flow record capacity (test knob)
  bool reach_split = true;         // DYG_REACH_SPLIT=0: reach walks in slot order
  bool keep_shadow = true;         // DYG_KEEP_SHADOW=0: deletion commit restores G
  bool flow_balance = true;        // DYG_FLOW_BALANCE=0: static event ownership
  bool walk_counters = false;      // dyg_session_set_walk_counters: instrumented walks
  unsigned long long last_t1 = 0;  // end stamp of the previous batch (stats)
  double mean_inv_w = 1.0;         // mean 1/w over G's edges (session creation)
};

namespace {


void maybe_sync(dyg_session* s, const char* what) {
  if (s->debug_sync) check(cudaStreamSynchronize(s->stream), what);
  else check(cudaGetLastError(), what);
}

void free_batch(dyg_session* s) {
  BatchDev& b = s->b;
  dev_free(b.state);
  dev_free(b.slot);
  dev_free(b.scan_in);
  dev_free(b.scan_out);
  dev_free(b.rq);
  dev_free(b.mq);
  dev_free(b.rq_sh);
  dev_free(b.mq_sh);
  dev_free(b.rout.reached);
  dev_free(b.rout.steps);
  dev_free(b.rout.best_bits);
  dev_free(b.mout.has_path);
  dev_free(b.mout.path_len);
  dev_free(b.mout.steps);
  dev_free(b.mout.resistance);
  dev_free(b.mout.paths);
  dev_free(b.mscratch.acc);
  dev_free(b.mscratch.term);
  dev_free(b.mscratch.steps);
  dev_free(b.mscratch.paths);
  dev_free(b.mscratch.rvals);
  dev_free(b.fl_row);
  dev_free(b.fl_ev);
  dev_free(b.fl_next);
  dev_free(b.fl_rank);
  dev_free(b.dec);
  dev_free(b.wpq);
  dev_free(b.saved_rows);
  dev_free(b.side_slab);
  dev_free(b.side_off);
  for (int i = 0; i < 2; ++i) dev_free(b.fp_next[i]);
  dev_free(b.fl_base);
  dev_free(b.fl_cnt);
  dev_free(b.fl_promo);
  dev_free(b.fl_heavy);
  dev_free(b.tile_state);
  cudaFree(b.scan_temp);
  b.scan_temp = nullptr;
  dev_free(s->d_events);
  if (s->h_events_pinned) cudaFreeHost(s->h_events_pinned);
  s->h_events_pinned = nullptr;
  s->nb_cap = s->nd_cap = 0;
}

// Sizes the batch buffers for nb events of which nd are deletions.
void ensure_batch(dyg_session* s, uint32_t nb, uint32_t nd) {
  BatchDev& b = s->b;
  const uint64_t T1 = static_cast<uint64_t>(s->opt.walk.step_cap) + 1;
  const uint64_t sw = s->opt.walk.walker_count;
  if (nb > s->nb_cap) {
    const uint32_t cap = std::max<uint32_t>(nb, 1024);
    const uint32_t keep_nd = s->nd_cap;
    free_batch(s);
    dev_alloc(&b.state, cap, "batch state");
    dev_alloc(&b.slot, cap, "batch slots");
    dev_alloc(&b.scan_in, cap, "batch scan");
    dev_alloc(&b.scan_out, cap, "batch scan");
    dev_alloc(&b.rq, cap, "reach queries");
    dev_alloc(&b.mq, cap, "minpath queries");
    dev_alloc(&b.rq_sh, cap, "shard reach queries");
    dev_alloc(&b.mq_sh, cap, "shard minpath queries");
    dev_alloc(&b.rout.reached, cap, "reach out");
    dev_alloc(&b.rout.steps, cap, "reach out");
    dev_alloc(&b.rout.best_bits, cap, "reach out");
    dev_alloc(&b.dec, cap, "decisions");
    dev_alloc(&b.wpq, cap, "w_pq");
    dev_alloc(&b.saved_rows, 2ull * cap, "saved rows");
    dev_alloc(&b.side_slab, 2ull * cap, "saved slabs");
    dev_alloc(&b.side_off, 2ull * cap, "saved offsets");
    dev_alloc(&s->d_events, cap, "batch events");
    check(cudaMallocHost(reinterpret_cast<void**>(&s->h_events_pinned), sizeof(DevEvent) * cap),
          "pinned events");
    b.scan_temp_bytes_ = scan_temp_bytes(cap);
    check(cudaMalloc(&b.scan_temp, std::max<size_t>(b.scan_temp_bytes_, 16)), "scan temp");
    for (int i = 0; i < 2; ++i) dev_alloc(&b.fp_next[i], 2ull * cap, "append links");
    dev_alloc(&b.fl_base, cap, "flow record ranges");
    dev_alloc(&b.fl_cnt, cap, "flow record ranges");
    dev_alloc(&b.fl_promo, cap, "flow fallback flags");
    dev_alloc(&b.fl_heavy, cap / 32 + 2, "flow heavy bitmap");
    check(cudaMemset(b.fl_heavy, 0, sizeof(uint32_t) * (cap / 32 + 2)), "flow heavy bitmap");
    b.q_cap = cap;
    dev_alloc(&b.tile_state, 3ull * (cap / 256 + 2), "scan tile states");
    check(cudaMemset(b.tile_state, 0, sizeof(unsigned long long) * 3ull * (cap / 256 + 2)),
          "scan tile states");
    s->nb_cap = cap;
    s->nd_cap = 0;
    (void)keep_nd;
  }
  if (nd > s->nd_cap || b.mout.has_path == nullptr) {
    const uint32_t cap = std::max<uint32_t>(nd, 256);
    dev_free(b.mout.has_path);
    dev_free(b.mout.path_len);
    dev_free(b.mout.steps);
    dev_free(b.mout.resistance);
    dev_free(b.mout.paths);
    dev_free(b.mscratch.acc);
    dev_free(b.mscratch.term);
    dev_free(b.mscratch.steps);
    dev_free(b.mscratch.paths);
    dev_free(b.mscratch.rvals);
    dev_alloc(&b.mout.has_path, cap, "minpath out");
    dev_alloc(&b.mout.path_len, cap, "minpath out");
    dev_alloc(&b.mout.steps, cap, "minpath out");
    dev_alloc(&b.mout.resistance, cap, "minpath out");
    dev_alloc(&b.mout.paths, cap * T1, "minpath paths");
    dev_alloc(&b.mscratch.acc, cap * sw, "minpath scratch");
    dev_alloc(&b.mscratch.term, cap * sw, "minpath scratch");
    dev_alloc(&b.mscratch.steps, cap * sw, "minpath scratch");
    dev_alloc(&b.mscratch.paths, cap * sw * trace_stride(s->opt.walk.step_cap), "minpath traces");
    dev_alloc(&b.mscratch.rvals, cap * T1, "minpath scratch");
    // Flow records: u, v and a path of <= T+1 vertices or two G rows per
    // deletion; overflow falls back to the round engine.
    dev_free(b.fl_row);
    dev_free(b.fl_ev);
    dev_free(b.fl_next);
    dev_free(b.fl_rank);
    b.fl_cap = s->flow_cap ? s->flow_cap : static_cast<uint64_t>(cap) * 48 + 65536;
    dev_alloc(&b.fl_row, b.fl_cap, "flow records");
    dev_alloc(&b.fl_ev, b.fl_cap, "flow records");
    dev_alloc(&b.fl_next, b.fl_cap, "flow records");
    dev_alloc(&b.fl_rank, b.fl_cap, "flow records");
    s->nd_cap = cap;
  }
}

// Side pool for saved overflow rows: bounded by G's pool (each row is saved
// at most once per batch).
void ensure_side_pool(dyg_session* s) {
  const uint64_t need = s->G.pool_capacity();
  if (s->side_cap >= need && s->b.side_id != nullptr) return;
  dev_free(s->b.side_id);
  dev_free(s->b.side_w);
  dev_alloc(&s->b.side_id, need, "side pool");
  dev_alloc(&s->b.side_w, need, "side pool");
  s->side_cap = need;
}

WalkOpts walk_opts(const dyg_session* s) {
  WalkOpts o;
  o.K = s->opt.walk.distortion_threshold;
  o.T = s->opt.walk.step_cap;
  o.s = s->opt.walk.walker_count;
  o.seed = s->opt.walk.global_seed;
  o.freeze = s->opt.freeze_sparsifier != 0;
  o.filtering = (o.K != 0.0 && !o.freeze) ? 1 : 0;  // sparsifier.cpp:409-410
  o.fastpath = s->no_fastpath ? 0 : 1;
  o.single_pass = s->single_pass ? 1 : 0;
  o.shadow_lists = s->shadow_lists ? 1 : 0;
  o.flow = s->flow ? 1 : 0;
  // Walk-order split threshold: a walker's acc grows by ~E[1/w] per step, so
  // the budget K / w_pq allows >= 0.8 T steps when w_pq <= K / (0.8 T E[1/w]).
  o.split_wpq = (s->reach_split && o.filtering && o.T > 0)
                    ? o.K / (0.8 * static_cast<double>(o.T) * s->mean_inv_w) : 0.0;
  o.keep_shadow = s->keep_shadow ? 1 : 0;
  o.count = s->walk_counters ? 1 : 0;
  o.flow_balance = s->flow_balance ? 1 : 0;
  return o;
}

std::string event_error_message(uint32_t code, uint64_t pos, const DevEvent& e) {
  char buf[256];
  switch (code) {
    case kErrRange:
      std::snprintf(buf, sizeof buf, "event %llu: vertex id out of range",
                    static_cast<unsigned long long>(pos));
      break;
    case kErrSelfLoop:
      std::snprintf(buf, sizeof buf, "event %llu: self-loop", static_cast<unsigned long long>(pos));
      break;
    case kErrWeight:
      std::snprintf(buf, sizeof buf, "event %llu: non-positive weight",
                    static_cast<unsigned long long>(pos));
      break;
    case kErrAbsent:
      std::snprintf(buf, sizeof buf, "event %llu: edge (%u, %u) does not exist",
                    static_cast<unsigned long long>(pos), e.u, e.v);
      break;
    default:
      std::snprintf(buf, sizeof buf, "event %llu: overflow pool exhausted",
                    static_cast<unsigned long long>(pos));
  }
  return buf;
}

// One deferred batch in phases, so the multi-GPU split (dyg_shard_*) can
// run the walk phase on a query range and exchange results before the
// replicated commit, and so a device-resident stream can enqueue many
// batches back to back with a single host sync (dyg_replay_uploaded_range).
struct Pending {
  const DevEvent* dev = nullptr;
  const DevEvent* host = nullptr;
  const uint64_t* pos = nullptr;
  uint64_t pos_base = 0;      // stream position of event 0 when pos is null
  uint32_t nb = 0, n_ins = 0, n_del = 0, batch = 0;
  bool imm_msgs = false;
  std::chrono::steady_clock::time_point wall0;
  int launches = 0;
  BatchCtl* dctl = nullptr;   // device control block of this batch
  BatchCtl* hctl = nullptr;   // pinned host copy
  uint32_t* hdec = nullptr;   // pinned: decision of a 1-event batch
  uint64_t counter_base = 0;  // update_counter at batch start
  bool g_appended = false;    // fast path: G appends already enqueued (forked)
  bool shard = false;         // multi-GPU split batch (dyg_shard_*)
  // Per-event decisions (nullable): the commit exports them to dec_dev and
  // copies them to dec_pin; deliver_decisions writes the caller's buffer at
  // dec_dst[k] (dec_idx null) or dec_dst[dec_idx[k]].
  uint8_t* dec_dev = nullptr;
  uint8_t* dec_pin = nullptr;
  uint8_t* dec_dst = nullptr;
  const uint64_t* dec_idx = nullptr;
};

// Staging for up to `n` per-event decisions.
void ensure_decisions(dyg_session* s, uint64_t n) {
  if (n <= s->dec_cap) return;
  if (s->d_dec) cudaFree(s->d_dec);
  if (s->h_dec) cudaFreeHost(s->h_dec);
  s->d_dec = nullptr;
  s->h_dec = nullptr;
  s->dec_cap = 0;
  check(cudaMalloc(reinterpret_cast<void**>(&s->d_dec), n), "decision staging");
  check(cudaMallocHost(reinterpret_cast<void**>(&s->h_dec), n), "pinned decisions");
  s->dec_cap = n;
}

// After the batch's stream work has completed and BEFORE commit_finalize
// (which throws for a failing batch): the events that committed get their
// decisions, the rest (a validation error, the failing event and those
// after it, :525-529) keep DYG_DECISION_NONE.
void deliver_decisions(const Pending& p) {
  if (p.dec_dst == nullptr || p.nb == 0) return;
  const BatchCtl& c = *p.hctl;
  uint64_t lim = p.nb;
  if (c.val_err != ~0ull) lim = 0;
  if (c.commit_err != ~0ull) lim = std::min<uint64_t>(lim, c.commit_err >> 8);
  if (c.use_absent_limit && c.first_absent != 0xFFFFFFFFu)
    lim = std::min<uint64_t>(lim, c.first_absent);
  for (uint64_t k = 0; k < p.nb; ++k)
    p.dec_dst[p.dec_idx ? p.dec_idx[k] : k] = k < lim ? p.dec_pin[k] : DYG_DECISION_NONE;
}

void bind_pending(dyg_session* s, Pending& p) {
  p.dctl = s->d_ctl;
  p.hctl = s->h_ctl;
  p.hdec = &s->h_counts[2];
  p.counter_base = s->counter;
}

// Event k of a pending batch for an error message: the host copy when there
// is one, else read back from the device (uploaded streams keep no host copy
// when they were DMA'd straight from the caller's page-locked buffer).
DevEvent event_at(const Pending& p, uint64_t k) {
  if (p.host) return p.host[k];
  DevEvent e{};
  check(cudaMemcpy(&e, p.dev + k, sizeof e, cudaMemcpyDeviceToHost), "event read-back");
  return e;
}

[[noreturn]] void fail_validation(dyg_session* s, const Pending& p, unsigned long long val_err) {
  const uint32_t k = static_cast<uint32_t>(val_err >> 8);
  const uint64_t pos = p.pos ? p.pos[k] : p.pos_base + k;
  std::string msg = event_error_message(static_cast<uint32_t>(val_err & 0xFF), pos, event_at(p, k));
  if (p.imm_msgs) {
    char pre[64];
    std::snprintf(pre, sizeof pre, "event %llu: ", static_cast<unsigned long long>(pos));
    msg = pre + msg;  // sparsifier.cpp:479+503-507 rewraps validate's message
  }
  (void)s;
  fail(DYG_ERR_DATA, msg);
}

// Pool headroom for appends of n_ins insertions and n_del deletions
// (sparsifier.cpp:474,483,503-519), with a 4x factor for relocations.
void ensure_pools(dyg_session* s, uint64_t n_ins, uint64_t n_del) {
  const uint64_t T1 = static_cast<uint64_t>(s->opt.walk.step_cap) + 1;
  const uint64_t g_app = 2ull * n_ins;
  const uint64_t h_app = 2ull * n_ins + n_del * (2 * T1 + 4);
  // (+ the worst-case appends of asynchronous shard commits not yet read back)
  s->G.ensure_pool(s->g_top + s->shard_pend_g, 4 * g_app + (1u << 16), s->stream);
  s->H.ensure_pool(s->h_top + s->shard_pend_h, 4 * h_app + (1u << 16), s->stream);
}

// validate (:405-407), walk shadow (:416-423), query build (:429-457).
// Buffers sized and the host-side batch binding (s->b) pointed at this
// batch: everything phase_prepare does besides enqueueing. Called before a
// capture too (nothing may allocate inside one, and a replayed graph does
// not re-run the host side).
void prepare_bind(dyg_session* s, const Pending& p) {
  ensure_batch(s, p.nb, p.n_del);
  ensure_pools(s, p.n_ins, p.n_del);
  BatchDev& b = s->b;
  b.ctl = p.dctl;
  b.events = const_cast<DevEvent*>(p.dev);
  b.locks = s->d_locks;
  b.round_ctr = s->d_round;
  b.abort_flag = s->d_abort;
  b.work = s->d_work;
  b.side_top = &b.ctl->side_top;
  b.scratch_edges = &b.ctl->scratch_edges;
  if (p.n_del > 0) ensure_side_pool(s);
}

void phase_prepare(dyg_session* s, Pending& p) {
  WalkOpts o = walk_opts(s);
  if (p.shard) o.split_wpq = 0.0;  // shard ranges need contiguous reach slots
  prepare_bind(s, p);
  BatchDev& b = s->b;
  const uint32_t use_absent_limit = (p.n_ins == 0 && p.n_del > 0) ? 1u : 0u;
  const uint32_t fast =
      (p.n_del == 0 && p.n_ins > 0 && o.fastpath && o.single_pass) ? 1u : 0u;
  p.launches += launch_ctl_init(
      CtlInitArgs{b.ctl, s->d_epoch, p.nb, use_absent_limit, fast, p.counter_base}, s->stream);
  if (p.n_del > 0 && !o.shadow_lists && ++s->stamp == 0) {  // stamps restart
    check(cudaMemsetAsync(b.mark, 0, sizeof(uint32_t) * s->n, s->stream), "marks");
    s->stamp = 1;
  }
  p.launches += launch_prepare(s->H.view(), s->G.view(), b, p.nb, p.n_del, s->n, s->stamp, o,
                               s->stream);
  maybe_sync(s, "validate + queries + walk shadow");
}

// Walks over query ranges. Full range (single GPU): counts stay on the
// device (no host sync). Shard range: counts written from the host.
void phase_walk(dyg_session* s, Pending& p, bool full, uint32_t lo_r, uint32_t n_r, uint32_t lo_m,
                uint32_t n_m, bool fork_g = false) {
  const WalkOpts o = walk_opts(s);
  BatchDev& b = s->b;
  b.ctl = p.dctl;
  WalkParams P = make_walk_params(o.K, o.T, o.s, o.seed);
  P.count = static_cast<uint32_t>(o.count);
  const uint32_t* cnt_r = &b.ctl->nq_reach;
  const uint32_t* cnt_m = &b.ctl->nq_min;
  uint32_t max_r = p.n_ins, max_m = p.n_del;
  const ReachQuery* rq = b.rq;
  const MinQuery* mq = b.mq;
  if (!full) {  // a shard range: its queries at [0, n) of rq_sh / mq_sh (launch_shard_range)
    cnt_r = s->d_counts + 5;
    cnt_m = s->d_counts + 7;
    max_r = n_r;  // upper bounds of the range sizes
    max_m = n_m;
    rq = b.rq_sh;
    mq = b.mq_sh;
    lo_r = lo_m = 0;
  }
  // Insertion fast path: G's appends do not depend on the walk (it reads H
  // alone); fork them onto the aux stream so they fill the walk's tail.
  const bool fast = p.n_del == 0 && p.n_ins > 0 && o.fastpath && o.single_pass;
  // A shard walk forks them only when the same Pending reaches the commit
  // (fork_g: the peer-exchange range enqueues walk and commit together).
  const bool fork = fast && (full || fork_g);
  // The fork point is recorded before the walk, but the aux kernels are
  // enqueued after it: the walk's blocks claim the SMs first (its start is
  // on the batch's critical path; the appends only need to finish by the
  // commit).
  auto fork_appends = [&] {
    check(cudaStreamWaitEvent(s->aux_stream, s->ev_fork, 0), "fork");
    p.launches += launch_fastpath_g(s->G.view(), b, p.nb, s->aux_stream);
    check(cudaEventRecord(s->ev_join, s->aux_stream), "join");
    p.g_appended = true;
  };
  if (fork) {
    check(cudaEventRecord(s->ev_fork, s->stream), "fork");
  }
  if (p.n_ins > 0 && o.filtering && max_r > 0) {
    // No best_bits: the commit reads `reached` and `steps` alone.
    ReachOut ro{b.rout.reached + lo_r, b.rout.steps + lo_r, nullptr, nullptr, 0};
    if (full && o.split_wpq > 0.0 && p.n_del == 0 && o.single_pass) {
      ro.nq_long = &b.ctl->nq_long;
      ro.cap = b.q_cap;
    }
    p.launches += launch_reach(s->H.view(), rq + lo_r, cnt_r, max_r, P, ro, &b.ctl->reach,
                               s->d_work, s->stream, /*standalone=*/!full);
    maybe_sync(s, "reach walks");
  }
  if (fork) fork_appends();
  if (p.g_appended) check(cudaStreamWaitEvent(s->stream, s->ev_join, 0), "join");
  if (p.n_del > 0 && !o.freeze && max_m > 0) {
    WalkParams Pd = P;
    Pd.K = std::numeric_limits<double>::infinity();  // sparsifier.cpp:458-459
    const uint64_t T1 = static_cast<uint64_t>(o.T) + 1;
    // No resistance: the commit uses the recovered path alone (:503-514).
    MinOut mo{b.mout.has_path + lo_m, b.mout.path_len + lo_m, b.mout.steps + lo_m,
              nullptr, b.mout.paths + lo_m * T1, &b.ctl->t_mp_end};
    // k_scatter reset the work counter; a mixed batch's reach walk used it,
    // and a shard range walk may follow another range's walk.
    const bool reset = !full || (p.n_ins > 0 && o.filtering);
    p.launches += launch_minpath(s->G.view(), mq + lo_m, cnt_m, max_m, Pd, b.mscratch, mo,
                                 &b.ctl->minpath, s->d_work, s->stream, reset);
    maybe_sync(s, "minpath walks");
  }
}

// Commit (:466-533) enqueue: the commit launch (shadow undo, commit engine,
// epilogue) and the async copy of the control block back.
void commit_enqueue(dyg_session* s, Pending& p, bool download = true) {
  const WalkOpts o = walk_opts(s);
  BatchDev& b = s->b;
  b.ctl = p.dctl;
  const bool fp = p.n_del == 0 && p.n_ins > 0 && o.fastpath && o.single_pass;
  if (fp && !p.g_appended) p.launches += launch_fastpath_g(s->G.view(), b, p.nb, s->stream);
  // The H appends open the commit launch (fp_h).
  p.launches += launch_commit(s->G.view(), s->H.view(), b, p.nb, p.n_del, o, s->stream, fp);
  maybe_sync(s, "commit");
  if (download)
    check(cudaMemcpyAsync(p.hctl, b.ctl, sizeof(BatchCtl), cudaMemcpyDeviceToHost, s->stream),
          "ctl download");
  if (p.nb == 1)
    check(cudaMemcpyAsync(p.hdec, b.dec, sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream),
          "decision download");
  if (p.dec_dev) {
    p.launches += launch_export_decisions(b.dec, p.dev, p.nb, p.dec_dev, s->stream);
    check(cudaMemcpyAsync(p.dec_pin, p.dec_dev, p.nb, cudaMemcpyDeviceToHost, s->stream),
          "decisions download");
  }
}

// After the stream has synchronised: error mapping (:525-529), counters and
// the BatchReport (:535-537).
void commit_finalize(dyg_session* s, Pending& p, dyg_batch_report* out) {
  const BatchCtl& c = *p.hctl;
  s->stats.d2h_bytes += sizeof c;
  s->stats.kernel_launches += p.launches;
  s->stats.batches += 1;
  if (c.val_err != ~0ull && (c.val_err & 0xFF) == kErrPeer)
    fail(DYG_ERR_DEVICE, "multi-GPU peer exchange timed out: a rank did not publish its walk "
                         "records (batch " + std::to_string(p.batch) + ")");
  if (c.val_err != ~0ull) fail_validation(s, p, c.val_err);
  // Commit-side state is now final for events < limit.
  s->g_edges = c.g_edges;
  s->h_edges = c.h_edges;
  s->g_top = c.g_pool_top;
  s->h_top = c.h_pool_top;
  uint64_t fail_k = ~0ull;
  uint32_t fail_code = 0;
  if (c.commit_err != ~0ull) {
    fail_k = c.commit_err >> 8;
    fail_code = static_cast<uint32_t>(c.commit_err & 0xFF);
  }
  if (c.use_absent_limit && c.first_absent != 0xFFFFFFFFu && c.first_absent < fail_k) {
    fail_k = c.first_absent;
    fail_code = kErrAbsent;
  }
  s->stats.reach_steps += c.reach.steps;
  s->stats.reach_row_bytes += c.reach.row_bytes;
  s->stats.reach_tail_row_bytes += c.reach.tail_bytes;
  s->stats.minpath_tail_row_bytes += c.minpath.tail_bytes;
  auto tail_ms = [](const WalkCounters& w) {
    return (w.t_end > w.t_drain && w.t_drain != ~0ull) ? (w.t_end - w.t_drain) * 1e-6 : 0.0;
  };
  s->stats.reach_tail_ms += tail_ms(c.reach);
  s->stats.minpath_tail_ms += tail_ms(c.minpath);
  s->stats.minpath_steps += c.minpath.steps;
  s->stats.minpath_row_bytes += c.minpath.row_bytes;
  s->stats.reach_queries += c.nq_reach;
  s->stats.minpath_queries += c.nq_min;
  s->stats.commit_rounds += c.rounds;
  if (c.flow_done && c.fl_t[5] > c.fl_t[0]) {
    s->stats.flow_ms_promote += (c.fl_t[1] - c.fl_t[0]) * 1e-6;
    s->stats.flow_ms_emit += (c.fl_t[2] - c.fl_t[1]) * 1e-6;
    s->stats.flow_ms_rank += (c.fl_t[3] - c.fl_t[2]) * 1e-6;
    s->stats.flow_ms_apply += (c.fl_t[4] - c.fl_t[3]) * 1e-6;
    s->stats.flow_ms_reset += (c.fl_t[5] - c.fl_t[4]) * 1e-6;
  }
  if (p.n_del > 0) {
    s->stats.commit_ms_deletion += span_ms(c.t_commit0, c.t_batch1);
    s->stats.commit_rounds_deletion += c.rounds;
  }
  // Phase times from %globaltimer stamps the kernels write into the control
  // block (CUDA events between the phases cost ~4 us each in the stream:
  // 8 per batch were 0.67 ms of a 10 ms C5 step).
  s->stats.reach_ms += span_ms(c.reach.t_start, c.reach.t_end);
  s->stats.minpath_ms += span_ms(c.minpath.t_start, c.t_mp_end);
  s->stats.minpath_walk_ms += span_ms(c.minpath.t_start, c.minpath.t_end);
  s->stats.commit_ms += span_ms(c.t_commit0, c.t_batch1);
  s->stats.total_ms += span_ms(c.t_batch0, c.t_batch1);
  {
    const unsigned long long w0 = std::min(c.reach.t_start, c.minpath.t_start);
    const unsigned long long w1 = std::max(c.reach.t_end == ~0ull ? 0ull : c.reach.t_end,
                                           c.t_mp_end == ~0ull ? 0ull : c.t_mp_end);
    if (w0 != ~0ull && w0 > c.t_batch0) s->stats.prep_ms += span_ms(c.t_batch0, w0);
    if (w1 != 0 && c.t_commit0 > w1) s->stats.walk_commit_gap_ms += span_ms(w1, c.t_commit0);
    // Consecutive batches of one replay (a gap over 1 ms is a host pause).
    double gap_prev_us = -1.0;
    if (s->last_t1 && c.t_batch0 > s->last_t1 && c.t_batch0 - s->last_t1 < 1000000ull) {
      s->stats.batch_gap_ms += span_ms(s->last_t1, c.t_batch0);
      gap_prev_us = (c.t_batch0 - s->last_t1) * 1e-3;
    }
    s->last_t1 = c.t_batch1;
    static const bool timeline = std::getenv("DYG_TIMELINE") != nullptr;
    if (timeline) {  // per-batch device timeline (us from batch start)
      auto rel = [&](unsigned long long t) {
        return (t == ~0ull || t == 0 || t < c.t_batch0) ? -1.0 : (t - c.t_batch0) * 1e-3;
      };
      std::fprintf(stderr,
                   "dyg timeline batch %u nb=%u del=%u: reach %.1f-%.1f (drain %.1f) min %.1f-%.1f "
                   "mp_end %.1f commit0 %.1f fl0 %.1f end %.1f gap_before %.1f prep %.1f-%.1f\n",
                   p.batch, p.nb, p.n_del, rel(c.reach.t_start), rel(c.reach.t_end),
                   rel(c.reach.t_drain), rel(c.minpath.t_start), rel(c.minpath.t_end),
                   rel(c.t_mp_end), rel(c.t_commit0), rel(c.fl_t[0]), rel(c.t_batch1),
                   gap_prev_us, rel(c.t_prep0), rel(c.t_prep1));
    }
  }
  if (fail_k != ~0ull) {
    s->counter = p.counter_base + fail_k + 1;  // ++update_counter_ precedes the throw (:469)
    const uint64_t pos = p.pos ? p.pos[fail_k] : p.pos_base + fail_k;
    fail(fail_code == kErrPool ? DYG_ERR_DEVICE : DYG_ERR_DATA,
         event_error_message(fail_code, pos, event_at(p, fail_k)));
  }
  s->counter = p.counter_base + p.nb;
  s->last_dec = p.nb == 1 ? *p.hdec : 0;
  dyg_batch_report rep{};
  rep.batch_index = p.batch;
  rep.insertions_seen = c.report[kInsSeen];
  rep.insertions_kept = c.report[kInsKept];
  rep.insertions_pruned = c.report[kInsPruned];
  rep.deletions_seen = c.report[kDelSeen];
  rep.deletions_in_sparsifier = c.report[kDelInH];
  rep.paths_recovered = c.report[kPaths];
  rep.edges_recovered = c.report[kEdgesRec];
  rep.fallback_activations = c.report[kFallbacks];
  rep.walker_steps = c.report[kWalkerSteps];
  rep.max_event_steps = c.report[kMaxEventSteps];
  rep.density_graph = density_of(s->g_edges, s->n);
  rep.density_sparsifier = density_of(s->h_edges, s->n);
  // T_update of the batch on the device: its first kernel's start stamp to
  // the commit's end stamp (in a range replay the host finalises all batches
  // after one synchronisation, so host time would not be per batch).
  rep.wall_ms = span_ms(c.t_batch0, c.t_batch1);
  *out = rep;
}

void empty_report(dyg_session* s, uint32_t batch_index, dyg_batch_report* out) {
  dyg_batch_report rep{};
  rep.batch_index = batch_index;
  rep.density_graph = density_of(s->g_edges, s->n);
  rep.density_sparsifier = density_of(s->h_edges, s->n);
  *out = rep;
}

void reset_abort(dyg_session* s) {
  check(cudaMemsetAsync(s->d_abort, 0, sizeof(unsigned int), s->stream), "abort flag");
}


// ------------------------------------------------------------ CUDA graphs
// A batch is ~15 short kernels; launched one by one, the host launch cost
// and the inter-kernel gaps are a visible share of a batch (tens of us on
// ~0.4 ms). The enqueue sequence of a batch -- or of a whole uploaded range
// -- is captured once into a CUDA graph and replayed with one launch. Every
// kernel argument except the update counter is a pure function of the batch
// shape and of the session's buffer pointers, so the graph is keyed by a
// fingerprint of exactly those; the counter lives in the k_ctl_init nodes
// and is re-pointed per launch when it differs.
bool graphs_usable(const dyg_session* s) { return s->graphs_on && !s->debug_sync; }

uint64_t session_fingerprint(dyg_session* s, uint64_t tag) {
  uint64_t h = fnv(1469598103934665603ull, &tag, sizeof tag);
  const auto add_graph = [&](auto v) {
    const void* ptrs[] = {v.slab, v.cap, v.pool_id, v.pool_w, v.pool_top, v.edges};
    h = fnv(h, ptrs, sizeof ptrs);
    h = fnv(h, &v.pool_cap, sizeof v.pool_cap);
    h = fnv(h, &v.n, sizeof v.n);
  };
  add_graph(s->G.view());
  add_graph(s->H.view());
  BatchDev b = s->b;  // all buffer pointers and capacities; per-batch fields blanked
  b.ctl = nullptr;
  b.events = nullptr;
  b.side_top = nullptr;
  b.scratch_edges = nullptr;
  h = fnv(h, &b, sizeof b);
  const WalkOpts o = walk_opts(s);
  h = fnv(h, &o, sizeof o);
  const void* fixed[] = {s->d_work, s->d_abort, s->d_counts, s->h_ctl};
  h = fnv(h, fixed, sizeof fixed);
  if (!o.shadow_lists) h = fnv(h, &s->stamp, sizeof s->stamp);
  return h;
}

void destroy_graph(CapturedGraph& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.graph) cudaGraphDestroy(g.graph);
  g.exec = nullptr;
  g.graph = nullptr;
}

CapturedGraph* find_graph(dyg_session* s, uint64_t key) {
  for (CapturedGraph& g : s->graphs)
    if (g.key == key) return &g;
  return nullptr;
}

// Capture `enqueue` (returns the kernels it launched) into a graph. Returns
// nullptr -- and turns graphs off for the session -- when capture is not
// possible; the caller then enqueues eagerly.
template <class F>
CapturedGraph* capture_graph(dyg_session* s, uint64_t key, uint64_t counter, F&& enqueue) {
  cudaGetLastError();
  if (cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    // e.g. the legacy default stream, which cannot be captured
    if (std::getenv("DYG_GRAPH_DEBUG"))
      std::fprintf(stderr, "dyg: stream capture unavailable (%s); launching eagerly\n",
                   cudaGetErrorString(cudaGetLastError()));
    cudaGetLastError();
    s->graphs_on = false;
    return nullptr;
  }
  s->capturing = true;
  int launches = 0;
  try {
    launches = enqueue();
  } catch (...) {
    s->capturing = false;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(s->stream, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    throw;
  }
  s->capturing = false;
  CapturedGraph cg;
  cudaError_t e1 = cudaStreamEndCapture(s->stream, &cg.graph);
  cudaError_t e2 = (e1 == cudaSuccess && cg.graph) ? cudaGraphInstantiate(&cg.exec, cg.graph, 0)
                                                   : cudaErrorUnknown;
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    if (std::getenv("DYG_GRAPH_DEBUG"))
      std::fprintf(stderr, "dyg: graph capture failed (%s / %s); launching eagerly\n",
                   cudaGetErrorString(e1), cudaGetErrorString(e2));
    cudaGetLastError();
    destroy_graph(cg);
    s->graphs_on = false;
    return nullptr;
  }
  size_t n = 0;
  check(cudaGraphGetNodes(cg.graph, nullptr, &n), "graph nodes");
  std::vector<cudaGraphNode_t> nodes(n);
  check(cudaGraphGetNodes(cg.graph, nodes.data(), &n), "graph nodes");
  for (cudaGraphNode_t node : nodes) {
    CtlInitArgs a{};
    if (ctl_init_node_args(node, &a)) {
      cg.ctl_nodes.push_back(node);
      cg.ctl_args.push_back(a);
    }
  }
  cg.key = key;
  cg.base = counter;
  cg.cap_base = counter;
  cg.launches = launches;
  constexpr size_t kMaxGraphs = 256;  // a whole stream's per-batch graphs (x3 segments when sharded)
  if (s->graphs.size() >= kMaxGraphs) {  // evict the least recently used
    size_t lru = 0;
    for (size_t i = 1; i < s->graphs.size(); ++i)
      if (s->graphs[i].last_use < s->graphs[lru].last_use) lru = i;
    destroy_graph(s->graphs[lru]);
    s->graphs.erase(s->graphs.begin() + lru);
  }
  s->graphs.push_back(std::move(cg));
  return &s->graphs.back();
}

void launch_graph(dyg_session* s, CapturedGraph& g, uint64_t counter) {
  if (counter != g.base) {
    for (size_t i = 0; i < g.ctl_nodes.size(); ++i) {
      CtlInitArgs a = g.ctl_args[i];
      a.counter_base = a.counter_base - g.cap_base + counter;
      check(ctl_init_node_update(g.exec, g.ctl_nodes[i], a), "graph counter update");
    }
    g.base = counter;
  }
  g.last_use = ++s->graph_clock;
  check(cudaGraphLaunch(g.exec, s->stream), "graph launch");
  s->stats.graph_launches += 1;
}

// Enqueue a device sequence through a captured graph keyed by `key` (its
// first use captures it), or eagerly when graphs are off. `enqueue` returns
// the kernels it launched; the return value is that count.
template <class F>
int enqueue_captured(dyg_session* s, uint64_t key, uint64_t counter, F&& enqueue) {
  if (graphs_usable(s)) {
    CapturedGraph* g = find_graph(s, key);
    if (g == nullptr) g = capture_graph(s, key, counter, enqueue);
    if (g != nullptr) {
      launch_graph(s, *g, counter);
      return g->launches;
    }
  }
  return enqueue();
}

void run_deferred(dyg_session* s, const DevEvent* dev_events, const DevEvent* host_events,
                  const uint64_t* positions, uint32_t nb, uint32_t n_ins, uint32_t n_del,
                  uint32_t batch_index, dyg_batch_report* out, bool immediate_msgs,
                  uint8_t* dec_dst = nullptr, const uint64_t* dec_idx = nullptr,
                  uint64_t pos_base = 0) {
  if (nb == 0) {
    empty_report(s, batch_index, out);
    return;
  }
  Pending p;
  bind_pending(s, p);
  if (dec_dst) {
    ensure_decisions(s, nb);
    p.dec_dev = s->d_dec;
    p.dec_pin = s->h_dec;
    p.dec_dst = dec_dst;
    p.dec_idx = dec_idx;
  }
  p.wall0 = std::chrono::steady_clock::now();
  p.dev = dev_events;
  p.host = host_events;
  p.pos = positions;
  p.pos_base = pos_base;
  p.nb = nb;
  p.n_ins = n_ins;
  p.n_del = n_del;
  p.batch = batch_index;
  p.imm_msgs = immediate_msgs;
  reset_abort(s);
  if (graphs_usable(s)) {
    // Size every buffer first: nothing may allocate inside a capture.
    ensure_batch(s, nb, n_del);
    ensure_pools(s, n_ins, n_del);
    if (n_del > 0) ensure_side_pool(s);
    uint64_t key = session_fingerprint(s, 1);
    const uint64_t shape[] = {reinterpret_cast<uint64_t>(p.dev), reinterpret_cast<uint64_t>(p.dctl),
                              reinterpret_cast<uint64_t>(p.hctl), reinterpret_cast<uint64_t>(p.hdec),
                              reinterpret_cast<uint64_t>(p.dec_dev), nb, n_ins, n_del};
    key = fnv(key, shape, sizeof shape);
    CapturedGraph* g = find_graph(s, key);
    if (g == nullptr) {
      g = capture_graph(s, key, p.counter_base, [&] {
        Pending q = p;
        phase_prepare(s, q);
        phase_walk(s, q, true, 0, 0, 0, 0);
        commit_enqueue(s, q);
        return q.launches;
      });
    }
    if (g != nullptr) {
      launch_graph(s, *g, p.counter_base);
      p.launches = g->launches;
      check(cudaStreamSynchronize(s->stream), "batch");
      deliver_decisions(p);
      commit_finalize(s, p, out);
      return;
    }
  }
  phase_prepare(s, p);
  phase_walk(s, p, true, 0, 0, 0, 0);
  commit_enqueue(s, p);
  check(cudaStreamSynchronize(s->stream), "batch");
  deliver_decisions(p);
  commit_finalize(s, p, out);
}

// True when p is page-locked host memory the DMA engines can read directly.
bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host events -> device (straight from page-locked buffers, else through the
// session's pinned staging copy), then the deferred pipeline.
void upload_events(dyg_session* s, const dyg_event* ev, size_t nb) {
  static_assert(sizeof(DevEvent) == sizeof(dyg_event), "event layout");
  if (nb == 0) return;
  const void* src = ev;
  if (!host_pinned(ev)) {
    std::memcpy(s->h_events_pinned, ev, sizeof(DevEvent) * nb);
    src = s->h_events_pinned;
  }
  check(cudaMemcpyAsync(s->d_events, src, sizeof(DevEvent) * nb, cudaMemcpyHostToDevice,
                        s->stream), "events upload");
  s->stats.h2d_bytes += sizeof(DevEvent) * nb;
}

// Insertion / deletion counts of the uploaded batch, counted on the device:
// one short round trip instead of a host pass over every event (at C5 that
// host pass read 2.5 MB per batch and cost more than the upload itself).
void count_kinds(dyg_session* s, uint32_t nb, uint32_t& n_ins, uint32_t& n_del) {
  n_ins = n_del = 0;
  if (nb == 0) return;
  s->stats.kernel_launches += launch_count_kinds(s->d_events, nb, s->d_counts + 2, s->stream);
  check(cudaMemcpyAsync(s->h_counts + 4, s->d_counts + 2, 2 * sizeof(uint32_t),
                        cudaMemcpyDeviceToHost, s->stream), "kind counts");
  check(cudaStreamSynchronize(s->stream), "kind counts");
  n_ins = s->h_counts[4];
  n_del = s->h_counts[5];
}

void run_host_batch(dyg_session* s, const dyg_event* ev, const uint64_t* positions, size_t nb,
                    uint32_t batch_index, dyg_batch_report* out, bool immediate_msgs,
                    uint8_t* dec_dst = nullptr, const uint64_t* dec_idx = nullptr) {
  ensure_batch(s, static_cast<uint32_t>(nb), 0);
  upload_events(s, ev, nb);
  uint32_t n_ins = 0, n_del = 0;
  count_kinds(s, static_cast<uint32_t>(nb), n_ins, n_del);
  ensure_batch(s, static_cast<uint32_t>(nb), n_del);
  run_deferred(s, s->d_events, reinterpret_cast<const DevEvent*>(ev), positions,
               static_cast<uint32_t>(nb), n_ins, n_del, batch_index, out, immediate_msgs, dec_dst,
               dec_idx);
}

// Kind counts of an asynchronously uploaded stream (dyg_stream_upload_batches):
// batch b's counts are read once its upload and count have landed; with
// b == ~0u every batch is settled and the structure fingerprint computed.
void settle_upload(dyg_session* s, uint32_t b) {
  if (!s->up_pending) return;
  const uint32_t nbat = static_cast<uint32_t>(s->batch_cnt.size());
  const uint32_t lo = b == ~0u ? 0 : b, hi = b == ~0u ? nbat : std::min(b + 1, nbat);
  for (uint32_t k = lo; k < hi; ++k) {
    if (s->up_settled[k]) continue;
    check(cudaEventSynchronize(s->up_ready[k]), "stream upload");
    s->batch_ins[k] = s->h_up_kinds[2ull * k];
    s->batch_del[k] = s->h_up_kinds[2ull * k + 1];
    s->up_settled[k] = 1;
  }
  if (b == ~0u) {
    s->stream_gen = fnv(fnv(fnv(0xcbf29ce484222325ull, s->batch_off.data(),
                                sizeof(uint64_t) * s->batch_off.size()),
                            s->batch_ins.data(), sizeof(uint64_t) * nbat),
                        s->batch_del.data(), sizeof(uint64_t) * nbat);
    s->up_pending = false;
  }
}

// Host copy / stream positions of uploaded event `off` (nullptr when the
// stream was DMA'd from a grouped page-locked buffer: positions are then the
// identity and events are read back from the device on an error).
const DevEvent* uploaded_host(const dyg_session* s, uint64_t off) {
  return s->stream_events.empty() ? nullptr
                                  : reinterpret_cast<const DevEvent*>(s->stream_events.data() + off);
}
const uint64_t* uploaded_pos(const dyg_session* s, uint64_t off) {
  return s->stream_positions.empty() ? nullptr : s->stream_positions.data() + off;
}

// Device-resident stream, batches [first, first + count) enqueued back to
// back; one host sync at the end (the device-side replay(stream),
// sparsifier.cpp:550-559). Buffers and pool headroom are sized for the whole
// range up front; a failing batch raises the device abort flag so the later
// batches of the range do nothing, and the error is reported for it.
void run_uploaded_range(dyg_session* s, uint32_t first, uint32_t count, dyg_batch_report* out,
                        uint8_t* dec_dst = nullptr) {
  if (count == 0) return;
  uint64_t sum_ins = 0, sum_del = 0;
  uint32_t max_nb = 0, max_nd = 0;
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t b = first + i;
    if (b >= s->batch_cnt.size()) continue;
    sum_ins += s->batch_ins[b];
    sum_del += s->batch_del[b];
    max_nb = std::max<uint32_t>(max_nb, static_cast<uint32_t>(s->batch_cnt[b]));
    max_nd = std::max<uint32_t>(max_nd, static_cast<uint32_t>(s->batch_del[b]));
  }
  ensure_batch(s, std::max<uint32_t>(max_nb, 1), max_nd);
  ensure_pools(s, sum_ins, sum_del);
  if (sum_del > 0) ensure_side_pool(s);
  if (dec_dst) ensure_decisions(s, sum_ins + sum_del);
  if (s->ctl_cap < count) {
    dev_free(s->d_ctls);
    if (s->h_ctls) cudaFreeHost(s->h_ctls);
    s->h_ctls = nullptr;
    dev_alloc(&s->d_ctls, count, "batch control blocks");
    // Empty batches never initialise their block; the whole-range download
    // then copies defined bytes (initcheck).
    check(cudaMemset(s->d_ctls, 0, sizeof(BatchCtl) * count), "batch control blocks");
    check(cudaMallocHost(reinterpret_cast<void**>(&s->h_ctls), sizeof(BatchCtl) * count),
          "pinned control blocks");
    s->ctl_cap = count;
  }
  std::vector<Pending> ps(count);
  const uint64_t counter0 = s->counter;
  const auto wall0 = std::chrono::steady_clock::now();
  reset_abort(s);
  // Host-side description of every batch (also what commit_finalize reads).
  {
    uint64_t counter = counter0, dec_off = 0;
    for (uint32_t i = 0; i < count; ++i) {
      const uint32_t b = first + i;
      Pending& p = ps[i];
      p.batch = b;
      p.wall0 = wall0;
      p.dctl = s->d_ctls + i;
      p.hctl = s->h_ctls + i;
      p.hdec = &s->h_counts[2];
      p.counter_base = counter;
      if (b >= s->batch_cnt.size() || s->batch_cnt[b] == 0) continue;
      const uint64_t off = s->batch_off[b];
      p.dev = s->d_stream + off;
      p.host = uploaded_host(s, off);
      p.pos = uploaded_pos(s, off);
      p.pos_base = off;
      p.nb = static_cast<uint32_t>(s->batch_cnt[b]);
      p.n_ins = static_cast<uint32_t>(s->batch_ins[b]);
      p.n_del = static_cast<uint32_t>(s->batch_del[b]);
      if (dec_dst) {  // indexed by stream position
        p.dec_dev = s->d_dec + dec_off;
        p.dec_pin = s->h_dec + dec_off;
        p.dec_dst = p.pos ? dec_dst : dec_dst + off;
        p.dec_idx = p.pos;
        dec_off += p.nb;
      }
      counter += p.nb;
    }
  }
  auto enqueue = [&] {
    int launches = 0;
    for (uint32_t i = 0; i < count; ++i) {
      Pending p = ps[i];
      if (p.nb == 0) continue;
      phase_prepare(s, p);
      phase_walk(s, p, true, 0, 0, 0, 0);
      commit_enqueue(s, p, false);
      ps[i].launches = p.launches;
      launches += p.launches;
    }
    // All control blocks in one transfer (one copy-engine round trip per range).
    check(cudaMemcpyAsync(s->h_ctls, s->d_ctls, sizeof(BatchCtl) * count, cudaMemcpyDeviceToHost,
                          s->stream), "ctl download");
    return launches;
  };
  CapturedGraph* g = nullptr;
  if (graphs_usable(s)) {
    uint64_t key = session_fingerprint(s, 2);
    const uint64_t shape[] = {first, count, s->stream_gen, reinterpret_cast<uint64_t>(s->d_stream),
                              reinterpret_cast<uint64_t>(s->d_ctls),
                              reinterpret_cast<uint64_t>(s->h_ctls),
                              dec_dst ? reinterpret_cast<uint64_t>(s->d_dec) : 0ull};
    key = fnv(key, shape, sizeof shape);
    g = find_graph(s, key);
    if (g == nullptr) g = capture_graph(s, key, counter0, enqueue);
    else
      for (uint32_t i = 0; i < count; ++i) ps[i].launches = g->per_batch[i];
    if (g != nullptr) {
      if (g->per_batch.empty())
        for (uint32_t i = 0; i < count; ++i) g->per_batch.push_back(ps[i].launches);
      launch_graph(s, *g, counter0);
    }
  }
  if (g == nullptr) enqueue();
  check(cudaStreamSynchronize(s->stream), "batch range");
  for (uint32_t i = 0; i < count; ++i) {
    if (ps[i].nb == 0) {
      empty_report(s, ps[i].batch, &out[i]);
      continue;
    }
    deliver_decisions(ps[i]);
    commit_finalize(s, ps[i], &out[i]);  // throws at the first failing batch
  }
}

// SparsifierState::replay(stream) (sparsifier.cpp:550-559) from a host
// stream whose events are grouped by batch (batch b = [off[b], off[b+1])).
// Uploads run on a copy stream, batch by batch, each followed by a device
// count of its insertions / deletions; batch b's kernels wait only for batch
// b's upload, so the PCIe transfer of later batches overlaps the walks and
// commits of earlier ones, and the host enqueues batch b + 1 while batch b
// runs. One synchronisation at the end; reports as in the uploaded-range
// replay (a failing batch stops the ones after it).
void run_stream(dyg_session* s, const dyg_event* events, size_t n, const uint64_t* off,
                uint32_t nbatches, dyg_batch_report* out, uint8_t* dec_dst = nullptr) {
  if (nbatches == 0) return;
  if (dec_dst) ensure_decisions(s, n);
  uint64_t max_nb = 1;
  for (uint32_t b = 0; b < nbatches; ++b) max_nb = std::max<uint64_t>(max_nb, off[b + 1] - off[b]);
  if (max_nb > 0xFFFFFFF0ull) fail(DYG_ERR_USAGE, "batch too large");
  ensure_batch(s, static_cast<uint32_t>(max_nb), 0);
  if (s->copy_stream == nullptr)
    check(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking), "copy stream");
  if (s->replay_cap < n) {
    dev_free(s->d_replay);
    dev_alloc(&s->d_replay, std::max<uint64_t>(n, 1), "replay events");
    s->replay_cap = n;
  }
  if (s->kinds_cap < nbatches) {
    dev_free(s->d_kinds);
    if (s->h_kinds) cudaFreeHost(s->h_kinds);
    s->h_kinds = nullptr;
    dev_alloc(&s->d_kinds, 2ull * nbatches, "kind counts");
    check(cudaMallocHost(reinterpret_cast<void**>(&s->h_kinds), 2 * sizeof(uint32_t) * nbatches),
          "pinned kind counts");
    s->kinds_cap = nbatches;
  }
  if (s->ctl_cap < nbatches) {
    dev_free(s->d_ctls);
    if (s->h_ctls) cudaFreeHost(s->h_ctls);
    s->h_ctls = nullptr;
    dev_alloc(&s->d_ctls, nbatches, "batch control blocks");
    check(cudaMemset(s->d_ctls, 0, sizeof(BatchCtl) * nbatches), "batch control blocks");
    check(cudaMallocHost(reinterpret_cast<void**>(&s->h_ctls), sizeof(BatchCtl) * nbatches),
          "pinned control blocks");
    s->ctl_cap = nbatches;
  }
  while (s->ready.size() < nbatches) {
    cudaEvent_t e;
    check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    s->ready.push_back(e);
  }
  // 1. Uploads and kind counts, all batches, on the copy stream.
  const bool pinned = host_pinned(events);
  for (uint32_t b = 0; b < nbatches; ++b) {
    const uint64_t nb = off[b + 1] - off[b];
    if (nb) {
      check(cudaMemcpyAsync(s->d_replay + off[b], events + off[b], sizeof(DevEvent) * nb,
                            pinned ? cudaMemcpyHostToDevice : cudaMemcpyDefault, s->copy_stream),
            "events upload");
      s->stats.h2d_bytes += sizeof(DevEvent) * nb;
      s->stats.kernel_launches += launch_count_kinds(s->d_replay + off[b], static_cast<uint32_t>(nb),
                                                     s->d_kinds + 2ull * b, s->copy_stream);
      check(cudaMemcpyAsync(s->h_kinds + 2ull * b, s->d_kinds + 2ull * b, 2 * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s->copy_stream), "kind counts");
    }
    check(cudaEventRecord(s->ready[b], s->copy_stream), "upload event");
  }
  // 2. Batches in order on the session stream.
  std::vector<Pending> ps(nbatches);
  const auto wall0 = std::chrono::steady_clock::now();
  reset_abort(s);
  uint64_t counter = s->counter, sum_ins = 0, sum_del = 0;
  for (uint32_t b = 0; b < nbatches; ++b) {
    Pending& p = ps[b];
    p.batch = b;
    p.wall0 = wall0;
    p.dctl = s->d_ctls + b;
    p.hctl = s->h_ctls + b;
    p.hdec = &s->h_counts[2];
    p.counter_base = counter;
    p.nb = static_cast<uint32_t>(off[b + 1] - off[b]);
    if (p.nb == 0) continue;
    p.dev = s->d_replay + off[b];
    p.host = reinterpret_cast<const DevEvent*>(events + off[b]);
    p.pos = nullptr;
    p.pos_base = off[b];
    if (dec_dst) {  // indexed by stream position (grouped: off[b] + k)
      p.dec_dev = s->d_dec + off[b];
      p.dec_pin = s->h_dec + off[b];
      p.dec_dst = dec_dst + off[b];
    }
    check(cudaEventSynchronize(s->ready[b]), "upload");
    p.n_ins = s->h_kinds[2ull * b];
    p.n_del = s->h_kinds[2ull * b + 1];
    sum_ins += p.n_ins;
    sum_del += p.n_del;
    // Pool growth copies on the session stream behind the enqueued batches;
    // the deletion buffers and the side pool are freed and reallocated, so
    // let the enqueued batches drain first when they have to grow.
    ensure_pools(s, sum_ins, sum_del);
    if (p.n_del > s->nd_cap ||
        (p.n_del > 0 && (s->b.side_id == nullptr || s->side_cap < s->G.pool_capacity())))
      check(cudaStreamSynchronize(s->stream), "buffer growth");
    ensure_batch(s, p.nb, p.n_del);
    if (p.n_del > 0) ensure_side_pool(s);
    check(cudaStreamWaitEvent(s->stream, s->ready[b], 0), "upload wait");
    auto enqueue = [&] {
      Pending q = p;
      phase_prepare(s, q);
      phase_walk(s, q, true, 0, 0, 0, 0);
      commit_enqueue(s, q, false);
      return q.launches;
    };
    CapturedGraph* g = nullptr;
    if (graphs_usable(s)) {  // one graph per batch slot, reused by later replays
      uint64_t key = session_fingerprint(s, 3);
      const uint64_t shape[] = {reinterpret_cast<uint64_t>(p.dev), reinterpret_cast<uint64_t>(p.dctl),
                                reinterpret_cast<uint64_t>(p.hctl),
                                reinterpret_cast<uint64_t>(p.dec_dev), p.nb, p.n_ins, p.n_del};
      key = fnv(key, shape, sizeof shape);
      g = find_graph(s, key);
      if (g == nullptr) g = capture_graph(s, key, p.counter_base, enqueue);
      if (g != nullptr) {
        launch_graph(s, *g, p.counter_base);
        p.launches = g->launches;
      }
    }
    if (g == nullptr) p.launches = enqueue();
    counter += p.nb;
  }
  check(cudaMemcpyAsync(s->h_ctls, s->d_ctls, sizeof(BatchCtl) * nbatches, cudaMemcpyDeviceToHost,
                        s->stream), "ctl download");
  check(cudaStreamSynchronize(s->stream), "stream replay");
  for (uint32_t b = 0; b < nbatches; ++b) {
    if (ps[b].nb == 0) {
      empty_report(s, b, &out[b]);
      continue;
    }
    deliver_decisions(ps[b]);
    commit_finalize(s, ps[b], &out[b]);  // throws at the first failing batch
  }
}

void accumulate(dyg_batch_report& acc, const dyg_batch_report& r) {
  acc.insertions_seen += r.insertions_seen;
  acc.insertions_kept += r.insertions_kept;
  acc.insertions_pruned += r.insertions_pruned;
  acc.deletions_seen += r.deletions_seen;
  acc.deletions_in_sparsifier += r.deletions_in_sparsifier;
  acc.paths_recovered += r.paths_recovered;
  acc.edges_recovered += r.edges_recovered;
  acc.fallback_activations += r.fallback_activations;
  acc.walker_steps += r.walker_steps;
  acc.max_event_steps = std::max(acc.max_event_steps, r.max_event_steps);
}

// replay_batch_immediate (sparsifier.cpp:347-393) as 1-event deferred
// batches (identical decisions).
void run_immediate(dyg_session* s, const dyg_event* ev, const uint64_t* positions, size_t nb,
                   uint32_t batch_index, dyg_batch_report* out, uint8_t* dec_dst = nullptr,
                   const uint64_t* dec_idx = nullptr) {
  const auto wall0 = std::chrono::steady_clock::now();
  dyg_batch_report acc{};
  acc.batch_index = batch_index;
  for (size_t i = 0; i < nb; ++i) {
    dyg_batch_report r{};
    const uint64_t pos = positions ? positions[i] : i;
    run_host_batch(s, ev + i, &pos, 1, batch_index, &r, true);
    if (dec_dst)
      dec_dst[dec_idx ? dec_idx[i] : i] =
          static_cast<uint8_t>(ev[i].kind == 0 ? (s->last_dec & 0xFF) : 2 + (s->last_dec & 0xFF));
    accumulate(acc, r);
  }
  acc.density_graph = density_of(s->g_edges, s->n);
  acc.density_sparsifier = density_of(s->h_edges, s->n);
  acc.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  *out = acc;
}

void check_csr(const dyg_csr* c, const char* what) {
  if (c == nullptr || c->row_ptr == nullptr) fail(DYG_ERR_USAGE, std::string(what) + " is null");
  if (c->n == 0) fail(DYG_ERR_USAGE, "graph must have at least one vertex");  // graph.cpp:9-13
  const uint64_t nnz = c->row_ptr[c->n];
  if (nnz && (c->ids == nullptr || c->w == nullptr))
    fail(DYG_ERR_USAGE, std::string(what) + " has null row arrays");
}

// is_connected (graph.cpp) on a host CSR: BFS from vertex 0.
bool csr_connected(const dyg_csr* c) {
  if (c->n <= 1) return true;
  std::vector<uint8_t> seen(c->n, 0);
  std::vector<uint32_t> stack{0};
  seen[0] = 1;
  uint32_t count = 1;
  while (!stack.empty()) {
    const uint32_t u = stack.back();
    stack.pop_back();
    for (uint64_t i = c->row_ptr[u]; i < c->row_ptr[u + 1]; ++i) {
      const uint32_t v = c->ids[i];
      if (v < c->n && !seen[v]) {
        seen[v] = 1;
        ++count;
        stack.push_back(v);
      }
    }
  }
  return count == c->n;
}

HostCsrView csr_view(const dyg_csr* c) { return HostCsrView{c->n, c->row_ptr, c->ids, c->w}; }

dyg_condition_options condition_defaults() {
  dyg_condition_options o{};
  o.method = 0;
  o.max_iterations = 400;
  o.tolerance = 1e-6;
  o.dense_cap = 5000;
  o.seed = 0x5eed;
  return o;
}

// condition_number (spectral.cpp:278-303) with the reference's checks.
dyg_condition_estimate condition_number_impl(const dyg_csr* g, const dyg_csr* h,
                                             const dyg_condition_options& opt, int device) {
  check_csr(g, "graph");
  check_csr(h, "sparsifier");
  if (g->n != h->n) fail(DYG_ERR_USAGE, "graphs must share a vertex set");
  if (g->n < 2) fail(DYG_ERR_USAGE, "condition number needs at least two vertices");
  if (!csr_connected(g)) fail(DYG_ERR_DATA, "graph is disconnected");
  if (!csr_connected(h)) fail(DYG_ERR_DATA, "sparsifier is disconnected");
  int method = opt.method;
  if (method == 0) method = g->n <= opt.dense_cap ? 1 : 2;
  if (method == 1 && g->n > opt.dense_cap) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "dense spectral path refused: n = %u exceeds cap %u", g->n,
                  opt.dense_cap);
    fail(DYG_ERR_USAGE, buf);
  }
  if (dyg_device_count() == 0) fail(DYG_ERR_DEVICE, "no CUDA device visible");
  check(cudaSetDevice(device), "set device");
  cudaStream_t st;
  check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  ConditionResult r;
  try {
    DevLapOwner lg(csr_view(g), st), lh(csr_view(h), st);
    check(cudaStreamSynchronize(st), "laplacian upload");
    if (method == 1) {
      r = condition_dense_device(lg.L, lh.L, st);
    } else {
      ConditionParams prm;
      prm.tolerance = opt.tolerance;
      prm.max_iterations = opt.max_iterations;
      prm.seed = opt.seed;
      r = condition_lanczos_device(lg.L, lh.L, csr_view(h), prm);
    }
  } catch (...) {
    cudaStreamDestroy(st);
    throw;
  }
  cudaStreamDestroy(st);
  dyg_condition_estimate e{};
  e.kappa = r.kappa;
  e.lambda_max = r.lambda_max;
  e.lambda_min = r.lambda_min;
  e.method = r.method;
  e.iterations_used = r.iterations;
  e.converged = r.converged;
  e.inner_iterations = r.inner_iterations;
  return e;
}

// calibrate_budget (sparsifier.cpp:561-577).
double calibrate_impl(const dyg_csr* g, const dyg_csr* h, double probe_fraction, double rho,
                      uint64_t seed, int device) {
  if (!(probe_fraction > 0.0) || probe_fraction > 1.0)
    fail(DYG_ERR_USAGE, "probe fraction must lie in (0, 1]");
  if (!(rho > 0.0)) fail(DYG_ERR_USAGE, "budget ratio must be positive");
  check_csr(g, "graph");
  dyg_condition_options o = condition_defaults();
  o.seed = seed;
  o.tolerance = 1e-3;
  const double probe = std::ceil(probe_fraction * g->n);
  o.max_iterations = static_cast<uint32_t>(std::clamp(probe, 30.0, 2000.0));
  const dyg_condition_estimate e = condition_number_impl(g, h, o, device);
  return std::clamp(rho * e.kappa, 1.0, 1e6);
}

// A session's G or H as a host CSR (owning buffers).
struct OwnedCsr {
  std::vector<uint64_t> rp;
  std::vector<uint32_t> ids;
  std::vector<double> w;
  dyg_csr c{};
};

bool csr_has_edge(const dyg_csr* c, uint32_t u, uint32_t v) {
  for (uint64_t i = c->row_ptr[u]; i < c->row_ptr[u + 1]; ++i)
    if (c->ids[i] == v) return true;
  return false;
}

}  // namespace

extern "C" {

const char* dyg_last_error(void) { return g_last_error.c_str(); }

void* dyg_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0 || cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dyg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

const char* dyg_version(void) {
  return "dyg-b200 0.1 (sm_100a; slabs H64B/G128B; fmad=false)";
}

int dyg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int dyg_session_create(const dyg_csr* g, const dyg_csr* h, const dyg_options* options,
                       int device, dyg_session** out) {
  return guarded([&] {
    if (out == nullptr || options == nullptr) fail(DYG_ERR_USAGE, "null argument");
    *out = nullptr;
    check_csr(g, "graph");
    check_csr(h, "sparsifier");
    // sparsifier.cpp:183-203
    if (g->n != h->n) fail(DYG_ERR_USAGE, "graph and sparsifier must share a vertex set");
    const dyg_walk_config& w = options->walk;
    if (w.distortion_threshold < 0.0 || w.step_cap == 0 || w.walker_count == 0)
      fail(DYG_ERR_USAGE, "invalid walk configuration");
    for (uint32_t u = 0; u < h->n; ++u) {
      for (uint64_t i = h->row_ptr[u]; i < h->row_ptr[u + 1]; ++i) {
        const uint32_t v = h->ids[i];
        if (u < v && !csr_has_edge(g, u, v)) {
          char buf[160];
          std::snprintf(buf, sizeof buf, "sparsifier edge (%u, %u) missing from the graph", u, v);
          fail(DYG_ERR_DATA, buf);
        }
      }
    }
    if (dyg_device_count() == 0) fail(DYG_ERR_DEVICE, "no CUDA device visible");
    auto* s = new dyg_session();
    try {
      s->device = device;
      check(cudaSetDevice(device), "set device");
      check(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "stream");
      check(cudaStreamCreateWithFlags(&s->aux_stream, cudaStreamNonBlocking), "aux stream");
      check(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming), "event");
      check(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming), "event");
      s->opt = *options;
      s->n = g->n;
      s->debug_sync = std::getenv("DYG_DEBUG_SYNC") != nullptr;
      s->no_fastpath = std::getenv("DYG_NO_FASTPATH") != nullptr;
      const auto env_is = [](const char* k, int v) {
        const char* e = std::getenv(k);
        return e != nullptr && std::atoi(e) == v;
      };
      s->single_pass = !env_is("DYG_SINGLE_PASS", 0);
      s->shadow_lists = !env_is("DYG_SHADOW_ROUNDS", 1);
      s->flow = !env_is("DYG_COMMIT_ROUNDS", 1);
      s->reach_split = !env_is("DYG_REACH_SPLIT", 0);
      s->keep_shadow = !env_is("DYG_KEEP_SHADOW", 0);
      s->flow_balance = !env_is("DYG_FLOW_BALANCE", 0);
      if (const char* e = std::getenv("DYG_FLOW_CAP")) s->flow_cap = std::strtoull(e, nullptr, 10);
      {
        const char* e = std::getenv("DYG_GRAPHS");
        s->graphs_on = !(e && std::atoi(e) == 0);
      }
      s->G.upload(g->n, g->row_ptr, g->ids, g->w, s->stream);
      {  // mean 1/w over G (the walk-order split's step-cost estimate)
        const uint64_t nnz = g->row_ptr[g->n];
        double acc = 0.0;
        for (uint64_t i = 0; i < nnz; ++i) acc += 1.0 / g->w[i];
        s->mean_inv_w = nnz ? acc / static_cast<double>(nnz) : 1.0;
      }
      s->H.upload(h->n, h->row_ptr, h->ids, h->w, s->stream);
      s->g_edges = g->row_ptr[g->n] / 2;
      s->h_edges = h->row_ptr[h->n] / 2;
      s->g_top = 0;
      s->h_top = 0;
      // pool_top after build: read once (setup).
      unsigned long long tops[2];
      check(cudaMemcpy(&tops[0], s->G.pool_top_ptr(), 8, cudaMemcpyDeviceToHost), "top");
      check(cudaMemcpy(&tops[1], s->H.pool_top_ptr(), 8, cudaMemcpyDeviceToHost), "top");
      s->g_top = tops[0];
      s->h_top = tops[1];
      dev_alloc(&s->d_locks, s->n, "row locks");
      check(cudaMemset(s->d_locks, 0, sizeof(unsigned long long) * s->n), "locks");
      dev_alloc(&s->d_round, 1, "round counter");
      dev_alloc(&s->d_work, 1, "walk work counter");
      dev_alloc(&s->b.mark, s->n, "row marks");
      for (int i = 0; i < 2; ++i) {
        dev_alloc(&s->b.fp_cnt[i], s->n, "append counts");
        dev_alloc(&s->b.fp_head[i], s->n, "append heads");
        check(cudaMemset(s->b.fp_cnt[i], 0, sizeof(uint32_t) * s->n), "append counts");
        check(cudaMemset(s->b.fp_head[i], 0xFF, sizeof(uint32_t) * s->n), "append heads");
      }
      check(cudaMemset(s->b.mark, 0, sizeof(uint32_t) * s->n), "row marks");
      dev_alloc(&s->b.fl_depth, s->n, "flow depths");
      dev_alloc(&s->b.save_idx, s->n, "saved-row index");
      s->b.n_vertices = s->n;
      check(cudaMemset(s->b.fl_depth, 0, sizeof(uint32_t) * s->n), "flow depths");
      check(cudaMemset(s->d_round, 0, sizeof(unsigned long long)), "round counter");
      dev_alloc(&s->d_ctl, 1, "batch ctl");
      s->b.ctl = s->d_ctl;
      dev_alloc(&s->d_counts, 8, "shard / kind counts");
      check(cudaMallocHost(reinterpret_cast<void**>(&s->h_counts), 8 * sizeof(uint32_t)),
            "pinned counts");
      check(cudaMallocHost(reinterpret_cast<void**>(&s->h_ctl), sizeof(BatchCtl)), "pinned ctl");
      s->coop_blocks = coop_grid_blocks(device);
      dev_alloc(&s->d_epoch, 1, "batch epoch");
      check(cudaMemset(s->d_epoch, 0, sizeof(unsigned long long)), "batch epoch");
      dev_alloc(&s->d_abort, 1, "abort flag");
      check(cudaMemset(s->d_abort, 0, sizeof(unsigned int)), "abort flag");
      ensure_batch(s, 1024, 256);
    } catch (...) {
      dyg_session_destroy(s);
      throw;
    }
    *out = s;
  });
}

void dyg_session_destroy(dyg_session* s) {
  if (s == nullptr) return;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (CapturedGraph& g : s->graphs) destroy_graph(g);
  s->graphs.clear();
  if (s->copy_stream) cudaStreamSynchronize(s->copy_stream);
  for (cudaEvent_t e : s->ready) cudaEventDestroy(e);
  s->ready.clear();
  dev_free(s->d_replay);
  dev_free(s->d_kinds);
  if (s->h_kinds) cudaFreeHost(s->h_kinds);
  s->h_kinds = nullptr;
  if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
  s->copy_stream = nullptr;
  if (s->aux_stream) {
    cudaStreamSynchronize(s->aux_stream);
    cudaStreamDestroy(s->aux_stream);
  }
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  free_batch(s);
  dev_free(s->b.mout.has_path);
  dev_free(s->b.mout.path_len);
  dev_free(s->b.mout.steps);
  dev_free(s->b.mout.resistance);
  dev_free(s->b.mout.paths);
  dev_free(s->b.mscratch.acc);
  dev_free(s->b.mscratch.term);
  dev_free(s->b.mscratch.steps);
  dev_free(s->b.mscratch.paths);
  dev_free(s->b.mscratch.rvals);
  dev_free(s->d_ctl);
  s->b.ctl = nullptr;
  dev_free(s->d_locks);
  dev_free(s->d_round);
  dev_free(s->d_work);
  dev_free(s->b.mark);
  for (int i = 0; i < 2; ++i) {
    dev_free(s->b.fp_cnt[i]);
    dev_free(s->b.fp_head[i]);
  }
  dev_free(s->b.fl_depth);
  dev_free(s->b.save_idx);
  dev_free(s->b.side_id);
  dev_free(s->b.side_w);
  dev_free(s->d_stream);
  if (s->h_ctl) cudaFreeHost(s->h_ctl);
  if (s->h_counts) cudaFreeHost(s->h_counts);
  dev_free(s->d_counts);
  dev_free(s->d_ctls);
  if (s->h_ctls) cudaFreeHost(s->h_ctls);
  if (s->h_shard_ctls) cudaFreeHost(s->h_shard_ctls);
  dev_free(s->d_abort);
  dev_free(s->d_up_kinds);
  dev_free(s->px_area);
  dev_free(s->px_ep);
  if (s->h_up_kinds) cudaFreeHost(s->h_up_kinds);
  for (cudaEvent_t e : s->up_ready) cudaEventDestroy(e);
  if (s->ev_up_fence) cudaEventDestroy(s->ev_up_fence);
  dev_free(s->d_epoch);
  s->G.release();
  s->G_snap.release();
  s->H.release();
  s->H_snap.release();
  if (s->stream && s->own_stream) cudaStreamDestroy(s->stream);
  delete s;
}

// Asynchronous shard commits leave the host-side counter, edge counts and
// pool tops behind the device until dyg_shard_finish; every other entry
// point that reads or writes session state refuses to run until then.
static void require_settled(const dyg_session* s) {
  if (s != nullptr && !s->shard_pending.empty())
    fail(DYG_ERR_USAGE, "asynchronous shard commits pending: call dyg_shard_finish first");
  if (s != nullptr && !s->px_pending.empty())
    fail(DYG_ERR_USAGE, "a peer-exchange range is pending: call dyg_shard_peer_range_end first");
}

int dyg_replay_events(dyg_session* s, const dyg_event* events, const uint64_t* positions,
                      size_t n, uint32_t batch_index, dyg_batch_report* out,
                      uint8_t* per_event_decision) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || out == nullptr || (n && events == nullptr))
      fail(DYG_ERR_USAGE, "null argument");
    check(cudaSetDevice(s->device), "set device");
    if (n > 0xFFFFFFF0ull) fail(DYG_ERR_USAGE, "batch too large");
    if (per_event_decision) std::memset(per_event_decision, DYG_DECISION_NONE, n);
    if (s->opt.batched) {
      run_host_batch(s, events, positions, n, batch_index, out, false, per_event_decision);
    } else {
      run_immediate(s, events, positions, n, batch_index, out, per_event_decision);
    }
  });
}

int dyg_replay_batch(dyg_session* s, const dyg_event* events, size_t n_events,
                     uint32_t batch_count, uint32_t batch_index, dyg_batch_report* out,
                     uint8_t* per_event_decision) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || out == nullptr || (n_events && events == nullptr))
      fail(DYG_ERR_USAGE, "null argument");
    // sparsifier.cpp:541-548
    if (batch_index >= batch_count && batch_count > 0) fail(DYG_ERR_USAGE, "batch index out of range");
    std::vector<dyg_event> sel;
    std::vector<uint64_t> pos;
    for (size_t i = 0; i < n_events; ++i) {
      if (events[i].batch_index == batch_index) {
        sel.push_back(events[i]);
        pos.push_back(i);
      }
    }
    check(cudaSetDevice(s->device), "set device");
    if (per_event_decision) std::memset(per_event_decision, DYG_DECISION_NONE, sel.size());
    if (s->opt.batched) {
      run_host_batch(s, sel.data(), pos.data(), sel.size(), batch_index, out, false,
                     per_event_decision);
    } else {
      run_immediate(s, sel.data(), pos.data(), sel.size(), batch_index, out, per_event_decision);
    }
  });
}

int dyg_stream_upload(dyg_session* s, const dyg_event* events, size_t n_events,
                      uint32_t batch_count) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || (n_events && events == nullptr)) fail(DYG_ERR_USAGE, "null argument");
    check(cudaSetDevice(s->device), "set device");
    settle_upload(s, ~0u);
    uint32_t nbatches = batch_count;
    for (size_t i = 0; i < n_events; ++i) nbatches = std::max(nbatches, events[i].batch_index + 1);
    s->batch_cnt.assign(nbatches, 0);
    s->batch_ins.assign(nbatches, 0);
    s->batch_del.assign(nbatches, 0);
    bool grouped = true;
    for (size_t i = 0; i < n_events; ++i) {
      const uint32_t bi = events[i].batch_index;
      if (i && bi < events[i - 1].batch_index) grouped = false;
      s->batch_cnt[bi]++;
      (events[i].kind == 0 ? s->batch_ins : s->batch_del)[bi]++;
    }
    s->batch_off.assign(nbatches + 1, 0);
    for (uint32_t b = 0; b < nbatches; ++b) s->batch_off[b + 1] = s->batch_off[b] + s->batch_cnt[b];
    // Captured range graphs bake in the batch structure, not the contents:
    // a re-upload with the same structure reuses them.
    s->stream_gen = fnv(fnv(fnv(0xcbf29ce484222325ull, s->batch_off.data(),
                                sizeof(uint64_t) * s->batch_off.size()),
                            s->batch_ins.data(), sizeof(uint64_t) * nbatches),
                        s->batch_del.data(), sizeof(uint64_t) * nbatches);
    if (s->stream_cap < n_events || s->d_stream == nullptr) {
      dev_free(s->d_stream);
      dev_alloc(&s->d_stream, std::max<size_t>(n_events, 1), "stream");
      s->stream_cap = std::max<size_t>(n_events, 1);
    }
    if (grouped && host_pinned(events)) {
      // Already in batch order and page-locked: DMA straight from the
      // caller's buffer, stream-ordered before any replay. No host copy:
      // positions are the identity, and an error message reads its event
      // back from the device.
      s->stream_events.clear();
      s->stream_positions.clear();
      if (n_events)
        check(cudaMemcpyAsync(s->d_stream, events, sizeof(DevEvent) * n_events,
                              cudaMemcpyHostToDevice, s->stream), "stream upload");
    } else {
      s->stream_events.resize(n_events);
      s->stream_positions.resize(n_events);
      std::vector<uint64_t> fill(s->batch_off.begin(), s->batch_off.end() - 1);
      for (size_t i = 0; i < n_events; ++i) {
        const uint64_t at = fill[events[i].batch_index]++;
        s->stream_events[at] = events[i];
        s->stream_positions[at] = i;
      }
      if (n_events)
        check(cudaMemcpy(s->d_stream, s->stream_events.data(), sizeof(DevEvent) * n_events,
                         cudaMemcpyHostToDevice), "stream upload");
    }
    s->stats.h2d_bytes += sizeof(DevEvent) * n_events;
    s->stream_batches = batch_count;
    s->have_stream = true;
  });
}

int dyg_stream_upload_batches(dyg_session* s, const dyg_event* events, size_t n_events,
                              const uint64_t* batch_offsets, uint32_t batch_count) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || batch_offsets == nullptr || (n_events && events == nullptr))
      fail(DYG_ERR_USAGE, "null argument");
    if (batch_offsets[0] != 0 || batch_offsets[batch_count] != n_events)
      fail(DYG_ERR_USAGE, "batch offsets do not cover the events");
    for (uint32_t b = 0; b < batch_count; ++b)
      if (batch_offsets[b + 1] < batch_offsets[b]) fail(DYG_ERR_USAGE, "batch offsets must not decrease");
    if (!host_pinned(events)) {  // pageable: the synchronous grouping path
      if (dyg_stream_upload(s, events, n_events, batch_count) != DYG_OK)
        fail(DYG_ERR_USAGE, std::string(g_last_error));
      return;
    }
    check(cudaSetDevice(s->device), "set device");
    settle_upload(s, ~0u);  // a previous asynchronous upload has landed
    if (s->copy_stream == nullptr)
      check(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking), "copy stream");
    if (s->ev_up_fence == nullptr)
      check(cudaEventCreateWithFlags(&s->ev_up_fence, cudaEventDisableTiming), "event");
    if (s->stream_cap < n_events || s->d_stream == nullptr) {
      check(cudaStreamSynchronize(s->stream), "stream buffer");
      dev_free(s->d_stream);
      dev_alloc(&s->d_stream, std::max<size_t>(n_events, 1), "stream");
      s->stream_cap = std::max<size_t>(n_events, 1);
    }
    if (s->up_kinds_cap < batch_count) {
      check(cudaStreamSynchronize(s->copy_stream), "kind counts");
      dev_free(s->d_up_kinds);
      if (s->h_up_kinds) cudaFreeHost(s->h_up_kinds);
      s->h_up_kinds = nullptr;
      dev_alloc(&s->d_up_kinds, 2ull * batch_count, "kind counts");
      check(cudaMallocHost(reinterpret_cast<void**>(&s->h_up_kinds),
                           2 * sizeof(uint32_t) * std::max<uint32_t>(batch_count, 1)),
            "pinned kind counts");
      s->up_kinds_cap = batch_count;
    }
    while (s->up_ready.size() < batch_count) {
      cudaEvent_t e;
      check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      s->up_ready.push_back(e);
    }
    s->batch_off.assign(batch_offsets, batch_offsets + batch_count + 1ull);
    s->batch_cnt.assign(batch_count, 0);
    for (uint32_t b = 0; b < batch_count; ++b) s->batch_cnt[b] = batch_offsets[b + 1] - batch_offsets[b];
    s->batch_ins.assign(batch_count, 0);
    s->batch_del.assign(batch_count, 0);
    s->up_settled.assign(batch_count, 0);
    s->stream_events.clear();
    s->stream_positions.clear();
    // The copy stream overwrites d_stream only after the session's enqueued
    // work (which may still read the previous stream) is done.
    check(cudaEventRecord(s->ev_up_fence, s->stream), "upload fence");
    check(cudaStreamWaitEvent(s->copy_stream, s->ev_up_fence, 0), "upload fence");
    for (uint32_t b = 0; b < batch_count; ++b) {
      const uint64_t nb = s->batch_cnt[b];
      if (nb) {
        check(cudaMemcpyAsync(s->d_stream + batch_offsets[b], events + batch_offsets[b],
                              sizeof(DevEvent) * nb, cudaMemcpyHostToDevice, s->copy_stream),
              "stream upload");
        s->stats.kernel_launches += launch_count_kinds(s->d_stream + batch_offsets[b],
                                                       static_cast<uint32_t>(nb),
                                                       s->d_up_kinds + 2ull * b, s->copy_stream);
        check(cudaMemcpyAsync(s->h_up_kinds + 2ull * b, s->d_up_kinds + 2ull * b,
                              2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->copy_stream),
              "kind counts");
      } else {
        s->h_up_kinds[2ull * b] = s->h_up_kinds[2ull * b + 1] = 0;
      }
      check(cudaEventRecord(s->up_ready[b], s->copy_stream), "upload event");
    }
    s->stats.h2d_bytes += sizeof(DevEvent) * n_events;
    s->stream_batches = batch_count;
    s->have_stream = true;
    s->up_pending = true;
  });
}

int dyg_replay_uploaded(dyg_session* s, uint32_t batch_index, dyg_batch_report* out) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || out == nullptr) fail(DYG_ERR_USAGE, "null argument");
    if (!s->have_stream) fail(DYG_ERR_USAGE, "no stream uploaded");
    if (batch_index >= s->stream_batches && s->stream_batches > 0)
      fail(DYG_ERR_USAGE, "batch index out of range");
    check(cudaSetDevice(s->device), "set device");
    settle_upload(s, ~0u);
    if (batch_index >= s->batch_cnt.size()) {
      run_deferred(s, nullptr, nullptr, nullptr, 0, 0, 0, batch_index, out, false);
      return;
    }
    const uint64_t off = s->batch_off[batch_index];
    const uint32_t nb = static_cast<uint32_t>(s->batch_cnt[batch_index]);
    if (!s->opt.batched) {
      std::vector<dyg_event> ev(nb);
      std::vector<uint64_t> pos(nb);
      if (uploaded_host(s, off)) {
        std::memcpy(ev.data(), s->stream_events.data() + off, sizeof(dyg_event) * nb);
        std::memcpy(pos.data(), s->stream_positions.data() + off, sizeof(uint64_t) * nb);
      } else {
        check(cudaMemcpy(ev.data(), s->d_stream + off, sizeof(dyg_event) * nb,
                         cudaMemcpyDeviceToHost), "batch read-back");
        for (uint32_t i = 0; i < nb; ++i) pos[i] = off + i;
      }
      run_immediate(s, ev.data(), pos.data(), nb, batch_index, out);
      return;
    }
    run_deferred(s, s->d_stream + off, uploaded_host(s, off), uploaded_pos(s, off), nb,
                 static_cast<uint32_t>(s->batch_ins[batch_index]),
                 static_cast<uint32_t>(s->batch_del[batch_index]), batch_index, out, false,
                 nullptr, nullptr, off);
  });
}

int dyg_replay_uploaded_range(dyg_session* s, uint32_t first, uint32_t count,
                              dyg_batch_report* out, uint8_t* per_event_decision) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || (count && out == nullptr)) fail(DYG_ERR_USAGE, "null argument");
    if (!s->have_stream) fail(DYG_ERR_USAGE, "no stream uploaded");
    if (count && static_cast<uint64_t>(first) + count > s->stream_batches && s->stream_batches > 0)
      fail(DYG_ERR_USAGE, "batch index out of range");
    if (!s->opt.batched) fail(DYG_ERR_USAGE, "batch ranges need batched (deferred) mode");
    check(cudaSetDevice(s->device), "set device");
    settle_upload(s, ~0u);
    if (per_event_decision)
      for (uint32_t b = first; b < first + count && b < s->batch_cnt.size(); ++b)
        for (uint64_t k = s->batch_off[b]; k < s->batch_off[b + 1]; ++k)
          per_event_decision[s->stream_positions.empty() ? k : s->stream_positions[k]] =
              DYG_DECISION_NONE;
    run_uploaded_range(s, first, count, out, per_event_decision);
  });
}

int dyg_replay_stream(dyg_session* s, const dyg_event* events, size_t n_events,
                      const uint64_t* batch_offsets, uint32_t batch_count,
                      dyg_batch_report* out, uint8_t* per_event_decision) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || (batch_count && out == nullptr) || (n_events && events == nullptr))
      fail(DYG_ERR_USAGE, "null argument");
    check(cudaSetDevice(s->device), "set device");
    // Batch ranges: given, or found by one pass when the events are grouped.
    std::vector<uint64_t> off;
    const uint64_t* o = batch_offsets;
    bool grouped = true;
    if (o == nullptr) {
      off.assign(batch_count + 1ull, 0);
      uint32_t prev = 0;
      for (size_t i = 0; i < n_events && grouped; ++i) {
        const uint32_t bi = events[i].batch_index;
        if (bi < prev || bi >= batch_count) grouped = false;
        else ++off[bi + 1ull];
        prev = bi;
      }
      for (uint32_t b = 0; b < batch_count; ++b) off[b + 1ull] += off[b];
      o = off.data();
    } else if (o[batch_count] != n_events || o[0] != 0) {
      fail(DYG_ERR_USAGE, "batch offsets do not cover the events");
    }
    if (per_event_decision) std::memset(per_event_decision, DYG_DECISION_NONE, n_events);
    if (grouped && s->opt.batched) {
      run_stream(s, events, n_events, o, batch_count, out, per_event_decision);
      return;
    }
    // Ungrouped events or immediate mode: the per-batch reference path.
    for (uint32_t b = 0; b < batch_count; ++b) {
      std::vector<dyg_event> ev;
      std::vector<uint64_t> pos;
      for (size_t i = 0; i < n_events; ++i)
        if (events[i].batch_index == b) {
          ev.push_back(events[i]);
          pos.push_back(i);
        }
      if (s->opt.batched)
        run_host_batch(s, ev.data(), pos.data(), ev.size(), b, &out[b], false, per_event_decision,
                       pos.data());
      else
        run_immediate(s, ev.data(), pos.data(), ev.size(), b, &out[b], per_event_decision,
                      pos.data());
    }
  });
}

int dyg_apply_insertion(dyg_session* s, uint32_t u, uint32_t v, double w, int* decision) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    check(cudaSetDevice(s->device), "set device");
    // apply_insertion validates through insert_edge (graph.cpp:64-73).
    if (u >= s->n || v >= s->n) {
      char buf[128];
      std::snprintf(buf, sizeof buf, "vertex id %u out of range (n = %u)", u >= s->n ? u : v, s->n);
      fail(DYG_ERR_USAGE, buf);
    }
    if (u == v) fail(DYG_ERR_USAGE, "self-loops are not allowed");
    if (!(w > 0.0) || !std::isfinite(w)) fail(DYG_ERR_USAGE, "edge weight must be a positive finite number");
    dyg_event e{0, u, v, 0, w};
    dyg_batch_report r{};
    const uint64_t pos = 0;
    run_host_batch(s, &e, &pos, 1, 0, &r, false);
    s->last_event_steps = r.walker_steps;
    if (decision) *decision = static_cast<int>(s->last_dec & 0xFF);
  });
}

int dyg_apply_deletion(dyg_session* s, uint32_t u, uint32_t v, int* kind, uint32_t* edges_added) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    check(cudaSetDevice(s->device), "set device");
    if (u >= s->n || v >= s->n) {
      char buf[128];
      std::snprintf(buf, sizeof buf, "vertex id %u out of range (n = %u)", u >= s->n ? u : v, s->n);
      fail(DYG_ERR_USAGE, buf);
    }
    dyg_event e{1, u, v, 0, 0.0};
    dyg_batch_report r{};
    const uint64_t pos = 0;
    try {
      run_host_batch(s, &e, &pos, 1, 0, &r, false);
    } catch (const ApiError& err) {
      // delete_edge's own message without the replay prefix (graph.cpp:90-95).
      if (err.code == DYG_ERR_DATA) {
        char buf[128];
        std::snprintf(buf, sizeof buf, "edge (%u, %u) does not exist", u, v);
        fail(DYG_ERR_DATA, buf);
      }
      throw;
    }
    s->last_event_steps = r.walker_steps;
    if (kind) *kind = static_cast<int>(s->last_dec & 0xFF);
    if (edges_added) *edges_added = s->last_dec >> 8;
  });
}

uint64_t dyg_last_event_steps(const dyg_session* s) { return s ? s->last_event_steps : 0; }
uint64_t dyg_update_counter(const dyg_session* s) { return s ? s->counter : 0; }

int dyg_graph_info(const dyg_session* s, int which, uint32_t* n, uint64_t* edges, double* density) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    const uint64_t e = which == 0 ? s->g_edges : s->h_edges;
    if (n) *n = s->n;
    if (edges) *edges = e;
    if (density) *density = density_of(e, s->n);
  });
}

int dyg_export_rows(dyg_session* s, int which, uint64_t* row_ptr, uint32_t* ids, double* w,
                    uint64_t capacity) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || row_ptr == nullptr) fail(DYG_ERR_USAGE, "null argument");
    check(cudaSetDevice(s->device), "set device");
    const uint64_t nnz = which == 0 ? s->G.export_rows(row_ptr, ids, w, capacity, s->stream)
                                    : s->H.export_rows(row_ptr, ids, w, capacity, s->stream);
    if (nnz > capacity) fail(DYG_ERR_USAGE, "export buffers too small");
  });
}

int dyg_session_snapshot(dyg_session* s) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    check(cudaSetDevice(s->device), "set device");
    s->G_snap.copy_from(s->G, s->stream);
    s->H_snap.copy_from(s->H, s->stream);
    check(cudaStreamSynchronize(s->stream), "snapshot");
    s->counter_snap = s->counter;
    s->g_edges_snap = s->g_edges;
    s->h_edges_snap = s->h_edges;
    s->g_top_snap = s->g_top;
    s->h_top_snap = s->h_top;
    s->have_snap = true;
  });
}

int dyg_session_restore(dyg_session* s) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    if (!s->have_snap) fail(DYG_ERR_USAGE, "no snapshot taken");
    s->last_t1 = 0;  // the restore is not a gap between batches of one replay
    check(cudaSetDevice(s->device), "set device");
    s->G.copy_from(s->G_snap, s->stream);
    s->H.copy_from(s->H_snap, s->stream);
    s->stats.kernel_launches += 2;
    s->counter = s->counter_snap;
    s->g_edges = s->g_edges_snap;
    s->h_edges = s->h_edges_snap;
    s->g_top = s->g_top_snap;
    s->h_top = s->h_top_snap;
    if (s->debug_sync) check(cudaStreamSynchronize(s->stream), "restore");
  });
}

// ---- cross-process checkpoint (SURVEY.md 5 "checkpoint / resume") --------
// A checkpoint is (options, update_counter, G rows, H rows) in reference row
// order: exactly the state SparsifierState carries (sparsifier.hpp:105-111),
// so a session resumed from it walks with the same keys
// (walker_seed(seed, update_id, i), sparsifier.cpp:431) and samples the same
// adjacency order as the one that wrote it. Layout (little-endian):
//   "DYGCKPT1" | dyg_options | u64 counter | 2 x {u32 n, u32 0, u64 nnz,
//   u64 row_ptr[n+1], u32 ids[nnz], f64 w[nnz]} | u64 FNV-1a of all before.
namespace {

constexpr char kCkptMagic[8] = {'D', 'Y', 'G', 'C', 'K', 'P', 'T', '1'};

struct CkptFile {
  std::FILE* f = nullptr;
  uint64_t h = 1469598103934665603ull;
  ~CkptFile() {
    if (f) std::fclose(f);
  }
  void hash(const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  }
  void put(const void* p, size_t n, const std::string& path) {
    hash(p, n);
    if (n && std::fwrite(p, 1, n, f) != n) fail(DYG_ERR_DATA, "cannot write checkpoint " + path);
  }
  void get(void* p, size_t n, const std::string& path) {
    if (n && std::fread(p, 1, n, f) != n)
      fail(DYG_ERR_DATA, "truncated checkpoint " + path);
    hash(p, n);
  }
};

struct HostRows {
  uint32_t n = 0;
  std::vector<uint64_t> row_ptr;
  std::vector<uint32_t> ids;
  std::vector<double> w;
  dyg_csr csr() const { return dyg_csr{n, 0, row_ptr.data(), ids.data(), w.data()}; }
};

}  // namespace

int dyg_session_options(const dyg_session* s, dyg_options* out) {
  return guarded([&] {
    if (s == nullptr || out == nullptr) fail(DYG_ERR_USAGE, "null argument");
    *out = s->opt;
  });
}

int dyg_session_save(dyg_session* s, const char* path) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || path == nullptr) fail(DYG_ERR_USAGE, "null argument");
    check(cudaSetDevice(s->device), "set device");
    HostRows rows[2];
    for (int which = 0; which < 2; ++which) {
      HostRows& r = rows[which];
      r.n = s->n;
      r.row_ptr.resize(static_cast<size_t>(s->n) + 1);
      const uint64_t nnz = 2 * (which == 0 ? s->g_edges : s->h_edges);
      r.ids.resize(nnz);
      r.w.resize(nnz);
      const uint64_t got = which == 0
                               ? s->G.export_rows(r.row_ptr.data(), r.ids.data(), r.w.data(), nnz, s->stream)
                               : s->H.export_rows(r.row_ptr.data(), r.ids.data(), r.w.data(), nnz, s->stream);
      if (got != nnz) fail(DYG_ERR_DEVICE, "checkpoint: edge count mismatch on export");
    }
    CkptFile out;
    const std::string p(path);
    out.f = std::fopen(path, "wb");
    if (out.f == nullptr) fail(DYG_ERR_DATA, "cannot open checkpoint " + p + " for writing");
    out.put(kCkptMagic, sizeof kCkptMagic, p);
    out.put(&s->opt, sizeof s->opt, p);
    out.put(&s->counter, sizeof s->counter, p);
    for (const HostRows& r : rows) {
      const uint32_t hdr[2] = {r.n, 0};
      const uint64_t nnz = r.ids.size();
      out.put(hdr, sizeof hdr, p);
      out.put(&nnz, sizeof nnz, p);
      out.put(r.row_ptr.data(), r.row_ptr.size() * sizeof(uint64_t), p);
      out.put(r.ids.data(), nnz * sizeof(uint32_t), p);
      out.put(r.w.data(), nnz * sizeof(double), p);
    }
    const uint64_t sum = out.h;
    out.put(&sum, sizeof sum, p);
    if (std::fflush(out.f) != 0) fail(DYG_ERR_DATA, "cannot write checkpoint " + p);
  });
}

int dyg_session_load(const char* path, int device, dyg_session** out) {
  int rc = guarded([&] {
    if (path == nullptr || out == nullptr) fail(DYG_ERR_USAGE, "null argument");
    *out = nullptr;
    CkptFile in;
    const std::string p(path);
    in.f = std::fopen(path, "rb");
    if (in.f == nullptr) fail(DYG_ERR_DATA, "cannot open checkpoint " + p);
    char magic[8];
    in.get(magic, sizeof magic, p);
    if (std::memcmp(magic, kCkptMagic, sizeof magic) != 0)
      fail(DYG_ERR_DATA, "not a checkpoint file: " + p);
    dyg_options opt{};
    uint64_t counter = 0;
    in.get(&opt, sizeof opt, p);
    in.get(&counter, sizeof counter, p);
    HostRows rows[2];
    for (HostRows& r : rows) {
      uint32_t hdr[2];
      uint64_t nnz = 0;
      in.get(hdr, sizeof hdr, p);
      in.get(&nnz, sizeof nnz, p);
      if (nnz > (1ull << 40) || hdr[0] == 0xFFFFFFFFu) fail(DYG_ERR_DATA, "corrupt checkpoint " + p);
      r.n = hdr[0];
      r.row_ptr.resize(static_cast<size_t>(r.n) + 1);
      r.ids.resize(nnz);
      r.w.resize(nnz);
      in.get(r.row_ptr.data(), r.row_ptr.size() * sizeof(uint64_t), p);
      in.get(r.ids.data(), nnz * sizeof(uint32_t), p);
      in.get(r.w.data(), nnz * sizeof(double), p);
      if (r.row_ptr[0] != 0 || r.row_ptr[r.n] != nnz) fail(DYG_ERR_DATA, "corrupt checkpoint " + p);
    }
    const uint64_t want = in.h;
    uint64_t sum = 0;
    in.get(&sum, sizeof sum, p);
    if (sum != want) fail(DYG_ERR_DATA, "checkpoint checksum mismatch: " + p);
    const dyg_csr g = rows[0].csr(), h = rows[1].csr();
    dyg_session* s = nullptr;
    const int created = dyg_session_create(&g, &h, &opt, device, &s);
    if (created != DYG_OK) fail(created, std::string(g_last_error));
    s->counter = counter;
    *out = s;
  });
  return rc;
}

int dyg_session_set_walk_counters(dyg_session* s, int on) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    s->walk_counters = on != 0;
  });
}

int dyg_session_stats(const dyg_session* s, dyg_stats* out) {
  return guarded([&] {
    if (s == nullptr || out == nullptr) fail(DYG_ERR_USAGE, "null argument");
    *out = s->stats;
    out->pool_used = s->g_top + s->h_top;
    out->pool_capacity = s->G.pool_capacity() + s->H.pool_capacity();
  });
}

int dyg_session_reset_stats(dyg_session* s) {
  return guarded([&] {
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    s->stats = dyg_stats{};
    s->last_t1 = 0;
  });
}

// Measurement switch DYG_L2_PERSIST_MB=X (read when a stream is bound): an
// L2 access-policy window over the head of H's slab table with X MB of
// persisting lines. Measured: no gain --
// the walks' row accesses are uniform over H, so persisting a part of it
// only moves hits between regions.
void apply_l2_window(dyg_session* s) {
  const char* e = std::getenv("DYG_L2_PERSIST_MB");
  if (e == nullptr) return;
  const double mb = std::atof(e);
  int max_win = 0;
  cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, s->device);
  const DevGraph<kCapH> h = s->H.view();
  const size_t bytes = std::min<size_t>(sizeof(Slab<kCapH>) * static_cast<size_t>(h.n),
                                        static_cast<size_t>(max_win));
  const size_t persist = static_cast<size_t>(mb * 1048576.0);
  if (bytes == 0 || persist == 0) return;
  check(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist), "persisting L2");
  cudaStreamAttrValue a{};
  a.accessPolicyWindow.base_ptr = h.slab;
  a.accessPolicyWindow.num_bytes = bytes;
  a.accessPolicyWindow.hitRatio = static_cast<float>(std::min(1.0, static_cast<double>(persist) / bytes));
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  check(cudaStreamSetAttribute(s->stream, cudaStreamAttributeAccessPolicyWindow, &a), "L2 window");
  if (std::getenv("DYG_GRAPH_DEBUG"))
    std::fprintf(stderr, "dyg: L2 window %zu MB over H, %zu MB persisting (max window %d MB)\n",
                 bytes >> 20, persist >> 20, max_win >> 20);
}

int dyg_set_stream(dyg_session* s, void* cuda_stream) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    check(cudaStreamSynchronize(s->stream), "set stream");
    if (s->own_stream) cudaStreamDestroy(s->stream);
    s->stream = static_cast<cudaStream_t>(cuda_stream);
    s->own_stream = false;
    apply_l2_window(s);
  });
}

// ---- multi-GPU split ---------------------------------------
namespace {
// dyg_shard_begin's body: `dev` == nullptr uploads `events`, else the batch
// is already on the device (the uploaded stream) with known kind counts.
void shard_begin_impl(dyg_session* s, const dyg_event* events, const uint64_t* positions,
                      size_t n, uint32_t batch_index, const DevEvent* dev, uint32_t n_ins0,
                      uint32_t n_del0, uint64_t* n_reach, uint64_t* n_minpath) {
    if (!s->opt.batched) fail(DYG_ERR_USAGE, "the multi-GPU split needs batched (deferred) mode");
    check(cudaSetDevice(s->device), "set device");
    s->shard_active = false;
    s->shard_host = reinterpret_cast<const DevEvent*>(events);
    s->shard_pos = positions;
    s->shard_dev = dev ? dev : s->d_events;
    uint32_t n_ins = n_ins0, n_del = n_del0;
    if (n > 0 && dev == nullptr) {
      ensure_batch(s, static_cast<uint32_t>(n), 0);
      upload_events(s, events, n);
      count_kinds(s, static_cast<uint32_t>(n), n_ins, n_del);
    }
    s->shard_nb = static_cast<uint32_t>(n);
    s->shard_ins = n_ins;
    s->shard_del = n_del;
    s->shard_batch = batch_index;
    s->shard_wall0 = std::chrono::steady_clock::now();
    const bool chained = !s->shard_pending.empty();  // after asynchronous commits
    s->shard_counter = chained ? s->shard_next_counter : s->counter;
    s->shard_nq_r = s->shard_nq_m = 0;
    if (n > 0) {
      ensure_batch(s, static_cast<uint32_t>(n), n_del);
      Pending p;
      bind_pending(s, p);
      p.counter_base = s->shard_counter;
      // A chained batch keeps the device abort flag: after a failed earlier
      // batch it does nothing (as in a range replay).
      if (!chained) reset_abort(s);
      p.dev = s->shard_dev;
      p.host = s->shard_host;
      p.pos = s->shard_pos;
      p.pos_base = s->shard_pos_base;
      p.nb = s->shard_nb;
      p.n_ins = n_ins;
      p.n_del = n_del;
      p.batch = batch_index;
      p.shard = true;
      // The prepare as a captured graph (the multi-GPU split launches its
      // three device segments per batch -- prepare, walk, commit -- each
      // as one graph, like the single-GPU path's one graph per batch).
      prepare_bind(s, p);
      uint64_t key = session_fingerprint(s, 7);
      const uint64_t shape[] = {reinterpret_cast<uint64_t>(p.dev), reinterpret_cast<uint64_t>(p.dctl),
                                p.nb, p.n_ins, p.n_del};
      key = fnv(key, shape, sizeof shape);
      p.launches += enqueue_captured(s, key, p.counter_base, [&] {
        Pending q = p;
        phase_prepare(s, q);
        return q.launches;
      });
      // No host round trip: the exchange is sized by upper bounds of the
      // query counts (a reach query per insertion at most, a min-path query
      // per deletion); the walk and the commit read the exact counts on the
      // device. Validation errors surface at dyg_shard_commit.
      s->shard_launches = p.launches;
      s->shard_nq_r = n_ins;
      s->shard_nq_m = n_del;
    }
    s->shard_active = true;
    if (n_reach) *n_reach = s->shard_nq_r;
    if (n_minpath) *n_minpath = s->shard_nq_m;
}
}  // namespace

int dyg_shard_begin(dyg_session* s, const dyg_event* events, const uint64_t* positions, size_t n,
                    uint32_t batch_index, uint64_t* n_reach, uint64_t* n_minpath) {
  return guarded([&] {
    if (s == nullptr || (n && events == nullptr)) fail(DYG_ERR_USAGE, "null argument");
    s->shard_pos_base = 0;
    shard_begin_impl(s, events, positions, n, batch_index, nullptr, 0, 0, n_reach, n_minpath);
  });
}

int dyg_shard_begin_uploaded(dyg_session* s, uint32_t batch_index, uint64_t* n_reach,
                             uint64_t* n_minpath) {
  return guarded([&] {
    if (s == nullptr) fail(DYG_ERR_USAGE, "null argument");
    if (batch_index >= s->batch_cnt.size()) fail(DYG_ERR_USAGE, "batch index out of range");
    check(cudaSetDevice(s->device), "set device");
    if (s->up_pending) {
      // Only this batch has to have landed: later uploads keep overlapping
      // the work enqueued before them.
      settle_upload(s, batch_index);
      check(cudaStreamWaitEvent(s->stream, s->up_ready[batch_index], 0), "upload wait");
    }
    const uint64_t off = s->batch_off[batch_index];
    const size_t n = s->batch_cnt[batch_index];
    s->shard_pos_base = off;
    shard_begin_impl(s, reinterpret_cast<const dyg_event*>(uploaded_host(s, off)),
                     uploaded_pos(s, off), n, batch_index, s->d_stream + off,
                     static_cast<uint32_t>(s->batch_ins[batch_index]),
                     static_cast<uint32_t>(s->batch_del[batch_index]), n_reach, n_minpath);
  });
}

size_t dyg_shard_record_bytes(const dyg_session* s, int minpath) {
  if (s == nullptr) return 0;
  return minpath ? min_record_bytes(s->opt.walk.step_cap) : sizeof(ReachRecord);
}

int dyg_shard_walk(dyg_session* s, int rank, int world, void* reach_records,
                   void* minpath_records) {
  return guarded([&] {
    if (s == nullptr || !s->shard_active) fail(DYG_ERR_USAGE, "no shard batch in progress");
    if (world < 1 || rank < 0 || rank >= world) fail(DYG_ERR_USAGE, "invalid rank / world");
    check(cudaSetDevice(s->device), "set device");
    if (s->shard_nb == 0) return;
    auto range = [&](uint32_t nq, uint32_t* lo, uint32_t* cnt, uint32_t* slots) {
      const uint64_t a = static_cast<uint64_t>(nq) * rank / world;
      const uint64_t b = static_cast<uint64_t>(nq) * (rank + 1) / world;
      *lo = static_cast<uint32_t>(a);
      *cnt = static_cast<uint32_t>(b - a);
      *slots = static_cast<uint32_t>((static_cast<uint64_t>(nq) + world - 1) / world);
    };
    // Slots per rank from the host bounds; the ranges themselves come from
    // the device counts (launch_shard_range).
    uint32_t lo_r, n_r, sl_r, lo_m, n_m, sl_m;
    range(s->shard_nq_r, &lo_r, &n_r, &sl_r);
    range(s->shard_nq_m, &lo_m, &n_m, &sl_m);
    if ((sl_r && reach_records == nullptr) || (sl_m && minpath_records == nullptr))
      fail(DYG_ERR_USAGE, "null record buffer");
    Pending p;
    bind_pending(s, p);
    p.nb = s->shard_nb;
    p.n_ins = s->shard_ins;
    p.n_del = s->shard_del;
    s->b.ctl = p.dctl;
    uint64_t key = session_fingerprint(s, 4);
    const uint64_t shape[] = {static_cast<uint64_t>(rank), static_cast<uint64_t>(world), sl_r, sl_m,
                              reinterpret_cast<uint64_t>(reach_records),
                              reinterpret_cast<uint64_t>(minpath_records),
                              reinterpret_cast<uint64_t>(p.dctl), p.nb, p.n_ins, p.n_del};
    key = fnv(key, shape, sizeof shape);
    p.launches += enqueue_captured(s, key, s->shard_counter, [&] {
      Pending q = p;
      q.launches = launch_shard_range(s->b, rank, world, s->d_counts + 4, sl_r, sl_m, s->stream);
      phase_walk(s, q, false, 0, sl_r, 0, sl_m);
      q.launches += launch_pack(s->b, s->d_counts + 4, sl_r, sl_m, s->opt.walk.step_cap,
                                reach_records, minpath_records, s->stream);
      return q.launches;
    });
    // No host sync: the records are consumed in stream order (the all-gather
    // is enqueued on the session's stream).
    maybe_sync(s, "shard walk");
    s->shard_launches += p.launches;
  });
}

namespace {
// The commit-side Pending of the shard batch in progress, with the unpack of
// the gathered records enqueued.
Pending shard_commit_pending(dyg_session* s, int world, const void* reach_gathered,
                             const void* minpath_gathered) {
    const uint32_t sl_r = static_cast<uint32_t>((s->shard_nq_r + world - 1ull) / world);
    const uint32_t sl_m = static_cast<uint32_t>((s->shard_nq_m + world - 1ull) / world);
    Pending p;
    bind_pending(s, p);
    p.counter_base = s->shard_counter;
    p.dev = s->shard_dev;
    p.host = s->shard_host;
    p.pos = s->shard_pos;
    p.pos_base = s->shard_pos_base;
    p.nb = s->shard_nb;
    p.n_ins = s->shard_ins;
    p.n_del = s->shard_del;
    p.batch = s->shard_batch;
    p.wall0 = s->shard_wall0;
    p.launches = s->shard_launches;
    s->b.ctl = p.dctl;
    s->b.events = const_cast<DevEvent*>(p.dev);
    s->b.side_top = &p.dctl->side_top;
    s->b.scratch_edges = &p.dctl->scratch_edges;
    s->shard_unpack = [=](dyg_session* ss) {
      return launch_unpack(ss->b, ss->shard_nq_r, ss->shard_nq_m, world, sl_r, sl_m,
                           ss->opt.walk.step_cap, reach_gathered, minpath_gathered, ss->stream);
    };
    const uint64_t shape[] = {static_cast<uint64_t>(world), sl_r, sl_m, s->shard_nq_r, s->shard_nq_m,
                              reinterpret_cast<uint64_t>(reach_gathered),
                              reinterpret_cast<uint64_t>(minpath_gathered)};
    s->shard_unpack_key = fnv(0x9e3779b97f4a7c15ull, shape, sizeof shape);
    return p;
}

// Unpack + commit of the shard batch as one captured segment (downloading
// the control block to p.hctl).
void shard_commit_enqueue(dyg_session* s, Pending& p) {
  uint64_t key = session_fingerprint(s, 5);
  const uint64_t shape[] = {s->shard_unpack_key, reinterpret_cast<uint64_t>(p.dev),
                            reinterpret_cast<uint64_t>(p.dctl), reinterpret_cast<uint64_t>(p.hctl),
                            reinterpret_cast<uint64_t>(p.hdec), p.nb, p.n_ins, p.n_del};
  key = fnv(key, shape, sizeof shape);
  p.launches += enqueue_captured(s, key, p.counter_base, [&] {
    Pending q = p;
    q.launches = s->shard_unpack(s);
    commit_enqueue(s, q, true);
    return q.launches;
  });
}
}  // namespace

int dyg_shard_commit(dyg_session* s, int world, const void* reach_gathered,
                     const void* minpath_gathered, dyg_batch_report* out) {
  return guarded([&] {
    if (s == nullptr || out == nullptr || !s->shard_active)
      fail(DYG_ERR_USAGE, "no shard batch in progress");
    if (world < 1) fail(DYG_ERR_USAGE, "invalid world");
    if (!s->shard_pending.empty())
      fail(DYG_ERR_USAGE, "asynchronous shard commits pending: call dyg_shard_finish first");
    check(cudaSetDevice(s->device), "set device");
    s->shard_active = false;
    if (s->shard_nb == 0) {
      empty_report(s, s->shard_batch, out);
      return;
    }
    Pending p = shard_commit_pending(s, world, reach_gathered, minpath_gathered);
    shard_commit_enqueue(s, p);
    check(cudaStreamSynchronize(s->stream), "batch");
    commit_finalize(s, p, out);
  });
}

int dyg_shard_commit_async(dyg_session* s, int world, const void* reach_gathered,
                           const void* minpath_gathered) {
  return guarded([&] {
    if (s == nullptr || !s->shard_active) fail(DYG_ERR_USAGE, "no shard batch in progress");
    if (world < 1) fail(DYG_ERR_USAGE, "invalid world");
    constexpr size_t kRing = 256;
    if (s->shard_pending.size() >= kRing)
      fail(DYG_ERR_USAGE, "too many asynchronous shard commits: call dyg_shard_finish");
    check(cudaSetDevice(s->device), "set device");
    if (s->h_shard_ctls == nullptr)
      check(cudaMallocHost(reinterpret_cast<void**>(&s->h_shard_ctls), sizeof(BatchCtl) * kRing),
            "pinned shard control blocks");
    s->shard_active = false;
    Pending p;
    if (s->shard_nb == 0) {  // an empty batch: reported at finish
      p.batch = s->shard_batch;
      p.nb = 0;
      s->shard_pending.push_back(p);
      s->shard_next_counter = s->shard_counter;
      return;
    }
    p = shard_commit_pending(s, world, reach_gathered, minpath_gathered);
    p.hctl = s->h_shard_ctls + s->shard_pending.size();
    shard_commit_enqueue(s, p);
    s->shard_pending.push_back(p);
    s->shard_next_counter = p.counter_base + p.nb;
    const uint64_t T1 = static_cast<uint64_t>(s->opt.walk.step_cap) + 1;
    s->shard_pend_g += 2ull * p.n_ins;
    s->shard_pend_h += 2ull * p.n_ins + p.n_del * (2 * T1 + 4);
  });
}

int dyg_shard_finish(dyg_session* s, dyg_batch_report* out, size_t cap, size_t* n_out) {
  return guarded([&] {
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    if (n_out) *n_out = 0;
    if (s->shard_pending.empty()) return;
    check(cudaSetDevice(s->device), "set device");
    std::vector<Pending> ps;
    ps.swap(s->shard_pending);
    s->shard_pend_g = s->shard_pend_h = 0;
    check(cudaStreamSynchronize(s->stream), "shard commits");
    for (size_t i = 0; i < ps.size(); ++i) {
      dyg_batch_report rep{};
      if (ps[i].nb == 0) empty_report(s, ps[i].batch, &rep);
      else commit_finalize(s, ps[i], &rep);  // throws at the first failing batch
      if (out && i < cap) out[i] = rep;
      if (n_out) *n_out = i + 1;
    }
  });
}

// ---- peer-memory exchange of the multi-GPU split (batch.cuh PeerX) --------
int dyg_shard_peer_create(dyg_session* s, int world, uint64_t max_reach, uint64_t max_minpath,
                          void** area, size_t* bytes, void* ipc_handle) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || area == nullptr || bytes == nullptr) fail(DYG_ERR_USAGE, "null argument");
    if (world < 1 || world > kMaxPeers)
      fail(DYG_ERR_USAGE, "peer exchange supports 1.." + std::to_string(kMaxPeers) + " ranks");
    if (!s->opt.batched) fail(DYG_ERR_USAGE, "the multi-GPU split needs batched (deferred) mode");
    check(cudaSetDevice(s->device), "set device");
    check(cudaStreamSynchronize(s->stream), "peer exchange");
    dev_free(s->px_area);
    if (s->px_ep == nullptr) dev_alloc(&s->px_ep, 1, "peer epoch");
    s->px_slots_r = static_cast<uint32_t>((max_reach + world - 1) / world);
    s->px_slots_m = static_cast<uint32_t>((max_minpath + world - 1) / world);
    s->px_world = static_cast<uint32_t>(world);
    s->px_bytes = peer_area_bytes(s->px_slots_r, s->px_slots_m, s->opt.walk.step_cap, &s->px_stride,
                                  &s->px_min_off);
    check(cudaMalloc(reinterpret_cast<void**>(&s->px_area), s->px_bytes), "peer exchange area");
    check(cudaMemset(s->px_area, 0, s->px_bytes), "peer exchange area");
    check(cudaMemset(s->px_ep, 0, sizeof(unsigned long long)), "peer epoch");
    s->px_bound = false;
    *area = s->px_area;
    *bytes = s->px_bytes;
    if (ipc_handle != nullptr) {
      cudaIpcMemHandle_t h;
      check(cudaIpcGetMemHandle(&h, s->px_area), "IPC handle of the exchange area");
      std::memcpy(ipc_handle, &h, sizeof h);
    }
  });
}

int dyg_ipc_open(const void* ipc_handle, int device, void** ptr) {
  return guarded([&] {
    if (ipc_handle == nullptr || ptr == nullptr) fail(DYG_ERR_USAGE, "null argument");
    check(cudaSetDevice(device), "set device");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof h);
    check(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "IPC open");
  });
}

int dyg_ipc_close(void* ptr) {
  return guarded([&] {
    if (ptr != nullptr) check(cudaIpcCloseMemHandle(ptr), "IPC close");
  });
}

int dyg_shard_peer_bind(dyg_session* s, int rank, int world, void* const* areas, double timeout_s) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || areas == nullptr) fail(DYG_ERR_USAGE, "null argument");
    if (s->px_area == nullptr) fail(DYG_ERR_USAGE, "no exchange area: call dyg_shard_peer_create");
    if (static_cast<uint32_t>(world) != s->px_world || rank < 0 || rank >= world)
      fail(DYG_ERR_USAGE, "invalid rank / world");
    if (areas[rank] != s->px_area) fail(DYG_ERR_USAGE, "areas[rank] must be this rank's own area");
    PeerX px{};
    px.own = s->px_area;
    for (int q = 0; q < world; ++q) {
      if (areas[q] == nullptr) fail(DYG_ERR_USAGE, "null peer area");
      px.base[q] = static_cast<const uint8_t*>(areas[q]);
    }
    px.ep = s->px_ep;
    px.stride = s->px_stride;
    px.min_off = s->px_min_off;
    px.world = world;
    px.rank = rank;
    px.timeout_ns = static_cast<unsigned long long>((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
    s->px = px;
    s->px_bound = true;
  });
}

namespace {
// The uploaded batches [first, first + count) through the peer exchange:
// every batch is prepare -> walk of this rank's query range -> pack into
// the own area + publish -> wait for the peers -> unpack from their areas
// -> commit, all enqueued (one captured graph for the range) with no host
// step; dyg_shard_peer_range_end synchronises and reports.
void peer_range_begin(dyg_session* s, uint32_t first, uint32_t count) {
  const uint32_t world = s->px_world;
  const int rank = s->px.rank;
  uint64_t sum_ins = 0, sum_del = 0;
  uint32_t max_nb = 0, max_nd = 0;
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t b = first + i;
    if (b >= s->batch_cnt.size()) continue;
    sum_ins += s->batch_ins[b];
    sum_del += s->batch_del[b];
    max_nb = std::max<uint32_t>(max_nb, static_cast<uint32_t>(s->batch_cnt[b]));
    max_nd = std::max<uint32_t>(max_nd, static_cast<uint32_t>(s->batch_del[b]));
    if ((s->batch_ins[b] + world - 1) / world > s->px_slots_r ||
        (s->batch_del[b] + world - 1) / world > s->px_slots_m)
      fail(DYG_ERR_USAGE, "batch " + std::to_string(b) +
                              " exceeds the exchange area (dyg_shard_peer_create maxima)");
  }
  ensure_batch(s, std::max<uint32_t>(max_nb, 1), max_nd);
  ensure_pools(s, sum_ins, sum_del);
  if (sum_del > 0) ensure_side_pool(s);
  if (s->ctl_cap < count) {
    dev_free(s->d_ctls);
    if (s->h_ctls) cudaFreeHost(s->h_ctls);
    s->h_ctls = nullptr;
    dev_alloc(&s->d_ctls, count, "batch control blocks");
    // Empty batches never initialise their block; the whole-range download
    // then copies defined bytes (initcheck).
    check(cudaMemset(s->d_ctls, 0, sizeof(BatchCtl) * count), "batch control blocks");
    check(cudaMallocHost(reinterpret_cast<void**>(&s->h_ctls), sizeof(BatchCtl) * count),
          "pinned control blocks");
    s->ctl_cap = count;
  }
  std::vector<Pending> ps(count);
  const uint64_t counter0 = s->counter;
  const auto wall0 = std::chrono::steady_clock::now();
  reset_abort(s);
  uint64_t counter = counter0;
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t b = first + i;
    Pending& p = ps[i];
    p.batch = b;
    p.wall0 = wall0;
    p.dctl = s->d_ctls + i;
    p.hctl = s->h_ctls + i;
    p.hdec = &s->h_counts[2];
    p.counter_base = counter;
    p.shard = true;
    if (b >= s->batch_cnt.size() || s->batch_cnt[b] == 0) continue;
    const uint64_t off = s->batch_off[b];
    p.dev = s->d_stream + off;
    p.host = uploaded_host(s, off);
    p.pos = uploaded_pos(s, off);
    p.pos_base = off;
    p.nb = static_cast<uint32_t>(s->batch_cnt[b]);
    p.n_ins = static_cast<uint32_t>(s->batch_ins[b]);
    p.n_del = static_cast<uint32_t>(s->batch_del[b]);
    counter += p.nb;
  }
  const uint32_t T = s->opt.walk.step_cap;
  auto enqueue = [&] {
    int launches = 0;
    for (uint32_t i = 0; i < count; ++i) {
      Pending p = ps[i];
      if (p.nb == 0) continue;
      const uint32_t sl_r = (p.n_ins + world - 1) / world, sl_m = (p.n_del + world - 1) / world;
      phase_prepare(s, p);
      p.launches += launch_shard_range(s->b, rank, static_cast<int>(world), s->d_counts + 4, sl_r,
                                       sl_m, s->stream);
      phase_walk(s, p, false, 0, sl_r, 0, sl_m, /*fork_g=*/true);
      p.launches += launch_pack_peer(s->b, s->d_counts + 4, sl_r, sl_m, T, s->px, s->stream);
      p.launches += launch_unpack_peer(s->b, p.n_ins, p.n_del, sl_r, sl_m, T, s->px, s->stream);
      commit_enqueue(s, p, false);
      ps[i].launches = p.launches;
      launches += p.launches;
    }
    check(cudaMemcpyAsync(s->h_ctls, s->d_ctls, sizeof(BatchCtl) * count, cudaMemcpyDeviceToHost,
                          s->stream), "ctl download");
    return launches;
  };
  CapturedGraph* g = nullptr;
  if (graphs_usable(s)) {
    uint64_t key = session_fingerprint(s, 6);
    const uint64_t shape[] = {first, count, s->stream_gen, reinterpret_cast<uint64_t>(s->d_stream),
                              reinterpret_cast<uint64_t>(s->d_ctls),
                              reinterpret_cast<uint64_t>(s->h_ctls), world,
                              static_cast<uint64_t>(rank)};
    key = fnv(key, shape, sizeof shape);
    key = fnv(key, &s->px, sizeof s->px);
    g = find_graph(s, key);
    if (g == nullptr) g = capture_graph(s, key, counter0, enqueue);
    else
      for (uint32_t i = 0; i < count; ++i) ps[i].launches = g->per_batch[i];
    if (g != nullptr) {
      if (g->per_batch.empty())
        for (uint32_t i = 0; i < count; ++i) g->per_batch.push_back(ps[i].launches);
      launch_graph(s, *g, counter0);
    }
  }
  if (g == nullptr) enqueue();
  s->px_pending = std::move(ps);
  s->px_first = first;
}

// The same batches while the stream is still being uploaded batch by batch
// (dyg_stream_upload_batches right before, as replay(stream) does): one
// graph per batch, each enqueued as soon as its own upload has landed, so
// the upload overlaps the earlier batches' work (run_stream's pipeline).
void peer_range_pipelined(dyg_session* s, uint32_t first, uint32_t count) {
  const uint32_t world = s->px_world;
  const int rank = s->px.rank;
  uint32_t max_nb = 1;
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t b = first + i;
    if (b < s->batch_cnt.size()) max_nb = std::max<uint32_t>(max_nb, static_cast<uint32_t>(s->batch_cnt[b]));
  }
  ensure_batch(s, max_nb, 0);
  if (s->ctl_cap < count) {
    dev_free(s->d_ctls);
    if (s->h_ctls) cudaFreeHost(s->h_ctls);
    s->h_ctls = nullptr;
    dev_alloc(&s->d_ctls, count, "batch control blocks");
    check(cudaMemset(s->d_ctls, 0, sizeof(BatchCtl) * count), "batch control blocks");
    check(cudaMallocHost(reinterpret_cast<void**>(&s->h_ctls), sizeof(BatchCtl) * count),
          "pinned control blocks");
    s->ctl_cap = count;
  }
  std::vector<Pending> ps(count);
  const auto wall0 = std::chrono::steady_clock::now();
  reset_abort(s);
  uint64_t counter = s->counter, sum_ins = 0, sum_del = 0;
  const uint32_t T = s->opt.walk.step_cap;
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t b = first + i;
    Pending& p = ps[i];
    p.batch = b;
    p.wall0 = wall0;
    p.dctl = s->d_ctls + i;
    p.hctl = s->h_ctls + i;
    p.hdec = &s->h_counts[2];
    p.counter_base = counter;
    p.shard = true;
    if (b >= s->batch_cnt.size() || s->batch_cnt[b] == 0) continue;
    settle_upload(s, b);  // this batch's upload and kind counts only
    const uint64_t off = s->batch_off[b];
    p.dev = s->d_stream + off;
    p.host = uploaded_host(s, off);
    p.pos = uploaded_pos(s, off);
    p.pos_base = off;
    p.nb = static_cast<uint32_t>(s->batch_cnt[b]);
    p.n_ins = static_cast<uint32_t>(s->batch_ins[b]);
    p.n_del = static_cast<uint32_t>(s->batch_del[b]);
    const uint32_t sl_r = (p.n_ins + world - 1) / world, sl_m = (p.n_del + world - 1) / world;
    if (sl_r > s->px_slots_r || sl_m > s->px_slots_m) {
      check(cudaStreamSynchronize(s->stream), "peer range");  // drain what is enqueued
      fail(DYG_ERR_USAGE, "batch " + std::to_string(b) +
                              " exceeds the exchange area (dyg_shard_peer_create maxima)");
    }
    sum_ins += p.n_ins;
    sum_del += p.n_del;
    ensure_pools(s, sum_ins, sum_del);
    if (p.n_del > s->nd_cap ||
        (p.n_del > 0 && (s->b.side_id == nullptr || s->side_cap < s->G.pool_capacity())))
      check(cudaStreamSynchronize(s->stream), "buffer growth");
    ensure_batch(s, p.nb, p.n_del);
    if (p.n_del > 0) ensure_side_pool(s);
    auto enqueue = [&] {
      Pending q = p;
      phase_prepare(s, q);
      q.launches += launch_shard_range(s->b, rank, static_cast<int>(world), s->d_counts + 4, sl_r,
                                       sl_m, s->stream);
      phase_walk(s, q, false, 0, sl_r, 0, sl_m, /*fork_g=*/true);
      q.launches += launch_pack_peer(s->b, s->d_counts + 4, sl_r, sl_m, T, s->px, s->stream);
      q.launches += launch_unpack_peer(s->b, q.n_ins, q.n_del, sl_r, sl_m, T, s->px, s->stream);
      commit_enqueue(s, q, false);
      return q.launches;
    };
    prepare_bind(s, p);
    uint64_t key = session_fingerprint(s, 8);
    const uint64_t shape[] = {reinterpret_cast<uint64_t>(p.dev), reinterpret_cast<uint64_t>(p.dctl),
                              p.nb, p.n_ins, p.n_del, world, static_cast<uint64_t>(rank)};
    key = fnv(key, shape, sizeof shape);
    key = fnv(key, &s->px, sizeof s->px);
    p.launches = enqueue_captured(s, key, p.counter_base, enqueue);
    counter += p.nb;
  }
  check(cudaMemcpyAsync(s->h_ctls, s->d_ctls, sizeof(BatchCtl) * count, cudaMemcpyDeviceToHost,
                        s->stream), "ctl download");
  // Every batch has been enqueued: settle the rest of the upload (the host
  // waits while the GPU works), so later ranges take the one-graph path.
  settle_upload(s, ~0u);
  s->px_pending = std::move(ps);
  s->px_first = first;
}

void peer_range_end(dyg_session* s, dyg_batch_report* out) {
  std::vector<Pending> ps;
  ps.swap(s->px_pending);
  check(cudaStreamSynchronize(s->stream), "peer range");
  for (size_t i = 0; i < ps.size(); ++i) {
    if (ps[i].nb == 0) {
      empty_report(s, ps[i].batch, &out[i]);
      continue;
    }
    commit_finalize(s, ps[i], &out[i]);  // throws at the first failing batch
  }
}
}  // namespace

int dyg_shard_peer_range_begin(dyg_session* s, uint32_t first, uint32_t count) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    if (!s->px_bound) fail(DYG_ERR_USAGE, "no peer exchange bound: call dyg_shard_peer_bind");
    if (!s->have_stream) fail(DYG_ERR_USAGE, "no stream uploaded");
    if (count && static_cast<uint64_t>(first) + count > s->stream_batches && s->stream_batches > 0)
      fail(DYG_ERR_USAGE, "batch index out of range");
    check(cudaSetDevice(s->device), "set device");
    if (s->up_pending) {  // the stream is still landing: pipeline behind it
      peer_range_pipelined(s, first, count);
      return;
    }
    peer_range_begin(s, first, count);
  });
}

int dyg_shard_peer_range_end(dyg_session* s, dyg_batch_report* out, size_t cap, size_t* n_out) {
  return guarded([&] {
    if (s == nullptr) fail(DYG_ERR_USAGE, "null session");
    if (n_out) *n_out = 0;
    if (s->px_pending.empty()) return;
    if (out == nullptr || cap < s->px_pending.size()) {
      // still drain the range (the device work is enqueued)
      std::vector<dyg_batch_report> tmp(s->px_pending.size());
      const size_t n = tmp.size();
      check(cudaSetDevice(s->device), "set device");
      peer_range_end(s, tmp.data());
      if (out) std::memcpy(out, tmp.data(), sizeof(dyg_batch_report) * std::min(cap, n));
      if (n_out) *n_out = n;
      return;
    }
    const size_t n = s->px_pending.size();
    check(cudaSetDevice(s->device), "set device");
    peer_range_end(s, out);
    if (n_out) *n_out = n;
  });
}

// ---- generate_update_stream with device insertion sampling ---------------
int dyg_generate_stream(const dyg_csr* g, double insert_fraction, double delete_fraction,
                        uint32_t batches, uint64_t seed, int device, dyg_event* out,
                        size_t capacity, size_t* n_out, uint32_t* batch_count) {
  return guarded([&] {
    if (n_out == nullptr || batch_count == nullptr) fail(DYG_ERR_USAGE, "null argument");
    *n_out = 0;
    *batch_count = 0;
    check_csr(g, "graph");
    check(cudaSetDevice(device), "set device");
    std::vector<dyg_event> ev;
    uint32_t nb = 0;
    try {
      generate_stream_device(*g, insert_fraction, delete_fraction, batches, seed, ev, nb, nullptr);
    } catch (const GenError& e) {
      fail(e.code, e.message);
    }
    *n_out = ev.size();
    *batch_count = nb;
    if (out == nullptr || capacity < ev.size())
      fail(DYG_ERR_USAGE, "event buffer too small: " + std::to_string(ev.size()) + " events");
    std::memcpy(out, ev.data(), sizeof(dyg_event) * ev.size());
  });
}

// ---- stateless run_batch twin (walk.hpp:86-92) ----------------------------
int dyg_build_initial_sparsifier(const dyg_csr* g, double target_density, uint64_t seed,
                                 int device, uint64_t* row_ptr_out, uint32_t* ids_out,
                                 double* w_out) {
  return guarded([&] {
    if (row_ptr_out == nullptr || ids_out == nullptr || w_out == nullptr)
      fail(DYG_ERR_USAGE, "null argument");
    check_csr(g, "graph");
    if (target_density < 0.0) fail(DYG_ERR_USAGE, "target density must be nonnegative");
    if (g->n == 0) fail(DYG_ERR_DATA, "graph must be connected to build a sparsifier");
    check(cudaSetDevice(device), "set device");
    build_initial_sparsifier_device(g->n, g->row_ptr, g->ids, g->w, target_density, seed,
                                    row_ptr_out, ids_out, w_out);
  });
}

void dyg_condition_options_default(dyg_condition_options* out) {
  if (out) *out = condition_defaults();
}

int dyg_condition_number(const dyg_csr* g, const dyg_csr* h, const dyg_condition_options* options,
                         int device, dyg_condition_estimate* out) {
  return guarded([&] {
    if (out == nullptr) fail(DYG_ERR_USAGE, "null argument");
    const dyg_condition_options o = options ? *options : condition_defaults();
    *out = condition_number_impl(g, h, o, device);
  });
}

int dyg_calibrate_budget(const dyg_csr* g, const dyg_csr* h, double probe_fraction, double rho,
                         uint64_t seed, int device, double* budget) {
  return guarded([&] {
    if (budget == nullptr) fail(DYG_ERR_USAGE, "null argument");
    *budget = calibrate_impl(g, h, probe_fraction, rho, seed, device);
  });
}

namespace {
void export_owned(dyg_session* s, int which, OwnedCsr& o) {
  const uint64_t e = which == 0 ? s->g_edges : s->h_edges;
  o.rp.resize(s->n + 1ull);
  o.ids.resize(std::max<uint64_t>(2 * e, 1));
  o.w.resize(std::max<uint64_t>(2 * e, 1));
  check(cudaSetDevice(s->device), "set device");
  const uint64_t nnz = which == 0 ? s->G.export_rows(o.rp.data(), o.ids.data(), o.w.data(),
                                                     o.ids.size(), s->stream)
                                  : s->H.export_rows(o.rp.data(), o.ids.data(), o.w.data(),
                                                     o.ids.size(), s->stream);
  if (nnz > o.ids.size()) fail(DYG_ERR_DEVICE, "row export size mismatch");
  o.c = dyg_csr{s->n, 0, o.rp.data(), o.ids.data(), o.w.data()};
}
}  // namespace

int dyg_session_condition_number(dyg_session* s, const dyg_condition_options* options,
                                 dyg_condition_estimate* out) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || out == nullptr) fail(DYG_ERR_USAGE, "null argument");
    OwnedCsr g, h;
    export_owned(s, 0, g);
    export_owned(s, 1, h);
    const dyg_condition_options o = options ? *options : condition_defaults();
    *out = condition_number_impl(&g.c, &h.c, o, s->device);
  });
}

int dyg_session_calibrate_budget(dyg_session* s, double probe_fraction, double rho,
                                 double* budget) {
  return guarded([&] {
    require_settled(s);
    if (s == nullptr || budget == nullptr) fail(DYG_ERR_USAGE, "null argument");
    OwnedCsr g, h;
    export_owned(s, 0, g);
    export_owned(s, 1, h);
    *budget = calibrate_impl(&g.c, &h.c, probe_fraction, rho, s->opt.walk.global_seed, s->device);
  });
}

int dyg_pcg_solve(const dyg_csr* g, const dyg_csr* h, uint32_t factor_cap, const double* rhs,
                  double tolerance, uint32_t max_iterations, int device, double* x,
                  dyg_pcg_result* out, double* energy_trace, size_t energy_cap) {
  return guarded([&] {
    if (rhs == nullptr || x == nullptr || out == nullptr) fail(DYG_ERR_USAGE, "null argument");
    check_csr(g, "graph");
    if (h != nullptr) {
      check_csr(h, "preconditioner graph");
      if (h->n != g->n) fail(DYG_ERR_USAGE, "solver dimensions disagree");
      if (!csr_connected(h)) fail(DYG_ERR_DATA, "preconditioner graph is disconnected");
    }
    if (factor_cap == 0) factor_cap = 2000000;  // Preconditioner::kDefaultFactorCap
    if (dyg_device_count() == 0) fail(DYG_ERR_DEVICE, "no CUDA device visible");
    check(cudaSetDevice(device), "set device");
    cudaStream_t st;
    check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    std::vector<double> energy;
    PcgOutcome r;
    try {
      DevLapOwner lg(csr_view(g), st);
      DevLapOwner* lh = h ? new DevLapOwner(csr_view(h), st) : nullptr;
      check(cudaStreamSynchronize(st), "laplacian upload");
      // Factorized (exact) up to factor_cap, InnerCg at 1e-10 beyond (solver.cpp:17-23).
      const bool factorized = h && h->n <= factor_cap;
      HostCsrView hv{};
      if (h) hv = csr_view(h);
      try {
        r = pcg_device(lg.L, lh ? &lh->L : nullptr, h ? &hv : nullptr, factorized, rhs, tolerance,
                       max_iterations, 1e-10, x, energy_trace ? &energy : nullptr);
      } catch (...) {
        delete lh;
        throw;
      }
      delete lh;
    } catch (...) {
      cudaStreamDestroy(st);
      throw;
    }
    cudaStreamDestroy(st);
    out->iterations = r.iterations;
    out->converged = r.converged;
    out->relative_residual = r.relative_residual;
    out->inner_iterations = r.inner_iterations;
    const size_t ne = std::min(energy.size(), energy_cap);
    if (energy_trace && ne) std::memcpy(energy_trace, energy.data(), sizeof(double) * ne);
    out->energy_count = ne;
  });
}

int dyg_spectral_ordering_stats(uint64_t* hits, uint64_t* near_hits, uint64_t* misses) {
  return guarded([&] {
    if (hits == nullptr || near_hits == nullptr || misses == nullptr) fail(DYG_ERR_USAGE, "null argument");
    ordering_cache_stats(hits, near_hits, misses);
  });
}

int dyg_random_rhs(uint32_t n, uint64_t seed, double* out) {
  return guarded([&] {
    if (out == nullptr && n) fail(DYG_ERR_USAGE, "null argument");
    uint64_t state = hash_mix(seed + 0xB0C4ull);
    auto next_double = [&] {
      state += kGamma;
      return static_cast<double>(hash_mix(state) >> 11) * 0x1.0p-53;
    };
    for (uint32_t i = 0; i < n; i += 2) {  // Box-Muller on the deterministic stream
      const double u1 = std::max(next_double(), 1e-300);
      const double u2 = next_double();
      const double radius = std::sqrt(-2.0 * std::log(u1));
      out[i] = radius * std::cos(2.0 * M_PI * u2);
      if (i + 1 < n) out[i + 1] = radius * std::sin(2.0 * M_PI * u2);
    }
    double sum = 0.0;
    for (uint32_t i = 0; i < n; ++i) sum += out[i];
    const double mean = n ? sum / n : 0.0;
    for (uint32_t i = 0; i < n; ++i) out[i] -= mean;
  });
}

int dyg_run_batch(const dyg_csr* g, const dyg_walk_query* queries, size_t n_queries,
                  const dyg_walk_config* cfg, dyg_walk_result* out, uint32_t* path_buf,
                  int device) {
  return guarded([&] {
    if (cfg == nullptr || (n_queries && (queries == nullptr || out == nullptr)))
      fail(DYG_ERR_USAGE, "null argument");
    check_csr(g, "graph");
    // single_walk's usage checks (walk.cpp:43-48), first failing query.
    for (size_t i = 0; i < n_queries; ++i) {
      const dyg_walk_query& q = queries[i];
      if (q.p == q.q) fail(DYG_ERR_USAGE, "walk endpoints must differ");
      if (q.p >= g->n) {
        char buf[128];
        std::snprintf(buf, sizeof buf, "vertex id %u out of range (n = %u)", q.p, g->n);
        fail(DYG_ERR_USAGE, buf);
      }
      if (g->row_ptr[q.p + 1] == g->row_ptr[q.p]) fail(DYG_ERR_USAGE, "walk started at an isolated vertex");
    }
    if (n_queries == 0) return;
    if (dyg_device_count() == 0) fail(DYG_ERR_DEVICE, "no CUDA device visible");
    check(cudaSetDevice(device), "set device");
    cudaStream_t st;
    check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    std::vector<ReachQuery> rq;
    std::vector<MinQuery> mq;
    std::vector<size_t> ri, mi;
    for (size_t i = 0; i < n_queries; ++i) {
      const dyg_walk_query& q = queries[i];
      if (q.kind == 0) {
        rq.push_back(ReachQuery{q.p, q.q, q.w_pq, query_seed(cfg->global_seed, q.update_id)});
        ri.push_back(i);
      } else {
        mq.push_back(MinQuery{q.p, q.q, query_seed(cfg->global_seed, q.update_id)});
        mi.push_back(i);
      }
    }
    const WalkParams P = make_walk_params(cfg->distortion_threshold, cfg->step_cap,
                                          cfg->walker_count, cfg->global_seed);
    const uint64_t T1 = static_cast<uint64_t>(cfg->step_cap) + 1;
    WalkCounters* ctr = nullptr;
    uint32_t* d_n = nullptr;
    unsigned int* d_work = nullptr;
    dev_alloc(&d_work, 1, "work counter");
    dev_alloc(&ctr, 2, "counters");
    dev_alloc(&d_n, 2, "counts");
    const uint32_t counts[2] = {static_cast<uint32_t>(rq.size()), static_cast<uint32_t>(mq.size())};
    check(cudaMemcpy(d_n, counts, sizeof counts, cudaMemcpyHostToDevice), "counts");
    check(cudaMemset(ctr, 0, 2 * sizeof(WalkCounters)), "counters");
    if (!rq.empty()) {
      GraphStore<kCapH> gh;
      gh.upload(g->n, g->row_ptr, g->ids, g->w, st);
      ReachQuery* d_q = nullptr;
      ReachOut ro{};
      dev_alloc(&d_q, rq.size(), "queries");
      dev_alloc(&ro.reached, rq.size(), "out");
      dev_alloc(&ro.steps, rq.size(), "out");
      dev_alloc(&ro.best_bits, rq.size(), "out");
      check(cudaMemcpy(d_q, rq.data(), sizeof(ReachQuery) * rq.size(), cudaMemcpyHostToDevice), "q");
      launch_reach(gh.view(), d_q, d_n, counts[0], P, ro, ctr, d_work, st);
      check(cudaGetLastError(), "reach launch");
      check(cudaStreamSynchronize(st), "reach");
      std::vector<uint32_t> reached(rq.size());
      std::vector<unsigned long long> steps(rq.size()), best(rq.size());
      check(cudaMemcpy(reached.data(), ro.reached, 4 * rq.size(), cudaMemcpyDeviceToHost), "out");
      check(cudaMemcpy(steps.data(), ro.steps, 8 * rq.size(), cudaMemcpyDeviceToHost), "out");
      check(cudaMemcpy(best.data(), ro.best_bits, 8 * rq.size(), cudaMemcpyDeviceToHost), "out");
      for (size_t j = 0; j < rq.size(); ++j) {
        dyg_walk_result& r = out[ri[j]];
        r = dyg_walk_result{};
        r.reached = reached[j];
        r.steps_used = steps[j];
        if (reached[j]) std::memcpy(&r.best_estimate, &best[j], 8);
      }
      cudaFree(d_q);
      cudaFree(ro.reached);
      cudaFree(ro.steps);
      cudaFree(ro.best_bits);
    }
    if (!mq.empty()) {
      GraphStore<kCapG> gg;
      gg.upload(g->n, g->row_ptr, g->ids, g->w, st);
      const size_t nm = mq.size();
      const uint64_t sw = cfg->walker_count;
      MinQuery* d_q = nullptr;
      MinOut mo{};
      MinScratch sc{};
      dev_alloc(&d_q, nm, "queries");
      dev_alloc(&mo.has_path, nm, "out");
      dev_alloc(&mo.path_len, nm, "out");
      dev_alloc(&mo.steps, nm, "out");
      dev_alloc(&mo.resistance, nm, "out");
      dev_alloc(&mo.paths, nm * T1, "out");
      // Entries past a path's length are never written: zero them so the
      // whole-buffer read-back below copies defined bytes (initcheck).
      check(cudaMemset(mo.paths, 0, sizeof(uint32_t) * nm * T1), "out");
      dev_alloc(&sc.acc, nm * sw, "scratch");
      dev_alloc(&sc.term, nm * sw, "scratch");
      dev_alloc(&sc.steps, nm * sw, "scratch");
      dev_alloc(&sc.paths, nm * sw * trace_stride(cfg->step_cap), "scratch");
      dev_alloc(&sc.rvals, nm * T1, "scratch");
      check(cudaMemcpy(d_q, mq.data(), sizeof(MinQuery) * nm, cudaMemcpyHostToDevice), "q");
      launch_minpath(gg.view(), d_q, d_n + 1, counts[1], P, sc, mo, ctr + 1, d_work, st);
      check(cudaGetLastError(), "minpath launch");
      check(cudaStreamSynchronize(st), "minpath");
      std::vector<uint32_t> has(nm), len(nm), paths(nm * T1);
      std::vector<unsigned long long> steps(nm);
      std::vector<double> res(nm);
      check(cudaMemcpy(has.data(), mo.has_path, 4 * nm, cudaMemcpyDeviceToHost), "out");
      check(cudaMemcpy(len.data(), mo.path_len, 4 * nm, cudaMemcpyDeviceToHost), "out");
      check(cudaMemcpy(steps.data(), mo.steps, 8 * nm, cudaMemcpyDeviceToHost), "out");
      check(cudaMemcpy(res.data(), mo.resistance, 8 * nm, cudaMemcpyDeviceToHost), "out");
      check(cudaMemcpy(paths.data(), mo.paths, 4 * nm * T1, cudaMemcpyDeviceToHost), "out");
      for (size_t j = 0; j < nm; ++j) {
        dyg_walk_result& r = out[mi[j]];
        r = dyg_walk_result{};
        r.reached = has[j];
        r.steps_used = steps[j];
        if (has[j]) {
          r.path_len = len[j];
          r.resistance = res[j];
          if (path_buf)
            std::memcpy(path_buf + mi[j] * T1, paths.data() + j * T1, 4ull * len[j]);
        }
      }
      cudaFree(d_q);
      cudaFree(mo.has_path);
      cudaFree(mo.path_len);
      cudaFree(mo.steps);
      cudaFree(mo.resistance);
      cudaFree(mo.paths);
      cudaFree(sc.acc);
      cudaFree(sc.term);
      cudaFree(sc.steps);
      cudaFree(sc.paths);
      cudaFree(sc.rvals);
    }
    cudaFree(ctr);
    cudaFree(d_n);
    cudaFree(d_work);
    cudaStreamDestroy(st);
  });
}

}  // extern "C"
