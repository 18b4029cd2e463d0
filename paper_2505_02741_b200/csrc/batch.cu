// batch.cu -- validation, walk shadow, query build and the commit engine of
// one deferred batch. See batch.cuh for the kernel map and the dependency
// round scheme.
#include <cooperative_groups.h>


#include <map>
#include <mutex>
#include <unordered_map>

#include "batch.cuh"
#include "graph_store.cuh"

namespace cg = cooperative_groups;

namespace dyg {

namespace {

__device__ __forceinline__ bool batch_aborted(const BatchCtl* ctl) {
  return *reinterpret_cast<const volatile unsigned long long*>(&ctl->val_err) != ~0ull;
}

// sparsifier.cpp:321-337 validate_event_shape; the lowest failing event
// wins (the reference validates in stream order before walking).
__global__ void k_validate(const DevEvent* __restrict__ ev, uint32_t nb, uint32_t n,
                           BatchCtl* ctl, const unsigned int* __restrict__ abort_flag) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  if (*abort_flag) {  // an earlier batch of this range failed: do nothing
    if (k == 0) atomicMin(&ctl->val_err, static_cast<unsigned long long>(kErrAborted));
    return;
  }
  const DevEvent e = ev[k];
  uint32_t code = 0;
  if (e.u >= n || e.v >= n) {
    code = kErrRange;
  } else if (e.u == e.v) {
    code = kErrSelfLoop;
  } else if (e.kind == 0 && (!(e.weight > 0.0) || !isfinite(e.weight))) {
    code = kErrWeight;
  }
  if (code) atomicMin(&ctl->val_err, (static_cast<unsigned long long>(k) << 8) | code);
}

// Per-thread accumulators of one round-engine launch: report counters and
// |E| deltas are summed locally and flushed once per warp at the end
// (one atomic per warp instead of several same-address atomics per event).
struct Acc {
  unsigned long long r[kReportFields];
  long long dg, dh;
};

// Commit start stamp (first block of the first commit kernel wins).
__device__ __forceinline__ void stamp_commit_start(BatchCtl* ctl) {
  if (threadIdx.x == 0) atomicMin(&ctl->t_commit0, global_ns());
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, off);
  return x;
}
__device__ __forceinline__ unsigned long long warp_max(unsigned long long x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, x, off);
    x = o > x ? o : x;
  }
  return x;
}
// Report counters and |E| deltas of a whole block: warp totals, then one
// atomic per field and BLOCK (per-warp atomics on these few addresses
// serialise in L2: ~5k warps x 6 fields per deletion commit). Every thread
// of the block must call it.
__device__ __forceinline__ void flush_acc(const Acc& a, BatchCtl* ctl, unsigned long long* g_edges,
                                          unsigned long long* h_edges) {
  constexpr int kF = kReportFields + 2;
  __shared__ unsigned long long s_acc[kF][32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int f = 0; f < kReportFields; ++f) {
    const unsigned long long v = f == kMaxEventSteps ? warp_max(a.r[f]) : warp_sum(a.r[f]);
    if (lane == 0) s_acc[f][wid] = v;
  }
  const unsigned long long dg = warp_sum(static_cast<unsigned long long>(a.dg));
  const unsigned long long dh = warp_sum(static_cast<unsigned long long>(a.dh));
  if (lane == 0) {
    s_acc[kReportFields][wid] = dg;
    s_acc[kReportFields + 1][wid] = dh;
  }
  __syncthreads();
  if (threadIdx.x < static_cast<uint32_t>(kF)) {
    const int f = static_cast<int>(threadIdx.x);
    unsigned long long v = 0;
    for (uint32_t w = 0; w < nw; ++w) {
      const unsigned long long x = s_acc[f][w];
      v = f == kMaxEventSteps ? (x > v ? x : v) : v + x;
    }
    if (v) {
      if (f == kMaxEventSteps) atomicMax(&ctl->report[f], v);
      else if (f < kReportFields) atomicAdd(&ctl->report[f], v);
      else if (f == kReportFields && g_edges) atomicAdd(g_edges, v);
      else if (f == kReportFields + 1 && h_edges) atomicAdd(h_edges, v);
    }
  }
  __syncthreads();  // s_acc may be reused by a later call
}

// Insertion fast path. In an insertion-only batch where every key is new to
// G (checked in k_prep) and no key repeats within the batch (k_fp_check),
// event k's whole commit (:473-488 with :220-241) is: push_back(u: v, w) and
// push_back(v: u, w) into G, and -- when kept -- the same two appends into H
// with weight G.w(u,v) = w. H lacks the key because H is a subgraph of G.
// Rows only receive appends, in event order. Each append record r = 2k +
// side (row u or v of event k) is pushed onto its row's lock-free list by
// k_prep (one atomic exchange per record and graph; the lists depend on the
// events only, not on the walks). The list head owns the row: a sole record
// (the vast majority) appends directly, a head with followers applies the
// row's records in increasing r, i.e. event order. G's appends do not depend
// on the walks (which read H alone), so k_fp_check + k_fp_write_g run on a
// second stream CONCURRENTLY with the reach walk, filling the SMs its tail
// leaves idle; the commit launch first appends the kept records to H (fp_write_h_pass) and
// does the per-event accounting. Any violated precondition sets not_simple
// BEFORE anything is written and the round engine (k_rounds) commits the
// batch instead. The list heads are left empty for the next batch.
__device__ __forceinline__ uint32_t rec_row(const DevEvent* ev, uint32_t rec) {
  const DevEvent& e = ev[rec >> 1];
  return (rec & 1) ? e.v : e.u;
}
__device__ __forceinline__ uint32_t other_end(const DevEvent* ev, uint32_t rec) {
  const DevEvent& e = ev[rec >> 1];
  return (rec & 1) ? e.u : e.v;
}

// A key repeated inside the batch shows up as a repeated neighbour on a
// G row with several records; its list head checks.
__global__ void k_fp_check(const DevEvent* __restrict__ ev, uint32_t n, BatchDev b) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n || batch_aborted(b.ctl) || b.ctl->not_simple) return;
  const uint32_t row = rec_row(ev, r);
  const uint32_t* next = b.fp_next[0];
  if (b.fp_head[0][row] != r || next[r] == kNoSlot) return;
  for (uint32_t x = r; x != kNoSlot; x = next[x])
    for (uint32_t y = next[x]; y != kNoSlot; y = next[y])
      if (other_end(ev, x) == other_end(ev, y)) b.ctl->not_simple = 1;
}

// Record r's row on one graph: the list head appends the row's records that
// pass `take` -- itself alone, or all of them in increasing r by repeated
// minimum selection over the short list -- and empties the list head.
template <int C, class Take>
__device__ __forceinline__ bool fp_apply(const DevGraph<C>& g, const DevEvent* ev, uint32_t* head,
                                         const uint32_t* next, uint32_t r, bool write, Take take,
                                         bool reset) {
  const uint32_t row = rec_row(ev, r);
  if (row >= g.n) return true;  // an invalid event (the batch fails validation): never linked
  // The row's slab is needed by the head's append: request it alongside the
  // list lookups.
  if (write) asm volatile("prefetch.global.L2 [%0];" ::"l"(g.slab + row));
  const uint32_t h = head[row];
  const uint32_t nx = next[r];
  if (h != r) return true;
  bool ok = true;
  if (write) {
    if (nx == kNoSlot) {
      if (take(r)) ok = row_push(g, row, other_end(ev, r), ev[r >> 1].weight);
    } else {
      uint32_t last = 0;
      for (bool first = true; ok; first = false) {
        uint32_t best = kNoSlot;
        for (uint32_t x = r; x != kNoSlot; x = next[x])
          if ((first || x > last) && x < best) best = x;
        if (best == kNoSlot) break;
        if (take(best)) ok = row_push(g, row, other_end(ev, best), ev[best >> 1].weight);
        last = best;
      }
    }
  }
  if (reset) head[row] = kNoSlot;
  return ok;
}

// commit_insertion's keep decision (sparsifier.cpp:228-233) for event k.
__device__ __forceinline__ bool event_kept(const BatchDev& b, const WalkOpts& o, uint32_t k,
                                           bool& have, unsigned long long& steps) {
  const uint32_t s = b.slot[k];
  have = s != kNoSlot;
  const bool reached = have && b.rout.reached[s] != 0;
  steps = have ? b.rout.steps[s] : 0ull;
  return !o.freeze && !(o.K != 0.0 && have && reached);
}

// Batch epilogue: fast-path report, |E| and pool tops for the host, and the
// device abort flag that stops the later batches of a range after an error.
__device__ void batch_finish(const DevGraph<kCapG>& G, const DevGraph<kCapH>& H,
                             const BatchDev& b) {
  BatchCtl* ctl = b.ctl;
  if (ctl->fast && !ctl->not_simple && ctl->val_err == ~0ull) {
    for (int f = 0; f < kReportFields; ++f) ctl->report[f] = ctl->fp_report[f];
    G.edges[0] += ctl->fp_report[kInsSeen];
    H.edges[0] += ctl->fp_report[kInsKept];
  }
  if (ctl->val_err != ~0ull || ctl->commit_err != ~0ull ||
      (ctl->use_absent_limit && ctl->first_absent != 0xFFFFFFFFu))
    *b.abort_flag = 1;
  ctl->g_pool_top = *G.pool_top;
  ctl->g_edges = *G.edges;
  ctl->h_pool_top = *H.pool_top;
  ctl->h_edges = *H.edges;
  ctl->t_batch1 = global_ns();
}


// Undo the in-place walk shadow (rows saved by k_sh_apply / k_save_rows).
__device__ void restore_rows(const DevGraph<kCapG>& G, const BatchDev& b, uint32_t tid,
                             uint32_t nth) {
  const uint32_t n = b.ctl->n_saved;
  for (uint32_t idx = tid; idx < n; idx += nth) {
    const uint32_t row = b.saved_rows[idx];
    const Slab<kCapG> sl = b.side_slab[idx];
    G.slab[row] = sl;
    if (sl.ext != kInline) {
      const unsigned long long off = b.side_off[idx];
      for (uint32_t i = 0; i < sl.deg; ++i) {
        G.pool_id[sl.ext + i] = b.side_id[off + i];
        G.pool_w[sl.ext + i] = b.side_w[off + i];
      }
    }
  }
}

// G appends, one thread per record (runs concurrently with the reach walk).
__global__ void k_fp_write_g(DevGraph<kCapG> G, const DevEvent* __restrict__ ev, uint32_t n,
                             BatchDev b) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  // An invalid batch or a violated precondition: only empty the lists.
  const bool write = !batch_aborted(b.ctl) && !b.ctl->not_simple;
  // The H pass (fp_write_h_pass, after the walk) reads the same lists and
  // empties them.
  if (!fp_apply(G, ev, b.fp_head[0], b.fp_next[0], r, write, [](uint32_t) { return true; },
                /*reset=*/false))
    atomicMin(&b.ctl->commit_err, static_cast<unsigned long long>(kErrPool));
}

// After the reach walk: H appends of the kept records and each event's
// decision and report counters, one thread per EVENT: its keep decision is
// read once for both records, and the two rows' list heads, slabs and appends
// are independent requests in flight together.
// The H pass over events k0, k0 + kstride, ... (every thread of the block
// must call it: the block totals end with a barrier).
__device__ void fp_write_h_pass(const DevGraph<kCapH>& H, const DevEvent* __restrict__ ev,
                                uint32_t nb, const WalkOpts& o, const BatchDev& b, uint32_t k0,
                                uint32_t kstride) {
  stamp_commit_start(b.ctl);
  unsigned long long kept_acc = 0, pruned_acc = 0, steps_sum = 0, steps_max = 0;
  for (uint32_t k = k0; k < nb; k += kstride) {
  const bool write = !batch_aborted(b.ctl) && !b.ctl->not_simple;
  unsigned long long kept_n = 0, pruned_n = 0, steps = 0;
  {
    const DevEvent e = ev[k];
    uint32_t* head = b.fp_head[0];  // the lists k_fp_write_g walked
    const uint32_t* next = b.fp_next[0];
    const uint32_t rows[2] = {e.u, e.v};
    if (write) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(H.slab + rows[0]));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(H.slab + rows[1]));
    }
    // An out-of-range endpoint fails validation (write is then false) and
    // was never linked: no list to read.
    const uint32_t h[2] = {e.u < H.n ? head[rows[0]] : kNoSlot,
                           e.v < H.n ? head[rows[1]] : kNoSlot};
    bool kept = false;
    if (write) {
      bool have;
      kept = event_kept(b, o, k, have, steps);
      b.dec[k] = kept ? 0u : 1u;
      (kept ? kept_n : pruned_n) = 1;
    }
    auto take = [&](uint32_t x) {
      if ((x >> 1) == k) return kept;
      bool have;
      unsigned long long st;
      return event_kept(b, o, x >> 1, have, st);
    };
    bool ok = true;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const uint32_t r = 2 * k + side;
      if (h[side] != r) continue;  // not the list head of its row
      const uint32_t row = rows[side];
      if (write) {
        const uint32_t nx = next[r];
        if (nx == kNoSlot) {
          if (kept) ok = ok && row_push(H, row, rows[side ^ 1], e.weight);
        } else {  // the row's records in increasing r
          uint32_t last = 0;
          for (bool first = true; ok; first = false) {
            uint32_t best = kNoSlot;
            for (uint32_t x = r; x != kNoSlot; x = next[x])
              if ((first || x > last) && x < best) best = x;
            if (best == kNoSlot) break;
            if (take(best)) ok = row_push(H, row, other_end(ev, best), ev[best >> 1].weight);
            last = best;
          }
        }
      }
      head[row] = kNoSlot;
    }
    if (!ok) atomicMin(&b.ctl->commit_err, static_cast<unsigned long long>(kErrPool));
  }
  kept_acc += kept_n;
  pruned_acc += pruned_n;
  steps_sum += steps;
  steps_max = steps_max > steps ? steps_max : steps;
  }
  // Block totals, then one atomic per field and block: per-warp atomics on
  // these five addresses serialise in L2 (~18k per C5 batch).
  __shared__ unsigned long long s_red[4][8];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  kept_acc = warp_sum(kept_acc);
  pruned_acc = warp_sum(pruned_acc);
  steps_sum = warp_sum(steps_sum);
  steps_max = warp_max(steps_max);
  if (lane == 0) {
    s_red[0][wid] = kept_acc;
    s_red[1][wid] = pruned_acc;
    s_red[2][wid] = steps_sum;
    s_red[3][wid] = steps_max;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long k = 0, p = 0, st = 0, m = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      k += s_red[0][w];
      p += s_red[1][w];
      st += s_red[2][w];
      m = m > s_red[3][w] ? m : s_red[3][w];
    }
    if (k | p) {
      atomicAdd(&b.ctl->fp_report[kInsSeen], k + p);
      atomicAdd(&b.ctl->fp_report[kInsKept], k);
      atomicAdd(&b.ctl->fp_report[kInsPruned], p);
      atomicAdd(&b.ctl->fp_report[kWalkerSteps], st);
      atomicMax(&b.ctl->fp_report[kMaxEventSteps], m);
    }
  }
}

// The round engine. Op provides for_rows(k, f) (every row event k reads or
// writes, possibly with repeats) and apply(k, acc) -> error code. For the
// commit (Op::kCommit) the launch also runs the batch epilogue; a batch the
// insertion fast path committed goes straight to it.
template <class Op>
__global__ void __launch_bounds__(256) k_rounds(Op op, uint32_t nev, BatchDev b) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t tid = static_cast<uint32_t>(grid.thread_rank());
  const uint32_t nth = static_cast<uint32_t>(grid.size());
  volatile BatchCtl* ctl = b.ctl;
  if constexpr (Op::kCommit) {
    stamp_commit_start(b.ctl);
    if (op.fp_h) {
      // The insertion fast path's H appends (fp_write_h_pass) inside this
      // launch instead of a kernel of their own. When they commit the batch
      // (the uniform condition below), the last block past them runs the
      // epilogue -- no grid barrier; otherwise the rounds follow a barrier.
      fp_write_h_pass(op.H, op.ev, nev, op.o, b, tid, nth);
      if (ctl->val_err == ~0ull && ctl->fast && !ctl->not_simple) {
        __shared__ bool s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          s_last = atomicAdd(&b.ctl->fl_blocks_done, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last && threadIdx.x == 0) {
          __threadfence();
          ctl->fl_t[0] = global_ns();  // (timeline only)
          batch_finish(op.G, op.H, b);
        }
        return;
      }
      grid.sync();
    }
  }
  if (ctl->val_err != ~0ull) {  // uniform: nothing below ran yet
    if constexpr (Op::kCommit) {
      if (tid == 0) batch_finish(op.G, op.H, b);
    }
    return;
  }
  if constexpr (Op::kCommit) {
    if (ctl->fast && !ctl->not_simple) {  // k_fp_write committed the batch
      if (tid == 0) ctl->fl_t[0] = global_ns();  // (timeline only)
      if (tid == 0) batch_finish(op.G, op.H, b);
      return;
    }
  }
  Acc acc{};
  unsigned long long round = *b.round_ctr;
  uint32_t r = 0;
  for (;; ++r) {
    ++round;
    const uint32_t lim = op.limit();
    if (tid == 0) ctl->remaining[(r + 1) % 3] = 0;
    for (uint32_t k = tid; k < nev; k += nth) {
      if (k >= lim || b.state[k] != 0) continue;
      const unsigned long long key = (round << 32) | (0xFFFFFFFFull - k);
      op.for_rows(k, [&](uint32_t row) { atomicMax(b.locks + row, key); });
      op.prefetch(k);
    }
    grid.sync();
    for (uint32_t k = tid; k < nev; k += nth) {
      if (k >= lim || b.state[k] != 0) continue;
      const unsigned long long key = (round << 32) | (0xFFFFFFFFull - k);
      bool ready = true;
      op.for_rows(k, [&](uint32_t row) {
        if (ready && *reinterpret_cast<volatile unsigned long long*>(b.locks + row) != key)
          ready = false;
      });
      if (ready) {
        const uint32_t e = op.apply(k, acc);
        b.state[k] = e ? 2 : 1;
        if (e) atomicMin(&b.ctl->commit_err, (static_cast<unsigned long long>(k) << 8) | e);
      } else {
        atomicAdd(&b.ctl->remaining[r % 3], 1u);
      }
    }
    grid.sync();
    if (ctl->remaining[r % 3] == 0) break;
  }
  op.flush(acc);
  if (tid == 0) {
    *b.round_ctr = round;
    ctl->rounds = ctl->rounds + r + 1;
  }
  if constexpr (Op::kCommit) {
    grid.sync();
    if (tid == 0) batch_finish(op.G, op.H, b);
  }
}

// Warp-per-event rounds for batches with deletions: the lanes of a warp
// reserve an event's rows (path vertices) in parallel and apply it together
// (path recovery is parallel over path edges, CommitOp::apply_warp). Same
// round protocol as k_rounds. Shared by k_rounds_warp (mixed batches) and
// k_del_flow (its fallback when the record buffer overflows).
template <class Op>
__device__ void rounds_warp_loop(const Op& op, uint32_t nev, const BatchDev& b,
                                 cg::grid_group& grid) {
  const uint32_t tid = static_cast<uint32_t>(grid.thread_rank());
  const uint32_t lane = tid & 31;
  const uint32_t wid = tid >> 5;
  const uint32_t nw = static_cast<uint32_t>(grid.size()) >> 5;
  volatile BatchCtl* ctl = b.ctl;
  Acc acc{};
  unsigned long long round = *b.round_ctr;
  uint32_t r = 0;
  for (;; ++r) {
    ++round;
    const uint32_t lim = op.limit();
    if (tid == 0) ctl->remaining[(r + 1) % 3] = 0;
    for (uint32_t k = wid; k < nev; k += nw) {
      if (k >= lim || b.state[k] != 0) continue;
      const unsigned long long key = (round << 32) | (0xFFFFFFFFull - k);
      op.for_rows_warp(k, lane, [&](uint32_t row) { atomicMax(b.locks + row, key); });
    }
    grid.sync();
    for (uint32_t k = wid; k < nev; k += nw) {
      if (k >= lim || b.state[k] != 0) continue;
      const unsigned long long key = (round << 32) | (0xFFFFFFFFull - k);
      bool ready = true;
      op.for_rows_warp(k, lane, [&](uint32_t row) {
        if (ready && *reinterpret_cast<volatile unsigned long long*>(b.locks + row) != key)
          ready = false;
      });
      ready = __all_sync(0xFFFFFFFFu, ready);
      if (ready) {
        const uint32_t e = op.apply_warp(k, lane, acc);
        if (lane == 0) {
          b.state[k] = e ? 2 : 1;
          if (e) atomicMin(&b.ctl->commit_err, (static_cast<unsigned long long>(k) << 8) | e);
        }
      } else if (lane == 0) {
        atomicAdd(&b.ctl->remaining[r % 3], 1u);
      }
      __syncwarp();
    }
    grid.sync();
    if (ctl->remaining[r % 3] == 0) break;
  }
  op.flush(acc);
  if (tid == 0) {
    *b.round_ctr = round;
    ctl->rounds = ctl->rounds + r + 1;
  }
}

// Commit of a batch with deletions by rounds: undo the walk shadow, the
// rounds, the epilogue -- one cooperative launch.
template <class Op>
__global__ void __launch_bounds__(256) k_rounds_warp(Op op, uint32_t nev, BatchDev b) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t tid = static_cast<uint32_t>(grid.thread_rank());
  volatile BatchCtl* ctl = b.ctl;
  stamp_commit_start(b.ctl);
  if (ctl->val_err == ~0ull) {
    restore_rows(op.G, b, tid, static_cast<uint32_t>(grid.size()));
    grid.sync();
    rounds_warp_loop(op, nev, b, grid);
    grid.sync();
  }
  if (tid == 0) batch_finish(op.G, op.H, b);
}

// Walk shadow (sparsifier.cpp:416-423): apply the batch's deletions to the
// copy of G in event order, skipping absent edges. first_absent records the
// lowest deletion that found no edge: in a deletion-only batch that is
// exactly the first event whose graph_.delete_edge throws (:491).
struct ShadowOp {
  static constexpr bool kCommit = false;
  DevGraph<kCapG> S;
  const DevEvent* ev;
  BatchCtl* ctl;
  __device__ uint32_t limit() const { return 0xFFFFFFFFu; }
  __device__ void prefetch(uint32_t) const {}
  template <class F>
  __device__ void for_rows(uint32_t k, F&& f) const {
    const DevEvent& e = ev[k];
    if (e.kind == 1) {
      f(e.u);
      f(e.v);
    }
  }
  __device__ void flush(const Acc& a) const { flush_acc(a, ctl, nullptr, nullptr); }
  __device__ uint32_t apply(uint32_t k, Acc& acc) const {
    const DevEvent e = ev[k];
    if (e.kind != 1) return 0;
    if (has_edge(S, e.u, e.v)) {
      delete_edge(S, e.u, e.v, acc.dg);
    } else {
      atomicMin(&ctl->first_absent, k);
    }
    return 0;
  }
};

// sparsifier.cpp:207-216 set_edge_weight.
__device__ __forceinline__ bool set_edge_weight(const DevGraph<kCapH>& h, uint32_t u, uint32_t v,
                                                double target, long long& dh) {
  const double current = edge_weight(h, u, v);
  if (target > current) {
    return insert_edge(h, u, v, __dsub_rn(target, current), dh) >= 0;
  } else if (target < current) {
    delete_edge(h, u, v, dh);
    return insert_edge(h, u, v, target, dh) >= 0;
  }
  return true;
}

// Max-weight G neighbour of x (tie -> lowest id) ignoring `skip`
// (sparsifier.cpp:270-276); kNoVertex when none.
__device__ __forceinline__ uint32_t best_neighbor(const DevGraph<kCapG>& g, uint32_t x,
                                                  uint32_t skip, double* wout) {
  const RowRef<kCapG> r = row(g, x);
  const uint32_t d = r.deg();
  uint32_t best = kNoVertex;
  double bw = 0.0;
  for (uint32_t i = 0; i < d; ++i) {
    const uint32_t id = r.id(i);
    if (id == skip) continue;
    const double w = r.w(i);
    if (best == kNoVertex || w > bw || (w == bw && id < best)) {
      best = id;
      bw = w;
    }
  }
  if (wout) *wout = bw;
  return best;
}

// The sequential commit of sparsifier.cpp:466-533, one event per apply().
struct CommitOp {
  static constexpr bool kCommit = true;
  DevGraph<kCapG> G;
  DevGraph<kCapH> H;
  const DevEvent* ev;
  const uint32_t* slot;
  ReachOut rout;
  MinOut mout;
  MinScratch mscratch;
  uint32_t* dec;
  BatchCtl* ctl;
  WalkOpts o;
  // Keep-shadow deletion commit (k_del_flow, deletion-only batch without an
  // absent deletion): G stays the walk shadow -- which IS the final G, the
  // batch's deletions applied in event order -- so the commit neither
  // restores nor re-deletes G. What a local fallback must read of LIVE G at
  // event k (the batch-start row minus the row's deletions up to k) comes
  // from the saved batch-start rows and the shadow's per-row deletion lists.
  int keep = 0;
  int fp_h = 0;  // insertion fast path: the H pass runs at the start of the commit launch
  int promo_pre = 0;  // k_prep<del> stored "edge in batch-start H" in fl_promo bit 1
  const uint32_t* save_idx = nullptr;     // vertex -> saved batch-start row
  const Slab<kCapG>* side_slab = nullptr;
  const unsigned long long* side_off = nullptr;
  const uint32_t* side_id = nullptr;
  const double* side_w = nullptr;
  const uint32_t* sh_head = nullptr;      // per-row deletion records r = 2k + side
  const uint32_t* sh_next = nullptr;

  // Entry i of x's batch-start row (keep mode; x is a deletion endpoint).
  __device__ uint32_t start_deg(uint32_t x) const { return side_slab[save_idx[x]].deg; }
  __device__ void start_entry(uint32_t x, uint32_t i, uint32_t& id, double& w) const {
    const uint32_t idx = save_idx[x];
    const Slab<kCapG>& sl = side_slab[idx];
    if (sl.ext == kInline) {
      id = sl.id[i];
      w = sl.w[i];
    } else {
      id = side_id[side_off[idx] + i];
      w = side_w[side_off[idx] + i];
    }
  }
  // Was (x, y) deleted by an event <= k of this batch?
  __device__ bool deleted_by(uint32_t x, uint32_t y, uint32_t k) const {
    for (uint32_t r = sh_head[x]; r != kNoSlot; r = sh_next[r]) {
      if ((r >> 1) > k) continue;
      const DevEvent& e = ev[r >> 1];
      if (((r & 1) ? e.u : e.v) == y) return true;
    }
    return false;
  }
  // run_local_fallback's view of x at event k (sparsifier.cpp:264-280): the
  // live degree and the max-weight live neighbour (ties: lowest id).
  __device__ uint32_t live_best(uint32_t x, uint32_t k, uint32_t& deg, double& bw) const {
    const uint32_t d = start_deg(x);
    uint32_t best = kNoVertex;
    deg = 0;
    bw = 0.0;
    for (uint32_t i = 0; i < d; ++i) {
      uint32_t id;
      double w;
      start_entry(x, i, id, w);
      if (deleted_by(x, id, k)) continue;
      ++deg;
      if (best == kNoVertex || w > bw || (w == bw && id < best)) {
        best = id;
        bw = w;
      }
    }
    return best;
  }
  // Keep mode: an event that can neither recover a path nor fall back
  // (its edge is not in batch-start H -- promo bit 1 -- and no earlier
  // fallback can put it there -- promo bit 0) only deletes from G, which the
  // shadow already did.
  __device__ bool flow_simple(uint32_t k, const uint8_t* promo, bool keep_g) const {
    return keep_g && !o.freeze && promo[k] == 0;
  }

  // Events at or past the first failing one never commit (the reference
  // stops there, :525-529). In a deletion-only batch the shadow pass already
  // found the first failing deletion exactly (first_absent).
  __device__ uint32_t limit() const {
    const volatile BatchCtl* c = ctl;
    const unsigned long long cerr = c->commit_err >> 8;
    unsigned long long l = c->limit;
    if (c->use_absent_limit && c->first_absent < l) l = c->first_absent;
    return static_cast<uint32_t>(cerr < l ? cerr : l);
  }

  __device__ const uint32_t* path_of(uint32_t s) const {
    return mout.paths + static_cast<uint64_t>(s) * (o.T + 1ull);
  }

  template <class F>
  __device__ void for_rows(uint32_t k, F&& f) const {
    const DevEvent& e = ev[k];
    f(e.u);
    f(e.v);
    if (e.kind != 1 || o.freeze) return;
    const uint32_t s = slot[k];
    if (s != kNoSlot && mout.has_path[s]) {
      const uint32_t* p = path_of(s);
      const uint32_t len = mout.path_len[s];
      for (uint32_t i = 0; i < len; ++i) f(p[i]);
    } else {
      // Local fallback may add the max-weight live-G edge of either end.
      const uint32_t bu = best_neighbor(G, e.u, e.v, nullptr);
      if (bu != kNoVertex) f(bu);
      const uint32_t bv = best_neighbor(G, e.v, e.u, nullptr);
      if (bv != kNoVertex) f(bv);
    }
  }

  // Lane-parallel row list: index 0 -> u, 1 -> v, then the recovery path
  // vertices or the two fallback candidates.
  template <class F>
  __device__ void for_rows_warp(uint32_t k, uint32_t lane, F&& f) const {
    const DevEvent& e = ev[k];
    uint32_t n = 2;
    const uint32_t* p = nullptr;
    bool fallback = false;
    if (e.kind == 1 && !o.freeze) {
      const uint32_t s = slot[k];
      if (s != kNoSlot && mout.has_path[s]) {
        p = path_of(s);
        n = 2 + mout.path_len[s];
      } else {
        fallback = true;
        n = 4;
      }
    }
    for (uint32_t i = lane; i < n; i += 32) {
      uint32_t row;
      if (i == 0) row = e.u;
      else if (i == 1) row = e.v;
      else if (!fallback) row = p[i - 2];
      else row = i == 2 ? best_neighbor(G, e.u, e.v, nullptr) : best_neighbor(G, e.v, e.u, nullptr);
      if (row != kNoVertex) f(row);
    }
  }

  // Row superset of deletion event k for k_del_flow, known before any event
  // of the batch commits: u, v, plus the recovery path when one was found,
  // or -- when the event may run the local fallback (`fb`) -- every
  // batch-start G neighbour of u and v (the fallback edge is a live-G edge of
  // u or v, and a deletion-only batch only removes G edges). Calls f(i, row)
  // for i = lane, lane + 32, ... < the returned (warp-uniform) count.
  __device__ bool has_path_of(uint32_t k) const {
    const uint32_t s = slot[k];
    return s != kNoSlot && mout.has_path[s] != 0;
  }
  template <class F>
  __device__ uint32_t flow_rows(uint32_t k, uint32_t lane, bool fb, bool keep_g, F&& f) const {
    const DevEvent& e = ev[k];
    const uint32_t* p = nullptr;
    uint32_t n = 2, du = 0, dv = 0;
    if (!o.freeze) {
      if (has_path_of(k)) {
        const uint32_t s = slot[k];
        p = path_of(s);
        n += mout.path_len[s];
      } else if (fb) {
        du = keep_g ? start_deg(e.u) : G.slab[e.u].deg;
        dv = keep_g ? start_deg(e.v) : G.slab[e.v].deg;
        n += du + dv;
      }
    }
    for (uint32_t i = lane; i < n; i += 32) {
      uint32_t r;
      if (i == 0) {
        r = e.u;
      } else if (i == 1) {
        r = e.v;
      } else if (p) {
        r = p[i - 2];
      } else if (keep_g) {
        double w;
        if (i - 2 < du) start_entry(e.u, i - 2, r, w);
        else start_entry(e.v, i - 2 - du, r, w);
      } else {
        r = i - 2 < du ? row(G, e.u).id(i - 2) : row(G, e.v).id(i - 2 - du);
      }
      f(i, r);
    }
    return n;
  }

  // Pull an insertion's four slabs toward L2 one grid barrier before the
  // apply phase needs them.
  __device__ void prefetch(uint32_t k) const {
    const DevEvent& e = ev[k];
    if (e.kind != 0) return;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(G.slab + e.u));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(G.slab + e.v));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(H.slab + e.u));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(H.slab + e.v));
  }

  // Warp-cooperative apply. Insertions run on lane 0. A deletion's path
  // recovery (sparsifier.cpp:503-514) runs over path edges in parallel: the
  // loop-erased path has distinct vertices, hence distinct edges, so each
  // edge's live-H membership and live-G weight are independent of the other
  // path edges' insertions; the appends then go row by row -- row p[j]
  // receives p[j-1] (from edge j-1) before p[j+1] (from edge j), exactly
  // the sequential order.
  __device__ uint32_t apply_warp(uint32_t k, uint32_t lane, Acc& acc, bool keep_g = false) const {
    constexpr unsigned kAll = 0xFFFFFFFFu;
    const DevEvent e = ev[k];
    if (e.kind == 0) {
      uint32_t err = 0;
      if (lane == 0) err = apply(k, acc);
      return __shfl_sync(kAll, err, 0);
    }
    const uint32_t u = e.u, v = e.v;
    const uint32_t s = slot[k];
    // G delete, H membership, H delete (:490-494), on four lanes: the four
    // rows (G u, G v, H u, H v) are distinct, so each lane scans and edits
    // its own row -- one dependent round of row fetches instead of the
    // sequential has_edge / delete_edge chain. has_edge scans the smaller
    // row; either row answers the same (rows are symmetric). H is edited only
    // once the G deletion is known to succeed (:491 throws first).
    int found = -1;
    if (lane < 4 && !(keep_g && lane < 2)) {
      const uint32_t a = (lane & 1) ? v : u, bb = (lane & 1) ? u : v;
      found = lane < 2 ? row_find(G, a, bb) : row_find(H, a, bb);
      if (lane < 2 && found >= 0) row_remove_at(G, a, static_cast<uint32_t>(found));
    }
    // keep mode: the shadow already deleted (u, v) from G, and it existed
    const bool in_g = keep_g || __shfl_sync(kAll, found, 0) >= 0;
    const bool in_h = __shfl_sync(kAll, found, 2) >= 0;
    if (in_g && in_h && (lane == 2 || lane == 3))
      row_remove_at(H, lane == 2 ? u : v, static_cast<uint32_t>(found));
    uint32_t stage = 0;  // 0 error/graph-only/freeze done, 1 path recovery, 2 fallback
    uint32_t err = 0;
    unsigned long long steps = 0;
    if (lane == 0) {
      acc.r[kDelSeen] += 1;
      if (!in_g) {
        err = kErrAbsent;
      } else {
        --acc.dg;
        if (in_h) {
          acc.r[kDelInH] += 1;
          --acc.dh;
          if (!o.freeze) {
            bool path = false;
            if (s != kNoSlot) {
              steps = mout.steps[s];
              path = mout.has_path[s] != 0;
            }
            stage = path ? 1u : 2u;
          } else {
            acc.r[kFallbacks] += 1;
            dec[k] = 2u;
          }
        } else {
          dec[k] = 0u;
        }
      }
    }
    __syncwarp();  // the row updates above visible to the other lanes
    err = __shfl_sync(kAll, err, 0);
    if (err) return err;
    stage = __shfl_sync(kAll, stage, 0);
    uint32_t added = 0;
    if (stage == 1) {
      const uint32_t* p = path_of(s);
      const uint32_t len = mout.path_len[s];
      double* need_w = mscratch.rvals + static_cast<uint64_t>(s) * (o.T + 1ull);
      // Phase 1: per edge i, w if H lacks (p[i], p[i+1]) else -1.
      for (uint32_t i = lane; i + 1 < len; i += 32) {
        const uint32_t a = p[i], bb = p[i + 1];
        need_w[i] = has_edge(H, a, bb) ? -1.0 : edge_weight(G, a, bb);
      }
      __syncwarp();
      // Phase 2: row p[j] appends p[j-1] then p[j+1] where needed.
      uint32_t my_added = 0, fail = 0;
      for (uint32_t j = lane; j < len; j += 32) {
        const uint32_t x = p[j];
        if (j >= 1 && need_w[j - 1] > 0.0) {
          if (!row_push(H, x, p[j - 1], need_w[j - 1])) fail = 1;
        }
        if (j + 1 < len && need_w[j] > 0.0) {
          if (!row_push(H, x, p[j + 1], need_w[j])) fail = 1;
          ++my_added;
        }
      }
      added = static_cast<uint32_t>(warp_sum(my_added));
      if (__any_sync(kAll, fail)) return kErrPool;
      if (lane == 0) {
        acc.dh += added;
        acc.r[kPaths] += 1;
        acc.r[kEdgesRec] += added;
        dec[k] = 1u | (added << 8);
      }
    } else if (stage == 2 && lane == 0) {
      // run_local_fallback (:264-280): u then v.
      const uint32_t ends[2] = {u, v};
      for (int j = 0; j < 2; ++j) {
        const uint32_t x = ends[j];
        if (H.slab[x].deg != 0) continue;
        double bw = 0.0;
        uint32_t b;
        if (keep_g) {  // live G at event k from the batch-start row
          uint32_t gdeg = 0;
          b = live_best(x, k, gdeg, bw);
          if (gdeg == 0) continue;
        } else {
          if (G.slab[x].deg == 0) continue;
          b = best_neighbor(G, x, kNoVertex, &bw);
        }
        if (insert_edge(H, x, b, bw, acc.dh) < 0) {
          err = kErrPool;
          break;
        }
        ++added;
      }
      acc.r[kFallbacks] += 1;
      acc.r[kEdgesRec] += added;
      dec[k] = 2u | (added << 8);
    }
    if (lane == 0) account(acc, steps);
    return __shfl_sync(kAll, err, 0);
  }

  __device__ void flush(const Acc& a) const { flush_acc(a, ctl, G.edges, H.edges); }

  __device__ static void account(Acc& acc, unsigned long long steps) {
    acc.r[kWalkerSteps] += steps;
    if (steps > acc.r[kMaxEventSteps]) acc.r[kMaxEventSteps] = steps;
  }

  __device__ uint32_t apply(uint32_t k, Acc& acc) const {
    const DevEvent e = ev[k];
    const uint32_t u = e.u, v = e.v;
    const uint32_t s = slot[k];
    unsigned long long steps = 0;
    if (e.kind == 0) {
      // :473-488
      acc.r[kInsSeen] += 1;
      if (insert_edge(G, u, v, e.weight, acc.dg) < 0) return kErrPool;
      bool have = false, reached = false;
      if (s != kNoSlot) {
        have = true;
        reached = rout.reached[s] != 0;
        steps = rout.steps[s];
      }
      // commit_insertion (:220-241)
      bool kept;
      if (o.freeze) {
        kept = false;
      } else {
        const double total = edge_weight(G, u, v);
        kept = !(o.K != 0.0 && have && reached);
        if (has_edge(H, u, v)) {
          if (!set_edge_weight(H, u, v, total, acc.dh)) return kErrPool;
        } else if (kept) {
          if (insert_edge(H, u, v, total, acc.dh) < 0) return kErrPool;
        }
      }
      acc.r[kept ? kInsKept : kInsPruned] += 1;
      dec[k] = kept ? 0u : 1u;
      account(acc, steps);
      return 0;
    }
    // Deletion (:489-523)
    acc.r[kDelSeen] += 1;
    if (!delete_edge(G, u, v, acc.dg)) return kErrAbsent;
    uint32_t outcome = 0, added = 0;
    if (has_edge(H, u, v)) {
      acc.r[kDelInH] += 1;
      delete_edge(H, u, v, acc.dh);
      if (!o.freeze) {
        bool path = false;
        if (s != kNoSlot) {
          steps = mout.steps[s];
          path = mout.has_path[s] != 0;
        }
        if (path) {
          const uint32_t* p = path_of(s);
          const uint32_t len = mout.path_len[s];
          for (uint32_t i = 0; i + 1 < len; ++i) {
            const uint32_t a = p[i], bb = p[i + 1];
            if (!has_edge(H, a, bb)) {
              if (insert_edge(H, a, bb, edge_weight(G, a, bb), acc.dh) < 0) return kErrPool;
              ++added;
            }
          }
          acc.r[kPaths] += 1;
          outcome = 1;
        } else {
          // run_local_fallback (:264-280): u then v.
          const uint32_t ends[2] = {u, v};
          for (int j = 0; j < 2; ++j) {
            const uint32_t x = ends[j];
            if (H.slab[x].deg != 0 || G.slab[x].deg == 0) continue;
            double bw = 0.0;
            const uint32_t b = best_neighbor(G, x, kNoVertex, &bw);
            if (insert_edge(H, x, b, bw, acc.dh) < 0) return kErrPool;
            ++added;
          }
          acc.r[kFallbacks] += 1;
          outcome = 2;
        }
        acc.r[kEdgesRec] += added;
      } else {
        acc.r[kFallbacks] += 1;
        outcome = 2;
      }
    }
    dec[k] = outcome | (added << 8);
    account(acc, steps);
    return 0;
  }
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Dataflow commit of a deletion-only batch (the sequential :489-523 loop),
// replacing the dependency rounds: every event lists the superset of rows it
// can touch (CommitOp::flow_rows); per row, the events touching it are
// ordered by event index, and event k may apply once, on each of its rows,
// every earlier event touching that row has applied. Record (row x, event k)
// carries rank = #records of earlier events on x; a row's done counter
// counts applied records, so "done[x] >= rank" is exactly that condition.
// Each warp applies its events in increasing order, so the lowest unapplied
// event is always some warp's current event and has no unapplied
// predecessor: progress is guaranteed, and the result equals the event-order commit bit for bit
// (disjoint events commute). No grid barrier per round: the critical path is
// the longest chain of row-sharing events, not rounds x barriers.
// Phases: emit records + per-row lists | apply (each warp first ranks its
// own events' records, then spins on done) | reset the per-row heads and
// counters; the last block to finish the reset runs the batch epilogue (no
// closing grid barrier). A record-buffer overflow skips the apply phase and
// leaves the batch to the round engine (flow_done = 0).
#ifndef DYG_FLOW_MINB
#define DYG_FLOW_MINB 4
#endif
__global__ void __launch_bounds__(256, DYG_FLOW_MINB) k_del_flow(CommitOp op, uint32_t nev, BatchDev b) {
  constexpr unsigned kAll = 0xFFFFFFFFu;
  cg::grid_group grid = cg::this_grid();
  const uint32_t tid = static_cast<uint32_t>(grid.thread_rank());
  const uint32_t nth = static_cast<uint32_t>(grid.size());
  const uint32_t lane = tid & 31;
  const uint32_t wid = tid >> 5;
  const uint32_t nw = nth >> 5;
  volatile BatchCtl* ctl = b.ctl;
  stamp_commit_start(b.ctl);
  // Keep mode: the shadow's per-row deletion lists stay alive for the
  // live-G reads and are cleared at the end (also on the abort path).
  auto clear_shadow_lists = [&]() {
    if (!op.keep) return;
    for (uint32_t k = tid; k < nev; k += nth) {
      const DevEvent& e = op.ev[k];
      if (e.kind != 1 || e.u >= b.n_vertices || e.v >= b.n_vertices) continue;
      b.fp_head[1][e.u] = kNoSlot;
      b.fp_head[1][e.v] = kNoSlot;
    }
  };
  if (ctl->val_err != ~0ull) {  // uniform
    clear_shadow_lists();
    if (tid == 0) batch_finish(op.G, op.H, b);
    return;
  }
  const uint32_t lim = min(nev, op.limit());
  uint32_t* head = b.fp_head[0];
  uint32_t* done = b.fp_cnt[0];
  uint32_t* mark = b.fp_cnt[1];
  // Balanced apply: the events the apply phase must order ("heavy": every
  // event but the keep-mode accounting-only ones) are dealt round-robin to
  // the warps in event order -- warp w owns the heavy events of rank w, w +
  // nw, ... -- instead of k = w, w + nw, ...: path recoveries (~37 % of a C5
  // deletion batch, each several dependent row round trips) then spread ~1
  // per warp instead of clumping Poisson-wise. The accounting-only events
  // are counted in the reset phase. Ranks come from a bitmap and its word
  // prefix (every block scans it into shared memory), so batches up to 32 x
  // kMaxWords events; larger ones keep the static deal.
  constexpr uint32_t kMaxWords = 1024;
  const uint32_t nwords = (lim + 31) / 32;
  const bool balanced = op.o.flow_balance && nwords <= kMaxWords;
  if (tid == 0) ctl->fl_t[0] = global_ns();
  // Keep the walk shadow as the new G when every deletion found its edge
  // (then the shadow IS the event-order result); otherwise the reference's
  // partial commit needs batch-start G back (restore, then the full commit).
  const bool keep = op.keep && ctl->first_absent == 0xFFFFFFFFu;
  // Undo the in-place walk shadow before anything reads G (same pass as the
  // first step of phase 0, which does not read G).
  if (!keep) restore_rows(op.G, b, tid, nth);
  // Phase 0: which events may run the local fallback. An event whose edge
  // is in batch-start H without a recovered path may. An event whose edge is
  // NOT in batch-start H may only if an earlier fallback inserted its edge
  // into H: recovery paths never do (they run on the shadow G, which lacks
  // every edge this batch deletes), and a fallback edge is incident to that
  // event's u or v. So: mark the endpoints of fallback-capable events and
  // promote the events touching a marked vertex, to a fixpoint (order-free,
  // hence a superset). Most deletions then list only {u, v}.
  // promo bit 0: may run the fallback; bit 1: edge in batch-start H.
  if (!op.o.freeze) {
    for (uint32_t k = tid; k < lim; k += nth) {
      const DevEvent& e = op.ev[k];
      // H is batch-start H until the apply phase. (An event can be in H with
      // no query: a shadow degree of 0 skips the walk, :448.)
      // The single-pass prepare already looked up batch-start H (promo bit 1).
      const bool in_h = op.slot[k] != kNoSlot ||
                        (op.promo_pre ? (b.fl_promo[k] & 2) != 0 : has_edge(op.H, e.u, e.v));
      const bool fb = in_h && !op.has_path_of(k);
      b.fl_promo[k] = (fb ? 1 : 0) | (in_h ? 2 : 0);
      if (fb) {
        mark[e.u] = 1;
        mark[e.v] = 1;
        ctl->fl_any_fb = 1;
      }
    }
  }
  grid.sync();
  // No fallback-capable event: no vertex is marked, nothing can be promoted.
  if (!op.o.freeze && ctl->fl_any_fb) {
    // Three rotating flags: flag (it + 1) % 3 was last read before the
    // barrier that ended iteration it - 1, so resetting it here is safe.
    for (uint32_t it = 0;; ++it) {
      if (tid == 0) ctl->fl_changed[(it + 1) % 3] = 0;
      for (uint32_t k = tid; k < lim; k += nth) {
        if (b.fl_promo[k]) continue;  // fallback-capable already, or in batch-start H
        const DevEvent& e = op.ev[k];
        if (*reinterpret_cast<volatile uint32_t*>(mark + e.u) ||
            *reinterpret_cast<volatile uint32_t*>(mark + e.v)) {
          b.fl_promo[k] = 1;
          mark[e.u] = 1;
          mark[e.v] = 1;
          ctl->fl_changed[it % 3] = 1;
        }
      }
      grid.sync();
      if (!ctl->fl_changed[it % 3]) break;
    }
  }
  if (tid == 0) ctl->fl_t[1] = global_ns();
  // Phase 1: records and per-row lists. Record ranges are allocated per
  // block (a block-wide scan, one atomic per block and pass): one global
  // counter bumped per event serialises ~12k same-address atomics.
  {
    __shared__ uint32_t wcnt[8];
    __shared__ uint32_t bbase;
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t passes = (lim + nw - 1) / nw;
    for (uint32_t pass = 0; pass < passes; ++pass) {
      const uint32_t k = pass * nw + wid;
      const bool fb = k < lim && !op.o.freeze && (b.fl_promo[k] & 1);
      const bool simple = k < lim && op.flow_simple(k, b.fl_promo, keep);
      if (balanced && k < lim && !simple && lane == 0)
        atomicOr(b.fl_heavy + (k >> 5), 1u << (k & 31));
      const uint32_t n =
          (k < lim && !simple) ? op.flow_rows(k, lane, fb, keep, [](uint32_t, uint32_t) {}) : 0;
      if (lane == 0) wcnt[wib] = n;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
          const uint32_t c = wcnt[w];
          wcnt[w] = t;
          t += c;
        }
        bbase = t ? atomicAdd(&b.ctl->fl_top, t) : 0;
      }
      __syncthreads();
      const uint32_t base = bbase + wcnt[wib];
      __syncthreads();  // wcnt / bbase are rewritten next pass
      if (k >= lim) continue;
      if (base + static_cast<uint64_t>(n) > b.fl_cap) {
        if (lane == 0) {
          b.fl_cnt[k] = 0;
          b.ctl->fl_overflow = 1;
        }
        continue;
      }
      if (lane == 0) {
        b.fl_base[k] = base;
        b.fl_cnt[k] = n;
      }
      if (simple) continue;
      op.flow_rows(k, lane, fb, keep, [&](uint32_t i, uint32_t r) {
        b.fl_row[base + i] = r;
        b.fl_ev[base + i] = k;
        b.fl_next[base + i] = atomicExch(head + r, base + i);
      });
    }
  }
  grid.sync();
  if (tid == 0) ctl->fl_t[2] = ctl->fl_t[3] = global_ns();  // (ranks are part of the apply phase)
  const bool overflow = ctl->fl_overflow != 0;
  Acc acc{};
  __shared__ uint32_t s_wpre[kMaxWords + 1];  // exclusive popcount prefix of fl_heavy's words
  if (!overflow) {
    if (balanced) {  // every block: the word prefix of the heavy bitmap
      __shared__ uint32_t s_part[256];
      const uint32_t per = (nwords + blockDim.x - 1) / blockDim.x;
      const uint32_t w0 = threadIdx.x * per;
      uint32_t local = 0;
      for (uint32_t w = w0; w < w0 + per && w < nwords; ++w) local += __popc(b.fl_heavy[w]);
      s_part[threadIdx.x] = local;
      __syncthreads();
      if (threadIdx.x < 32) {  // exclusive scan of the 256 partials, one warp
        uint32_t v[8], run = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[i] = s_part[threadIdx.x * 8 + i];
          run += v[i];
        }
        uint32_t inc = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t t = __shfl_up_sync(kAll, inc, off);
          if (lane >= static_cast<uint32_t>(off)) inc += t;
        }
        uint32_t ex = inc - run;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          s_part[threadIdx.x * 8 + i] = ex;
          ex += v[i];
        }
        if (threadIdx.x == 31) s_wpre[nwords] = inc;
      }
      __syncthreads();
      uint32_t run = s_part[threadIdx.x];
      for (uint32_t w = w0; w < w0 + per && w < nwords; ++w) {
        s_wpre[w] = run;
        run += __popc(b.fl_heavy[w]);
      }
      __syncthreads();
    }
    // Phase 3: apply in dataflow order.
    // Each warp owns events k = wid + j*nw (j = 0, 1, ...) and keeps a
    // window of its 8 lowest unapplied ones, applying whichever is ready
    // (non-blocking readiness polls), so an event stuck behind a long chain
    // does not hold up the warp's independent later events. The lowest
    // unapplied event overall is always inside its owner's window and ready:
    // no deadlock, and no shared work counter to contend on.
    const uint32_t nown = balanced ? s_wpre[nwords] : lim;
    const uint32_t count = wid < nown ? (nown - wid + nw - 1) / nw : 0;
    // The warp's j-th event: rank wid + j * nw among the heavy events
    // (binary search of the word prefix, then the bit within the word).
    auto ev_of = [&](uint32_t j) -> uint32_t {
      const uint32_t h = wid + j * nw;
      if (!balanced) return h;
      uint32_t lo = 0, hi = nwords;  // s_wpre[lo] <= h < s_wpre[hi]
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_wpre[mid] <= h) lo = mid;
        else hi = mid;
      }
      return lo * 32 + __fns(b.fl_heavy[lo], 0, static_cast<int>(h - s_wpre[lo]) + 1);
    };
    // Rank this warp's own events' records (rank = records of earlier events
    // on the row; only the owner's lanes read them), and pull every row the
    // events will touch (G and H slabs) toward L2 now, so the dependent
    // lookups inside apply_warp hit L2 instead of each paying a DRAM round
    // trip in sequence.
    for (uint32_t j = 0; j < count; ++j) {
      const uint32_t k = ev_of(j);
      const uint32_t base = b.fl_base[k], n = b.fl_cnt[k];
      for (uint32_t t = lane; t < n; t += 32) {
        const uint32_t x = b.fl_row[base + t];
        asm volatile("prefetch.global.L2 [%0];" ::"l"(op.G.slab + x));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(op.H.slab + x));
        uint32_t r = 0;
        for (uint32_t q = head[x]; q != kNoSlot; q = b.fl_next[q]) r += b.fl_ev[q] < k;
        b.fl_rank[base + t] = r;
      }
    }
    constexpr uint32_t kWin = 8;
    uint32_t jlo = 0;
    uint32_t mask = count >= kWin ? 0xFFu : ((1u << count) - 1u);
    // The window's event indices (shared memory: registers are the limit
    // at 4 blocks per SM).
    __shared__ uint32_t s_kw[8][kWin];
    uint32_t* kw = s_kw[threadIdx.x >> 5];
    for (uint32_t i = 0; i < kWin; ++i) {
      const uint32_t v = i < count ? ev_of(i) : 0u;
      if (lane == 0) kw[i] = v;
    }
    __syncwarp();
    while (mask) {
      bool progressed = false;
      for (uint32_t i = 0; i < kWin; ++i) {
        if (!((mask >> i) & 1u)) continue;
        const uint32_t k = kw[i];
        const uint32_t base = b.fl_base[k], n = b.fl_cnt[k];
        bool ready = true;
        for (uint32_t t = lane; t < n && ready; t += 32)
          ready = ld_acquire(done + b.fl_row[base + t]) >= b.fl_rank[base + t];
        if (!__all_sync(kAll, ready)) continue;
        __threadfence();
        uint32_t e = 0;
        if ((ctl->commit_err >> 8) > k) {
          if (op.flow_simple(k, b.fl_promo, keep)) {  // G: done by the shadow
            if (lane == 0) {
              acc.r[kDelSeen] += 1;
              --acc.dg;
              op.dec[k] = 0;
            }
          } else {
            e = op.apply_warp(k, lane, acc, keep);
          }
        }
        if (lane == 0) {
          b.state[k] = e ? 2 : 1;
          if (e) atomicMin(&b.ctl->commit_err, (static_cast<unsigned long long>(k) << 8) | e);
        }
        __threadfence();
        __syncwarp();
        for (uint32_t t = lane; t < n; t += 32) atomicAdd(done + b.fl_row[base + t], 1u);
        mask &= ~(1u << i);
        progressed = true;
      }
      // Slide the window past applied events at its bottom.
      while (!(mask & 1u) && jlo < count) {
        mask >>= 1;
        ++jlo;
        uint32_t nxt = 0;
        if (jlo + kWin - 1 < count) {
          mask |= 1u << (kWin - 1);
          nxt = ev_of(jlo + kWin - 1);
        }
        __syncwarp();
        if (lane == 0) {
          for (uint32_t i = 0; i + 1 < kWin; ++i) kw[i] = kw[i + 1];
          kw[kWin - 1] = nxt;
        }
        __syncwarp();
      }
      if (!progressed) __nanosleep(64);
    }
  }
  grid.sync();
  if (tid == 0) ctl->fl_t[4] = global_ns();
  // Phase 4: reset the per-row state for the next batch.
  for (uint32_t k = wid; k < lim; k += nw) {
    const uint32_t base = b.fl_base[k], n = b.fl_cnt[k];
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t x = b.fl_row[base + i];
      head[x] = kNoSlot;
      done[x] = 0;
    }
    if (lane == 0 && (b.fl_promo[k] & 1)) {
      const DevEvent& e = op.ev[k];
      mark[e.u] = 0;
      mark[e.v] = 0;
    }
    // Balanced mode: the accounting-only events, now that commit_err is
    // final (events at or past a failing one never commit, :525-529).
    if (lane == 0 && balanced && !overflow && op.flow_simple(k, b.fl_promo, keep)) {
      b.state[k] = 1;
      if ((ctl->commit_err >> 8) > k) {
        acc.r[kDelSeen] += 1;
        --acc.dg;
        op.dec[k] = 0;
      }
    }
  }
  if (balanced)
    for (uint32_t w = tid; w < nwords; w += nth) b.fl_heavy[w] = 0;
  if (!overflow) op.flush(acc);
  clear_shadow_lists();
  if (overflow) {  // record buffer too small: the dependency rounds commit the batch
    grid.sync();
    if (tid == 0) ctl->fl_t[5] = global_ns();
    if (keep) {  // they re-apply the deletions: batch-start G first
      restore_rows(op.G, b, tid, nth);
      grid.sync();
    }
    rounds_warp_loop(op, nev, b, grid);
    grid.sync();
    if (tid == 0) batch_finish(op.G, op.H, b);
    return;
  }
  // The last block past this point runs the epilogue (its counters are the
  // other blocks' flushed atomics: fence, count, fence).
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&b.ctl->fl_blocks_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    ctl->fl_t[5] = global_ns();
    ctl->flow_done = 1;
    ctl->rounds = ctl->rounds + 1;
    batch_finish(op.G, op.H, b);
  }
}

// Query build (sparsifier.cpp:429-457), phase 1 on batch-start H and G:
// insertion flags and w_pq = G.w(u,v) + w (:441). Runs before the walk
// shadow is applied to G.
__global__ void k_flags_ins(DevGraph<kCapH> H, DevGraph<kCapG> G,
                            const DevEvent* __restrict__ ev, uint32_t nb, WalkOpts o,
                            BatchDev b) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb || batch_aborted(b.ctl)) return;
  const DevEvent e = ev[k];
  unsigned long long flag = 0;
  if (e.kind == 0) {
    const double gw = edge_weight(G, e.u, e.v);
    // Insertion fast path precondition: the key is new to G (no coalescing).
    if (gw != 0.0) b.ctl->not_simple = 1;
    if (o.filtering && H.slab[e.u].deg > 0 && H.slab[e.v].deg > 0) {
      flag = 1ull;
      b.wpq[k] = __dadd_rn(gw, e.weight);
    }
  }
  b.scan_in[k] = flag;
  b.state[k] = 0;
  b.dec[k] = 0;
}

// Phase 2, deletions: batch-start H (:447) and shadow degrees (:448). With
// deletions in the batch G currently IS the shadow (see k_save_rows).
__global__ void k_flags_del(DevGraph<kCapH> H, DevGraph<kCapG> S,
                            const DevEvent* __restrict__ ev, uint32_t nb, WalkOpts o,
                            BatchDev b) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb || batch_aborted(b.ctl)) return;
  const DevEvent e = ev[k];
  if (e.kind == 1 && !o.freeze && has_edge(H, e.u, e.v) && S.slab[e.u].deg > 0 &&
      S.slab[e.v].deg > 0)
    b.scan_in[k] = 1ull << 32;
  b.state[k] = 0;
}

// ------------------------------------------------- single-pass batch prepare
// Validation + query flags + the query scan + the query scatter in ONE
// launch (decoupled look-back scan over 256-event tiles) for insertion-only
// and deletion-only batches: the separate k_validate / k_flags_* / tile scan
// (2 kernels) / k_scatter chain costs five launches and their gaps per batch.
// Same results as that chain: a thread checks its own event's shape before
// touching the graph, and an invalid batch's queries are never committed
// (the commit reads val_err), exactly like the aborted chain.

// Shape check of one event (sparsifier.cpp:321-337); 0 when valid.
__device__ __forceinline__ uint32_t event_code(const DevEvent& e, uint32_t n) {
  if (e.u >= n || e.v >= n) return kErrRange;
  if (e.u == e.v) return kErrSelfLoop;
  if (e.kind == 0 && (!(e.weight > 0.0) || !isfinite(e.weight))) return kErrWeight;
  return 0;
}

// Writes the queries of event k given its scan offsets (ri, mi).
__device__ __forceinline__ void scatter_event(const DevEvent& e, uint32_t k, unsigned long long f,
                                              uint32_t ri, uint32_t mi, uint64_t seed,
                                              const BatchDev& b) {
  const uint64_t uid = b.ctl->counter_base + k;  // update_id = update_counter_ + k (:431)
  uint32_t s = kNoSlot;
  if (f & 0xFFFFFFFFull) {
    ReachQuery q;
    q.p = e.u;
    q.q = e.v;
    q.w_pq = b.wpq[k];
    q.qseed = query_seed(seed, uid);
    b.rq[ri] = q;
    b.rout.reached[ri] = 0;  // the reach walk's OR / SUM / MIN start here
    b.rout.steps[ri] = 0;
    s = ri;
  } else if (f >> 32) {
    MinQuery q;
    q.p = e.u;
    q.q = e.v;
    q.qseed = query_seed(seed, uid);
    b.mq[mi] = q;
    s = mi;
  }
  b.slot[k] = s;
}

// Exclusive prefix of this tile's aggregate over all earlier tiles: the tile
// publishes its aggregate ({value, epoch << 2 | 1}), then the whole block
// sums every earlier tile's aggregate directly, each thread polling its share
// of the predecessors. Aggregates are published as soon as each tile's events
// are processed (all tiles run concurrently), so this waits for the slowest
// predecessor plus one or two L2 round trips -- a look-back chained through
// inclusive prefixes propagates only a window of tiles per round trip (C5:
// 410 tiles, ~13 dependent rounds). Every thread of the block must call it.
__device__ unsigned long long tile_prefix(const BatchDev& b, uint32_t tile,
                                          unsigned long long agg) {
  __shared__ unsigned long long s_part[32];
  const unsigned long long ep = b.ctl->epoch << 2;
  volatile unsigned long long* ts = b.tile_state;
  if (threadIdx.x == 0) {
    ts[3ull * tile] = agg;
    __threadfence();
    ts[3ull * tile + 2] = ep | 1ull;
  }
  unsigned long long sum = 0;
  for (uint32_t j = threadIdx.x; j < tile; j += blockDim.x) {
    while ((ts[3ull * j + 2] & ~3ull) != ep) __nanosleep(32);
    __threadfence();
    sum += ts[3ull * j];
  }
  sum = warp_sum(sum);
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_part[wid] = sum;
  __syncthreads();
  unsigned long long pre = 0;
  for (uint32_t w = 0; w < blockDim.x / 32; ++w) pre += s_part[w];
  return pre;
}

// kDel = false: insertion-only batch (validate + insertion flags).
// kDel = true: deletion-only batch after the shadow (deletion flags).
template <bool kDel>
__global__ void __launch_bounds__(256) k_prep(DevGraph<kCapH> H, DevGraph<kCapG> G,
                                              const DevEvent* __restrict__ ev, uint32_t nb,
                                              uint32_t n, WalkOpts o, BatchDev b) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_warp[8];
  __shared__ unsigned long long s_prefix;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(&b.ctl->tile_ctr, 1u);
    atomicMin(&b.ctl->t_prep0, global_ns());
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t k = tile * 256 + threadIdx.x;
  const bool aborted = kDel ? batch_aborted(b.ctl) : (*b.abort_flag != 0);
  unsigned long long f = 0;
  DevEvent e{};
  if (k < nb && !aborted) {
    e = ev[k];
    if constexpr (!kDel) {
      const uint32_t code = event_code(e, n);
      if (code) {
        atomicMin(&b.ctl->val_err, (static_cast<unsigned long long>(k) << 8) | code);
      } else if (e.kind == 0) {
        // Every request of the event is independent of the others: the
        // list links, G's row u (whole, vector loads) and both H degrees go
        // out together -- one dependent memory round instead of a chain of
        // six. (This kernel runs for insertion-only single-pass batches, so
        // ctl->fast == o.fastpath here.)
        uint32_t gu = 0, gv = 0;
        if (o.fastpath) {  // the fast path's append lists (one set for G and H)
          gu = atomicExch(b.fp_head[0] + e.u, 2 * k);
          gv = atomicExch(b.fp_head[0] + e.v, 2 * k + 1);
        }
        RowRegs<kCapG> gr;
        const uint4* src = reinterpret_cast<const uint4*>(G.slab + e.u);
#pragma unroll
        for (int i = 0; i < RowRegs<kCapG>::kChunks; ++i) gr.v[i] = __ldg(src + i);
        const uint32_t hdu = H.slab[e.u].deg, hdv = H.slab[e.v].deg;
        // G.w(u, v) (either row holds it, graph.cpp symmetric storage)
        double gw = 0.0;
        if (gr.s.ext == kInline) {
#pragma unroll
          for (int i = 0; i < kCapG; ++i)
            if (static_cast<uint32_t>(i) < gr.s.deg && gr.s.id[i] == e.v) gw = gr.s.w[i];
        } else {
          gw = edge_weight(G, e.u, e.v);
        }
        if (gw != 0.0) b.ctl->not_simple = 1;  // fast-path precondition: new key
        if (o.filtering && hdu > 0 && hdv > 0) {
          const double wpq = __dadd_rn(gw, e.weight);
          // long-walking queries count in the low half, the others (with a
          // split) in the high half -- no min-path queries in this batch
          f = (o.split_wpq > 0.0 && wpq > o.split_wpq) ? (1ull << 32) : 1ull;
          b.wpq[k] = wpq;
        }
        if (o.fastpath) {
          b.fp_next[0][2 * k] = gu;
          b.fp_next[0][2 * k + 1] = gv;
        }
      }
      b.dec[k] = 0;
    } else {
      if (e.kind == 1 && !o.freeze) {
        // H's row u (whole) and both shadow-G degrees in one memory round.
        RowRegs<kCapH> hr;
        const uint4* src = reinterpret_cast<const uint4*>(H.slab + e.u);
#pragma unroll
        for (int i = 0; i < RowRegs<kCapH>::kChunks; ++i) hr.v[i] = __ldg(src + i);
        const uint32_t gdu = G.slab[e.u].deg, gdv = G.slab[e.v].deg;
        bool in_h = false;
        if (hr.s.ext == kInline) {
#pragma unroll
          for (int i = 0; i < kCapH; ++i)
            in_h |= static_cast<uint32_t>(i) < hr.s.deg && hr.s.idr(i) == e.v;
        } else {
          in_h = has_edge(H, e.u, e.v);
        }
        if (in_h && gdu > 0 && gdv > 0) f = 1ull << 32;
        b.fl_promo[k] = in_h ? 2 : 0;  // for the flow commit's phase 0
      }
    }
    b.state[k] = 0;
  }
  if (!kDel && k == 0 && *b.abort_flag)
    atomicMin(&b.ctl->val_err, static_cast<unsigned long long>(kErrAborted));
  if (k == 0) *b.work = 0;  // the walk's work counter
  // Block exclusive scan of f (reach count in the low half, min-path high).
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long x = f;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, off);
    if (lane >= static_cast<uint32_t>(off)) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;  // warp totals -> exclusive warp offsets
    for (int w = 0; w < 8; ++w) {
      const unsigned long long t = s_warp[w];
      s_warp[w] = run;
      run += t;
    }
    s_prefix = run;  // the tile's aggregate
  }
  __syncthreads();
  const unsigned long long pre = tile_prefix(b, tile, s_prefix);
  const unsigned long long excl = pre + s_warp[wid] + x - f;
  if (k < nb && !aborted) {
    if (!kDel && (f >> 32)) {
      // short-walking reach query: slots from the top of the buffer
      scatter_event(e, k, 1ull, b.q_cap - 1 - static_cast<uint32_t>(excl >> 32), 0, o.seed, b);
    } else {
      scatter_event(e, k, f, static_cast<uint32_t>(excl & 0xFFFFFFFFull),
                    static_cast<uint32_t>(excl >> 32), o.seed, b);
    }
    if (k == nb - 1) {
      const uint32_t lo = static_cast<uint32_t>((excl + f) & 0xFFFFFFFFull);
      const uint32_t hi = static_cast<uint32_t>((excl + f) >> 32);
      if (kDel) {
        b.ctl->nq_reach = lo;
        b.ctl->nq_min = hi;
      } else {
        b.ctl->nq_reach = lo + hi;
        b.ctl->nq_long = lo;
      }
    }
  }
  if (threadIdx.x == 0) atomicMax(&b.ctl->t_prep1, global_ns());
}

// Deletion-only batch, first launch: validation + the shadow's row lists.
__global__ void k_val_link(const DevEvent* __restrict__ ev, uint32_t nb, uint32_t n,
                           BatchDev b) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  if (*b.abort_flag) {  // an earlier batch of this range failed: do nothing
    if (k == 0) atomicMin(&b.ctl->val_err, static_cast<unsigned long long>(kErrAborted));
    return;
  }
  const DevEvent e = ev[k];
  const uint32_t code = event_code(e, n);
  if (code) {
    atomicMin(&b.ctl->val_err, (static_cast<unsigned long long>(k) << 8) | code);
    return;
  }
  b.dec[k] = 0;
  if (e.kind != 1) return;
  // Lists in slot [1]: the flow commit may keep them alive (fp_head[0] is
  // its own record list head).
  const uint32_t hu = atomicExch(b.fp_head[1] + e.u, 2 * k);
  const uint32_t hv = atomicExch(b.fp_head[1] + e.v, 2 * k + 1);
  b.fp_next[1][2 * k] = hu;
  b.fp_next[1][2 * k + 1] = hv;
}

__global__ void k_scatter(const DevEvent* __restrict__ ev, uint32_t nb, uint64_t seed,
                          BatchDev b) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb || batch_aborted(b.ctl)) return;
  const uint64_t counter = b.ctl->counter_base;
  const unsigned long long f = b.scan_in[k];
  const unsigned long long x = b.scan_out[k];
  const uint32_t ri = static_cast<uint32_t>(x & 0xFFFFFFFFull);
  const uint32_t mi = static_cast<uint32_t>(x >> 32);
  const DevEvent e = ev[k];
  const uint64_t uid = counter + k;  // update_id = update_counter_ + k (:431)
  if (k == 0) *b.work = 0;           // the walk's work counter
  uint32_t s = kNoSlot;
  if (f & 0xFFFFFFFFull) {
    ReachQuery q;
    q.p = e.u;
    q.q = e.v;
    q.w_pq = b.wpq[k];
    q.qseed = query_seed(seed, uid);
    b.rq[ri] = q;
    // The reach walk's order-free reductions start from here (reached = OR,
    // steps = SUM, best = MIN).
    b.rout.reached[ri] = 0;
    b.rout.steps[ri] = 0;
    s = ri;
  } else if (f >> 32) {
    MinQuery q;
    q.p = e.u;
    q.q = e.v;
    q.qseed = query_seed(seed, uid);
    b.mq[mi] = q;
    s = mi;
  }
  b.slot[k] = s;
  if (k == nb - 1) {
    b.ctl->nq_reach = ri + static_cast<uint32_t>(f & 0xFFFFFFFFull);
    b.ctl->nq_min = mi + static_cast<uint32_t>(f >> 32);
  }
}

// Walk shadow without copying G (sparsifier.cpp:416-423 deep-copies it):
// every row a batch deletion will touch is saved once (first claimer of a
// per-vertex stamp), the deletions are then applied to G in place, the
// recovery walks run on G, and k_restore_rows puts the saved rows back
// before the event-order commit. Deletions never relocate a row, so a row's
// overflow block index and capacity are unchanged by the shadow pass.
__global__ void k_save_rows(DevGraph<kCapG> G, const DevEvent* __restrict__ ev, uint32_t nb,
                            uint32_t stamp, BatchDev b) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * nb || batch_aborted(b.ctl)) return;
  const DevEvent e = ev[t >> 1];
  if (e.kind != 1) return;
  const uint32_t row = (t & 1) ? e.v : e.u;
  if (atomicExch(b.mark + row, stamp) == stamp) return;
  const uint32_t idx = atomicAdd(&b.ctl->n_saved, 1u);
  b.saved_rows[idx] = row;
  const Slab<kCapG> sl = G.slab[row];
  b.side_slab[idx] = sl;
  if (sl.ext != kInline) {
    const unsigned long long off = atomicAdd(b.side_top, static_cast<unsigned long long>(sl.deg));
    b.side_off[idx] = off;
    for (uint32_t i = 0; i < sl.deg; ++i) {
      b.side_id[off + i] = G.pool_id[sl.ext + i];
      b.side_w[off + i] = G.pool_w[sl.ext + i];
    }
  }
}

// Walk shadow by per-row event lists (replaces a dependency-round pass):
// the shadow only applies the batch's deletions to G in event order
// (:416-423), and a deletion edits rows u and v alone, so each row can
// replay its own deletions in increasing event order independently. Every
// deletion record r = 2k + side goes onto its row's list (k_sh_link); the
// list head owns the row (k_sh_apply): it saves the row once for
// k_restore_rows, then removes the row's entries in event order. A record
// that finds its edge already gone is an absent deletion; first_absent =
// the lowest such event, exactly the first event whose graph_.delete_edge
// would throw in a deletion-only batch (:491).
__global__ void k_sh_link(const DevEvent* __restrict__ ev, uint32_t nb, BatchDev b) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb || batch_aborted(b.ctl)) return;
  const DevEvent e = ev[k];
  if (e.kind != 1) return;
  const uint32_t hu = atomicExch(b.fp_head[0] + e.u, 2 * k);
  const uint32_t hv = atomicExch(b.fp_head[0] + e.v, 2 * k + 1);
  b.fp_next[0][2 * k] = hu;
  b.fp_next[0][2 * k + 1] = hv;
}

__global__ void k_sh_apply(DevGraph<kCapG> G, const DevEvent* __restrict__ ev, uint32_t nb,
                           uint32_t n, BatchDev b, int list, int keep_lists) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= 2 * nb) return;
  const DevEvent& e = ev[r >> 1];
  if (e.kind != 1 || e.u >= n || e.v >= n || e.u == e.v) return;  // never linked
  const uint32_t row = (r & 1) ? e.v : e.u;
  uint32_t* head = b.fp_head[list];
  if (batch_aborted(b.ctl)) {  // linked before validation finished: just clear
    if (head[row] == r) head[row] = kNoSlot;
    return;
  }
  asm volatile("prefetch.global.L2 [%0];" ::"l"(G.slab + row));
  const uint32_t* next = b.fp_next[list];
  if (head[row] != r) return;
  // Save the row (the owner is its only writer in this pass).
  const uint32_t idx = atomicAdd(&b.ctl->n_saved, 1u);
  b.saved_rows[idx] = row;
  b.save_idx[row] = idx;
  const Slab<kCapG> sl = G.slab[row];
  b.side_slab[idx] = sl;
  if (sl.ext != kInline) {
    const unsigned long long off = atomicAdd(b.side_top, static_cast<unsigned long long>(sl.deg));
    b.side_off[idx] = off;
    for (uint32_t i = 0; i < sl.deg; ++i) {
      b.side_id[off + i] = G.pool_id[sl.ext + i];
      b.side_w[off + i] = G.pool_w[sl.ext + i];
    }
  }
  // The row's deletions in increasing event order.
  uint32_t last = 0;
  for (bool first = true;; first = false) {
    uint32_t best = kNoSlot;
    for (uint32_t x = r; x != kNoSlot; x = next[x])
      if ((first || x > last) && x < best) best = x;
    if (best == kNoSlot) break;
    const DevEvent& eb = ev[best >> 1];
    const uint32_t other = (best & 1) ? eb.u : eb.v;
    const int i = row_find(G, row, other);
    if (i < 0) atomicMin(&b.ctl->first_absent, best >> 1);
    else row_remove_at(G, row, static_cast<uint32_t>(i));
    last = best;
  }
  // The flow commit keeps the lists for its live-G reads and clears them.
  if (!keep_lists) head[row] = kNoSlot;
}


// ---------------------------------------------------------------------------
unsigned grid_for(uint64_t n, unsigned bs = 256) {
  return static_cast<unsigned>((n + bs - 1) / bs);
}

// Rank's contiguous query ranges [floor(nq*r/W), floor(nq*(r+1)/W)) from
// the device counts of the prepare, and its queries moved to
// the front of rq_sh / mq_sh, so the walk runs on [0, n) with a device count.
__global__ void k_shard_range(const BatchCtl* ctl, int rank, int world, uint32_t* rng) {
  const unsigned long long nr = ctl->nq_reach, nm = ctl->nq_min;
  const uint32_t lr = static_cast<uint32_t>(nr * rank / world);
  const uint32_t lm = static_cast<uint32_t>(nm * rank / world);
  rng[0] = lr;
  rng[1] = static_cast<uint32_t>(nr * (rank + 1) / world) - lr;
  rng[2] = lm;
  rng[3] = static_cast<uint32_t>(nm * (rank + 1) / world) - lm;
}
__global__ void k_shard_gather(const ReachQuery* __restrict__ rq, const MinQuery* __restrict__ mq,
                               ReachQuery* rq_sh, MinQuery* mq_sh, const uint32_t* rng,
                               uint32_t max_n) {
  const uint32_t lr = rng[0], nr = rng[1], lm = rng[2], nm = rng[3];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < max_n;
       i += gridDim.x * blockDim.x) {
    if (i < nr) rq_sh[i] = rq[lr + i];
    if (i < nm) mq_sh[i] = mq[lm + i];
  }
}

// The rank's walk results sit at [0, n) (its queries were moved to the
// front, launch_shard_range); n is the device count.
__global__ void k_pack_reach(ReachOut r, const uint32_t* n_dev, uint32_t slots,
                             ReachRecord* rec) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= slots) return;
  const uint32_t n = *n_dev;
  ReachRecord x{0, 0, 0ull};
  if (i < n) {
    x.reached = r.reached[i];
    x.steps = r.steps[i];
  }
  rec[i] = x;
}

__global__ void k_pack_min(MinOut m, const uint32_t* n_dev, uint32_t slots, uint32_t T,
                           uint8_t* rec, size_t rec_bytes) {
  const uint32_t i = blockIdx.x;
  if (i >= slots) return;
  const uint32_t n = *n_dev;
  constexpr uint32_t lo = 0;
  uint8_t* base = rec + static_cast<size_t>(i) * rec_bytes;
  MinRecordHead* h = reinterpret_cast<MinRecordHead*>(base);
  uint32_t* path = reinterpret_cast<uint32_t*>(base + sizeof(MinRecordHead));
  const bool have = i < n;
  const uint32_t len = have ? m.path_len[lo + i] : 0;
  if (threadIdx.x == 0) {
    h->has_path = have ? m.has_path[lo + i] : 0;
    h->path_len = len;
    h->steps = have ? m.steps[lo + i] : 0ull;
    h->resistance = 0.0;  // unused by the commit (K3 skips it in replays)
  }
  const uint32_t* src = m.paths + static_cast<uint64_t>(lo + i) * (T + 1ull);
  for (uint32_t j = threadIdx.x; j < T + 1; j += blockDim.x) path[j] = (j < len) ? src[j] : 0u;
}

// Query q of a world-way split lives on rank r = owner with
// lo_r = floor(nq*r/world) (contiguous ranges).
__device__ __forceinline__ void locate(uint32_t q, uint32_t nq, int world, uint32_t* rank,
                                       uint32_t* idx) {
  uint32_t r = static_cast<uint32_t>((static_cast<unsigned long long>(q) * world) / (nq ? nq : 1));
  while (r + 1 < static_cast<uint32_t>(world) &&
         (static_cast<unsigned long long>(nq) * (r + 1)) / world <= q)
    ++r;
  while (r > 0 && (static_cast<unsigned long long>(nq) * r) / world > q) --r;
  *rank = r;
  *idx = q - static_cast<uint32_t>((static_cast<unsigned long long>(nq) * r) / world);
}

__global__ void k_unpack_reach(ReachOut r, const uint32_t* nq_dev, int world, uint32_t slots,
                               const ReachRecord* rec) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nq = *nq_dev;
  if (q >= nq) return;
  uint32_t rank, idx;
  locate(q, nq, world, &rank, &idx);
  const ReachRecord x = rec[static_cast<size_t>(rank) * slots + idx];
  r.reached[q] = x.reached;
  r.steps[q] = x.steps;
}

__global__ void k_unpack_min(MinOut m, const uint32_t* nq_dev, int world, uint32_t slots,
                             uint32_t T, const uint8_t* rec, size_t rec_bytes) {
  const uint32_t q = blockIdx.x;
  const uint32_t nq = *nq_dev;
  if (q >= nq) return;
  uint32_t rank, idx;
  locate(q, nq, world, &rank, &idx);
  const uint8_t* base = rec + (static_cast<size_t>(rank) * slots + idx) * rec_bytes;
  const MinRecordHead* h = reinterpret_cast<const MinRecordHead*>(base);
  const uint32_t* path = reinterpret_cast<const uint32_t*>(base + sizeof(MinRecordHead));
  if (threadIdx.x == 0) {
    m.has_path[q] = h->has_path;
    m.path_len[q] = h->path_len;
    m.steps[q] = h->steps;
  }
  uint32_t* dst = m.paths + static_cast<uint64_t>(q) * (T + 1ull);
  for (uint32_t j = threadIdx.x; j < h->path_len; j += blockDim.x) dst[j] = path[j];
}

// ---- peer-memory exchange (batch.cuh) -------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint8_t* peer_next_buffer(const PeerX& px) {
  return px.own + kPeerHeader + ((*px.ep + 1ull) & 1ull) * px.stride;
}

__global__ void k_pack_reach_peer(ReachOut r, const uint32_t* n_dev, uint32_t slots, PeerX px) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= slots) return;
  ReachRecord* rec = reinterpret_cast<ReachRecord*>(peer_next_buffer(px));
  const uint32_t n = *n_dev;
  ReachRecord x{0, 0, 0ull};
  if (i < n) {
    x.reached = r.reached[i];
    x.steps = r.steps[i];
  }
  rec[i] = x;
}

// One warp per record (a record is ~0.4 KB: block-per-record grids of 12 k
// small blocks cost more in scheduling than in bytes).
__global__ void k_pack_min_peer(MinOut m, const uint32_t* n_dev, uint32_t slots, uint32_t T,
                                PeerX px) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const size_t rec_bytes = min_record_bytes(T);
  uint8_t* const buf = peer_next_buffer(px) + px.min_off;
  const uint32_t n = *n_dev;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < slots; i += nw) {
    uint8_t* base = buf + static_cast<size_t>(i) * rec_bytes;
    MinRecordHead* h = reinterpret_cast<MinRecordHead*>(base);
    uint32_t* path = reinterpret_cast<uint32_t*>(base + sizeof(MinRecordHead));
    const bool have = i < n;
    const uint32_t len = have ? m.path_len[i] : 0;
    if (lane == 0) {
      h->has_path = have ? m.has_path[i] : 0;
      h->path_len = len;
      h->steps = have ? m.steps[i] : 0ull;
      h->resistance = 0.0;  // unused by the commit (K3 skips it in replays)
    }
    const uint32_t* src = m.paths + static_cast<uint64_t>(i) * (T + 1ull);
    for (uint32_t j = lane; j < len; j += 32) path[j] = src[j];
  }
}

// Publish this rank's records of the batch: epoch += 1, then the release
// store peers acquire. (Stream order: the pack kernels have completed, their
// writes sit in this GPU's L2, where peers' P2P loads are served.) A range
// whose earlier batch failed (abort flag, raised identically on every rank)
// exchanges nothing, on every rank alike.
__global__ void k_peer_signal(PeerX px, const unsigned int* abort_flag) {
  if (*abort_flag) return;
  __threadfence_system();
  const unsigned long long e = *px.ep + 1ull;
  *px.ep = e;
  st_release_sys(reinterpret_cast<unsigned long long*>(px.own), e);
}

// Wait until every rank has published this batch's epoch. A peer that does
// not publish within px.timeout_ns fails the batch (validation slot, code
// kErrPeer) and raises the abort flag: the host then reports a device error
// instead of hanging.
__global__ void k_peer_wait(PeerX px, unsigned int* abort_flag, BatchCtl* ctl) {
  if (*abort_flag) return;
  const unsigned long long e = *px.ep;
  const unsigned long long t0 = global_ns();
  for (int q = 0; q < px.world; ++q) {
    const unsigned long long* f = reinterpret_cast<const unsigned long long*>(px.base[q]);
    while (ld_acquire_sys(f) < e) {
      if (global_ns() - t0 > px.timeout_ns) {
        atomicMin(&ctl->val_err, static_cast<unsigned long long>(kErrPeer));
        atomicExch(abort_flag, 1u);
        return;
      }
      __nanosleep(200);
    }
  }
}

__device__ __forceinline__ const uint8_t* peer_cur_buffer(const PeerX& px, uint32_t rank) {
  return px.base[rank] + kPeerHeader + (*px.ep & 1ull) * px.stride;
}

__global__ void k_unpack_reach_peer(ReachOut r, const uint32_t* nq_dev, uint32_t slots, PeerX px) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nq = *nq_dev;
  if (q >= nq) return;
  uint32_t rank, idx;
  locate(q, nq, px.world, &rank, &idx);
  const ReachRecord x =
      reinterpret_cast<const ReachRecord*>(peer_cur_buffer(px, rank))[idx];
  r.reached[q] = x.reached;
  r.steps[q] = x.steps;
}

__global__ void k_unpack_min_peer(MinOut m, const uint32_t* nq_dev, uint32_t T, PeerX px) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nq = *nq_dev;
  for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nq; q += nw) {
    uint32_t rank, idx;
    locate(q, nq, px.world, &rank, &idx);
    const uint8_t* base =
        peer_cur_buffer(px, rank) + px.min_off + static_cast<size_t>(idx) * min_record_bytes(T);
    const MinRecordHead* h = reinterpret_cast<const MinRecordHead*>(base);
    const uint32_t* path = reinterpret_cast<const uint32_t*>(base + sizeof(MinRecordHead));
    const uint32_t len = h->path_len;
    if (lane == 0) {
      m.has_path[q] = h->has_path;
      m.path_len[q] = len;
      m.steps[q] = h->steps;
    }
    uint32_t* dst = m.paths + static_cast<uint64_t>(q) * (T + 1ull);
    for (uint32_t j = lane; j < len; j += 32) dst[j] = path[j];
  }
}

// Co-resident grid for a cooperative kernel, cached per kernel (not per
// kernel type: several cooperative kernels share a signature).
template <typename K>
int coop_blocks_for(K kernel) {
  // Keyed by (kernel, device), like the walks' shared-memory opt-in.
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  const std::pair<const void*, int> key{reinterpret_cast<const void*>(kernel), dev};
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0);
  const int blocks = sms * (per_sm > 0 ? per_sm : 1);
  cache.emplace(key, blocks);
  return blocks;
}

template <bool kWarp, class Op>
int launch_rounds(const Op& op, uint32_t nev, const BatchDev& b, cudaStream_t st) {
  if (nev == 0) return 0;
  Op op_copy = op;
  BatchDev b_copy = b;
  void* args[] = {&op_copy, &nev, &b_copy};
  if constexpr (kWarp) {
    auto kern = k_rounds_warp<Op>;
    const int need = static_cast<int>(grid_for(static_cast<uint64_t>(nev) * 32));
    const int cap = coop_blocks_for(kern);
    cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern),
                                           dim3(need < cap ? need : cap), dim3(256), args, 0, st),
               "cooperative round launch");
  } else {
    auto kern = k_rounds<Op>;
    const int need = static_cast<int>(grid_for(nev));
    const int cap = coop_blocks_for(kern);
    cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern),
                                           dim3(need < cap ? need : cap), dim3(256), args, 0, st),
               "cooperative round launch");
  }
  return 1;
}

}  // namespace

int coop_grid_blocks(int device) {
  int sms = 0;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");
  return sms;
}

// Query-slot scan of a mixed batch (the packed reach | min-path flags of
// k_flags_ins / k_flags_del): exclusive sum over 2048-event tiles in three
// launches -- per-tile totals, one block scanning the totals in place, then
// every tile scans its own events from its offset. Scratch: one u64 per tile.
constexpr uint32_t kScanThreads = 256;
constexpr uint32_t kScanPer = 8;  // events per thread
constexpr uint32_t kScanTile = kScanThreads * kScanPer;

size_t scan_temp_bytes(uint32_t nb_cap) {
  return sizeof(unsigned long long) * ((static_cast<size_t>(nb_cap) + kScanTile - 1) / kScanTile + 1);
}

__device__ __forceinline__ unsigned long long block_exclusive_u64(unsigned long long x,
                                                                  unsigned long long* total) {
  __shared__ unsigned long long warp_tot[kScanThreads / 32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long inc = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, inc, off);
    if (lane >= static_cast<uint32_t>(off)) inc += y;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  unsigned long long before = 0, all = 0;
  for (uint32_t i = 0; i < kScanThreads / 32; ++i) {
    if (i < w) before += warp_tot[i];
    all += warp_tot[i];
  }
  __syncthreads();  // warp_tot is reused by the next call
  if (total) *total = all;
  return before + inc - x;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const unsigned long long* __restrict__ in,
                                                             uint32_t n,
                                                             unsigned long long* __restrict__ tile_sum) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
  unsigned long long x = 0;
#pragma unroll
  for (uint32_t j = 0; j < kScanPer; ++j) {
    const uint64_t i = base + j * kScanThreads + threadIdx.x;  // coalesced
    if (i < n) x += in[i];
  }
  unsigned long long tot = 0;
  block_exclusive_u64(x, &tot);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_mid(unsigned long long* __restrict__ tile_sum,
                                                           uint32_t tiles) {
  unsigned long long carry = 0;
  for (uint32_t b0 = 0; b0 < tiles; b0 += kScanThreads) {
    const uint32_t t = b0 + threadIdx.x;
    const unsigned long long x = t < tiles ? tile_sum[t] : 0ull;
    unsigned long long tot = 0;
    const unsigned long long ex = block_exclusive_u64(x, &tot);
    if (t < tiles) tile_sum[t] = carry + ex;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const unsigned long long* __restrict__ in,
                                                             uint32_t n,
                                                             const unsigned long long* __restrict__ tile_sum,
                                                             unsigned long long* __restrict__ out) {
  const unsigned long long offset = tile_sum[blockIdx.x];  // exclusive, from k_scan_mid
  // This thread's kScanPer consecutive events.
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanPer;
  unsigned long long v[kScanPer], run = 0;
#pragma unroll
  for (uint32_t j = 0; j < kScanPer; ++j) {
    v[j] = base + j < n ? in[base + j] : 0ull;
    run += v[j];
  }
  unsigned long long acc = offset + block_exclusive_u64(run, nullptr);
#pragma unroll
  for (uint32_t j = 0; j < kScanPer; ++j) {
    if (base + j < n) out[base + j] = acc;
    acc += v[j];
  }
}

// Batch control block initialisation on the device (a kernel instead of a
// host->device copy: a copy-engine transfer in the stream costs several
// microseconds of latency per batch).
__global__ void k_ctl_init(CtlInitArgs a) {
  constexpr uint32_t kWords = sizeof(BatchCtl) / sizeof(uint32_t);
  BatchCtl* ctl = a.ctl;
  uint32_t* w = reinterpret_cast<uint32_t*>(ctl);
  for (uint32_t i = threadIdx.x; i < kWords; i += blockDim.x) w[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl->val_err = ~0ull;
    ctl->commit_err = ~0ull;
    ctl->first_absent = 0xFFFFFFFFu;
    ctl->limit = a.limit;
    ctl->use_absent_limit = a.use_absent_limit;
    ctl->reach.t_start = ctl->reach.t_drain = ctl->minpath.t_start = ctl->minpath.t_drain = ~0ull;
    ctl->fast = a.fast;
    ctl->counter_base = a.counter_base;
    ctl->t_commit0 = ~0ull;
    ctl->t_prep0 = ~0ull;
    ctl->t_batch0 = global_ns();
    ctl->epoch = atomicAdd(a.epoch_ctr, 1ull) + 1ull;
  }
}

int launch_ctl_init(const CtlInitArgs& a, cudaStream_t st) {
  static_assert(sizeof(BatchCtl) % sizeof(uint32_t) == 0, "BatchCtl words");
  k_ctl_init<<<1, 128, 0, st>>>(a);
  return 1;
}

bool ctl_init_node_args(cudaGraphNode_t n, CtlInitArgs* out) {
  cudaGraphNodeType t;
  if (cudaGraphNodeGetType(n, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) return false;
  cudaKernelNodeParams kp{};
  if (cudaGraphKernelNodeGetParams(n, &kp) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (kp.func != reinterpret_cast<void*>(k_ctl_init)) return false;
  *out = *static_cast<const CtlInitArgs*>(kp.kernelParams[0]);
  return true;
}

cudaError_t ctl_init_node_update(cudaGraphExec_t ex, cudaGraphNode_t n, const CtlInitArgs& a) {
  CtlInitArgs copy = a;
  void* args[] = {&copy};
  cudaKernelNodeParams kp{};
  kp.func = reinterpret_cast<void*>(k_ctl_init);
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(128);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  kp.extra = nullptr;
  return cudaGraphExecKernelNodeSetParams(ex, n, &kp);
}

// Insertion (kind 0) / other event counts of a batch: out[0], out[1].
__global__ void k_count_kinds(const DevEvent* __restrict__ ev, uint32_t nb, uint32_t* out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ins = k < nb && ev[k].kind == 0;
  const bool oth = k < nb && ev[k].kind != 0;
  const uint32_t ci = __popc(__ballot_sync(0xFFFFFFFFu, ins));
  const uint32_t co = __popc(__ballot_sync(0xFFFFFFFFu, oth));
  if ((threadIdx.x & 31) == 0) {
    if (ci) atomicAdd(out, ci);
    if (co) atomicAdd(out + 1, co);
  }
}

__global__ void k_export_decisions(const uint32_t* __restrict__ dec,
                                   const DevEvent* __restrict__ ev, uint32_t nb,
                                   uint8_t* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  // dec[k]: insertion 0 Kept / 1 Pruned; deletion 0 GraphOnly /
  // 1 PathRecovered / 2 LocalFallback, edges added in bits 8+.
  const uint32_t d = dec[k] & 0xFFu;
  out[k] = static_cast<uint8_t>(ev[k].kind == 0 ? d : 2u + d);
}

int launch_export_decisions(const uint32_t* dec, const DevEvent* ev, uint32_t nb, uint8_t* out,
                            cudaStream_t st) {
  if (nb == 0) return 0;
  k_export_decisions<<<grid_for(nb), 256, 0, st>>>(dec, ev, nb, out);
  return 1;
}

int launch_count_kinds(const DevEvent* ev, uint32_t nb, uint32_t* out, cudaStream_t st) {
  cuda_check(cudaMemsetAsync(out, 0, 2 * sizeof(uint32_t), st), "kind counts");
  k_count_kinds<<<grid_for(nb), 256, 0, st>>>(ev, nb, out);
  return 1;
}

int launch_validate(const BatchDev& b, uint32_t nb, uint32_t n, const unsigned int* abort_flag,
                    cudaStream_t st) {
  if (nb == 0) return 0;
  k_validate<<<grid_for(nb), 256, 0, st>>>(b.events, nb, n, b.ctl, abort_flag);
  return 1;
}

// The deletion-only commit keeps the walk shadow as G (k_del_flow keep mode):
// needs the single-pass path's kept per-row deletion lists.
bool keep_shadow_commit(const WalkOpts& o, uint32_t nb, uint32_t n_del) {
  return n_del == nb && o.keep_shadow && o.single_pass && o.shadow_lists && o.flow;
}

int launch_prepare(const DevGraph<kCapH>& H, DevGraph<kCapG> G, const BatchDev& b, uint32_t nb,
                   uint32_t n_del, uint32_t n, uint32_t stamp, const WalkOpts& o,
                   cudaStream_t st) {
  if (nb == 0) return 0;
  const unsigned tiles = grid_for(nb);
  if (o.single_pass && n_del == 0) {
    k_prep<false><<<tiles, 256, 0, st>>>(H, G, b.events, nb, n, o, b);
    return 1;
  }
  if (o.single_pass && n_del == nb && o.shadow_lists) {
    k_val_link<<<grid_for(nb), 256, 0, st>>>(b.events, nb, n, b);
    k_sh_apply<<<grid_for(2ull * nb), 256, 0, st>>>(G, b.events, nb, n, b, 1,
                                                    keep_shadow_commit(o, nb, n_del) ? 1 : 0);
    k_prep<true><<<tiles, 256, 0, st>>>(H, G, b.events, nb, n, o, b);
    return 3;
  }
  const int l = launch_validate(b, nb, n, b.abort_flag, st);
  return l + launch_queries(H, G, b, nb, n_del, 0, stamp, o, 0, st);
}

int launch_queries(const DevGraph<kCapH>& H, DevGraph<kCapG> G, const BatchDev& b,
                   uint32_t nb, uint32_t n_del, uint64_t counter, uint32_t stamp,
                   const WalkOpts& o, int coop_blocks, cudaStream_t st) {
  if (nb == 0) return 0;
  int l = 0;
  k_flags_ins<<<grid_for(nb), 256, 0, st>>>(H, G, b.events, nb, o, b);
  ++l;
  if (n_del > 0) {
    if (o.shadow_lists) {
      k_sh_link<<<grid_for(nb), 256, 0, st>>>(b.events, nb, b);
      k_sh_apply<<<grid_for(2ull * nb), 256, 0, st>>>(G, b.events, nb, G.n, b, 0, 0);
      l += 2;
    } else {
      k_save_rows<<<grid_for(2ull * nb), 256, 0, st>>>(G, b.events, nb, stamp, b);
      ++l;
      // The shadow pass must not move G's |E| counter: give it a scratch one.
      DevGraph<kCapG> Gs = G;
      Gs.edges = b.scratch_edges;
      ShadowOp op{Gs, b.events, b.ctl};
      l += launch_rounds<false>(op, nb, b, st);
    }
    k_flags_del<<<grid_for(nb), 256, 0, st>>>(H, G, b.events, nb, o, b);
    ++l;
  }
  const uint32_t tiles = (nb + kScanTile - 1) / kScanTile;
  auto* tile_sum = static_cast<unsigned long long*>(b.scan_temp);
  k_scan_tiles<<<tiles, kScanThreads, 0, st>>>(b.scan_in, nb, tile_sum);
  k_scan_mid<<<1, kScanThreads, 0, st>>>(tile_sum, tiles);
  k_scan_apply<<<tiles, kScanThreads, 0, st>>>(b.scan_in, nb, tile_sum, b.scan_out);
  cuda_check(cudaGetLastError(), "query scan");
  (void)counter;  // read on the device from the control block (graph replay)
  k_scatter<<<grid_for(nb), 256, 0, st>>>(b.events, nb, o.seed, b);
  return l + 4;
}

int launch_commit(const DevGraph<kCapG>& G, const DevGraph<kCapH>& H, const BatchDev& b,
                  uint32_t nb, uint32_t n_del, const WalkOpts& o, cudaStream_t st, bool fp_h) {
  CommitOp op{G, H, b.events, b.slot, b.rout, b.mout, b.mscratch, b.dec, b.ctl, o};
  op.fp_h = fp_h && n_del == 0 ? 1 : 0;
  if (n_del == 0) return launch_rounds<false>(op, nb, b, st);
  if (n_del == nb && o.flow) {
    CommitOp op_copy = op;
    op_copy.promo_pre = (o.single_pass && o.shadow_lists && !o.freeze) ? 1 : 0;
    if (keep_shadow_commit(o, nb, n_del)) {
      op_copy.keep = 1;
      op_copy.save_idx = b.save_idx;
      op_copy.side_slab = b.side_slab;
      op_copy.side_off = b.side_off;
      op_copy.side_id = b.side_id;
      op_copy.side_w = b.side_w;
      op_copy.sh_head = b.fp_head[1];
      op_copy.sh_next = b.fp_next[1];
    }
    BatchDev b_copy = b;
    uint32_t nev = nb;
    void* args[] = {&op_copy, &nev, &b_copy};
    const int need = static_cast<int>(grid_for(static_cast<uint64_t>(nb) * 32));
    const int cap = coop_blocks_for(k_del_flow);
    cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_del_flow),
                                           dim3(need < cap ? need : cap), dim3(256), args, 0, st),
               "cooperative flow launch");
    return 1;
  }
  return launch_rounds<true>(op, nb, b, st);
}

__global__ void k_set_u32x2(uint32_t* dst, uint32_t a, uint32_t b) {
  dst[0] = a;
  dst[1] = b;
}

// Two device words set in stream order from kernel arguments (a host-buffer
// copy would race with the next call's rewrite of that buffer).
int launch_set_u32x2(uint32_t* dst, uint32_t a, uint32_t b, cudaStream_t st) {
  k_set_u32x2<<<1, 1, 0, st>>>(dst, a, b);
  return 1;
}

int launch_fastpath_g(const DevGraph<kCapG>& G, const BatchDev& b, uint32_t nb, cudaStream_t st) {
  if (nb == 0) return 0;
  const uint32_t n = 2 * nb;
  k_fp_check<<<grid_for(n), 256, 0, st>>>(b.events, n, b);
  k_fp_write_g<<<grid_for(n), 256, 0, st>>>(G, b.events, n, b);
  return 2;
}

int launch_shard_range(const BatchDev& b, int rank, int world, uint32_t* rng, uint32_t max_r,
                       uint32_t max_m, cudaStream_t st) {
  k_shard_range<<<1, 1, 0, st>>>(b.ctl, rank, world, rng);
  const uint32_t mx = max_r > max_m ? max_r : max_m;
  if (mx == 0) return 1;
  k_shard_gather<<<grid_for(mx), 256, 0, st>>>(b.rq, b.mq, b.rq_sh, b.mq_sh, rng, mx);
  return 2;
}

int launch_pack(const BatchDev& b, const uint32_t* rng, uint32_t slots_r, uint32_t slots_m,
                uint32_t T, void* rrec, void* mrec, cudaStream_t st) {
  int l = 0;
  if (slots_r) {
    k_pack_reach<<<grid_for(slots_r), 256, 0, st>>>(b.rout, rng + 1, slots_r,
                                                     static_cast<ReachRecord*>(rrec));
    ++l;
  }
  if (slots_m) {
    k_pack_min<<<slots_m, 128, 0, st>>>(b.mout, rng + 3, slots_m, T, static_cast<uint8_t*>(mrec),
                                        min_record_bytes(T));
    ++l;
  }
  return l;
}

size_t peer_area_bytes(uint32_t slots_r, uint32_t slots_m, uint32_t T, size_t* stride,
                       size_t* min_off) {
  const size_t r = (sizeof(ReachRecord) * static_cast<size_t>(slots_r) + 255) & ~size_t(255);
  const size_t m = (min_record_bytes(T) * static_cast<size_t>(slots_m) + 255) & ~size_t(255);
  *min_off = r;
  *stride = r + m;
  return kPeerHeader + 2 * (r + m);
}

int launch_pack_peer(const BatchDev& b, const uint32_t* rng, uint32_t slots_r, uint32_t slots_m,
                     uint32_t T, const PeerX& px, cudaStream_t st) {
  int l = 0;
  if (slots_r) {
    k_pack_reach_peer<<<grid_for(slots_r), 256, 0, st>>>(b.rout, rng + 1, slots_r, px);
    ++l;
  }
  if (slots_m) {
    k_pack_min_peer<<<(slots_m + 7) / 8, 256, 0, st>>>(b.mout, rng + 3, slots_m, T, px);
    ++l;
  }
  k_peer_signal<<<1, 1, 0, st>>>(px, b.abort_flag);
  return l + 1;
}

int launch_unpack_peer(const BatchDev& b, uint32_t max_r, uint32_t max_m, uint32_t slots_r,
                       uint32_t slots_m, uint32_t T, const PeerX& px, cudaStream_t st) {
  k_peer_wait<<<1, 1, 0, st>>>(px, b.abort_flag, b.ctl);
  int l = 1;
  if (max_r && slots_r) {
    k_unpack_reach_peer<<<grid_for(max_r), 256, 0, st>>>(b.rout, &b.ctl->nq_reach, slots_r, px);
    ++l;
  }
  if (max_m && slots_m) {
    k_unpack_min_peer<<<(max_m + 7) / 8, 256, 0, st>>>(b.mout, &b.ctl->nq_min, T, px);
    ++l;
  }
  return l;
}

// Gathered rank-major records -> query order (device query counts; max_r /
// max_m bound them for the grids).
int launch_unpack(const BatchDev& b, uint32_t max_r, uint32_t max_m, int world, uint32_t slots_r,
                  uint32_t slots_m, uint32_t T, const void* rrec, const void* mrec,
                  cudaStream_t st) {
  int l = 0;
  if (max_r && slots_r) {
    k_unpack_reach<<<grid_for(max_r), 256, 0, st>>>(b.rout, &b.ctl->nq_reach, world, slots_r,
                                                    static_cast<const ReachRecord*>(rrec));
    ++l;
  }
  if (max_m && slots_m) {
    k_unpack_min<<<max_m, 128, 0, st>>>(b.mout, &b.ctl->nq_min, world, slots_m, T,
                                        static_cast<const uint8_t*>(mrec), min_record_bytes(T));
    ++l;
  }
  return l;
}



}  // namespace dyg
