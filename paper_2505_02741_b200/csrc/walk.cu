// walk.cu -- reach / min-path walk kernels and the min-path winner kernel.
//
// Kernel map (kernel table):
//   K1 k_reach          nbrw_reach + single_walk + sample_neighbor
//                       (proj/src/walk.cpp:17-98)
//   K2 k_minpath        the s walkers of nbrw_min_path (walk.cpp:119-134),
//                       budget +inf, raw traces kept
//   K3 k_minpath_finish winner (strict-< min, lowest walker on ties,
//                       walk.cpp:131-133), loop_erase (walk.cpp:100-117),
//                       resistance recompute (walk.cpp:140-143)
#include <math.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <utility>

#include "walk.cuh"

namespace dyg {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;


inline unsigned blocks_for(uint64_t threads, unsigned per_block) {
  return static_cast<unsigned>((threads + per_block - 1) / per_block);
}

// Cooperative slab gather. A per-lane 16-byte vector load of 32 scattered
// slabs touches 32 different lines per warp instruction, and the L1TEX data
// pipe processes one line per wavefront (ncu: ~42-58% busy, long-scoreboard
// stalls dominate). Here each load instruction covers WHOLE slabs instead --
// 8 lanes x 16 B per 128 B G slab (4 slabs per instruction), 4 lanes x 16 B
// per 64 B H head (8 per instruction) -- so every slab costs one wavefront.
// The slabs are staged in shared memory (row stride padded to 9 / 5 x 16 B,
// conflict-free) and each lane reads its own back. Lanes pass kNoVertex when
// they need no row this iteration.
template <int C>
struct Gather {
  static constexpr int kChunks = C == kCapH ? 4 : 8;  // 16 B chunks fetched
  static constexpr int kLanesPerRow = kChunks;
  static constexpr int kRowsPerRound = 32 / kLanesPerRow;
  static constexpr int kRounds = 32 / kRowsPerRound;
  static constexpr int kStride = kChunks + 1;          // uint4 per staged row
  static constexpr int kWarpWords = 32 * kStride;      // uint4 per warp
};

// 16-byte global->shared async copy (LDGSTS); src_bytes = 0 zero-fills
// without reading (lanes with no row this round).
__device__ __forceinline__ void cp_async16(uint4* dst, const void* src, uint32_t src_bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
               "r"(src_bytes)
               : "memory");
}
// The same through L2 only (no L1 allocation): the min-path walks' G rows,
// whose L1 hit rate is ~9 % (K2 0.5 % faster; the reach walks keep .ca: 31 %).
__device__ __forceinline__ void cp_async16_cg(uint4* dst, const void* src, uint32_t src_bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
               "r"(src_bytes)
               : "memory");
}


// sample_neighbor (walk.cpp:17-37) on an inline row held in registers,
// given this step's uniform draw u01. The reference's pass 1 sums candidate
// weights in row order and its pass 2 re-accumulates the same running sums
// until target < cumulative; both passes produce the identical sequence of
// partial sums, so they are computed ONCE (prefix[i]) and pass 2 becomes
// independent compares -- bit-identical, with half the dependent fp64 adds.
// Candidate weights are pre-masked (non-candidates add +0.0, an exact no-op:
// weights are positive finite, graph.cpp:71), so the chain is DADD after
// DADD. The prefix is then non-decreasing, so {i : target < prefix[i]} is a
// suffix whose first index is a candidate (its prefix rose there): the pick
// is C - popc(hit). None -> the rounding fallback, the last candidate.
// Returns false on a dead end.
template <int C>
__device__ __forceinline__ bool sample_inline(const Slab<C>& s, uint32_t prev, double u01,
                                              uint32_t& next, double& ew) {
  const uint32_t deg = s.deg;
  const uint32_t live = (1u << deg) - 1u;  // deg <= C < 32
  uint32_t cand = 0;
  double prefix[C];
  double total = 0.0;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const uint32_t id = const_cast<Slab<C>&>(s).idr(i);
    const bool c = ((live >> i) & 1u) && id != prev;
    cand |= static_cast<uint32_t>(c) << i;
    total = __dadd_rn(total, c ? const_cast<Slab<C>&>(s).wr(i) : 0.0);
    prefix[i] = total;
  }
  if (total <= 0.0) return false;
  const double target = __dmul_rn(u01, total);
  uint32_t hit = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) hit |= static_cast<uint32_t>(target < prefix[i]) << i;
  const uint32_t sel = hit ? static_cast<uint32_t>(C - __popc(hit)) : 31u - __clz(cand);
  // Select entry `sel` by a mux tree (depth log2 C, not a chain of C moves).
  uint32_t ids[C];
  double ws[C];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    ids[i] = const_cast<Slab<C>&>(s).idr(i);
    ws[i] = const_cast<Slab<C>&>(s).wr(i);
  }
#pragma unroll
  for (int st = 1; st < C; st <<= 1) {
    const bool up = (sel & static_cast<uint32_t>(st)) != 0;
#pragma unroll
    for (int i = 0; i + st < C; i += 2 * st) {
      ids[i] = up ? ids[i + st] : ids[i];
      ws[i] = up ? ws[i + st] : ws[i];
    }
  }
  next = ids[0];
  ew = ws[0];
  return true;
}

// sample_neighbor on an overflow-pool row (rows longer than the slab).
__device__ __forceinline__ bool sample_pool(const uint32_t* __restrict__ ids,
                                            const double* __restrict__ ws, uint32_t deg,
                                            uint32_t prev, double u01, uint32_t& next,
                                            double& ew) {
  double total = 0.0;
  // Both loads of an entry issue together (the weight is not predicated on
  // the id), so an unrolled group costs one round trip, not two.
#pragma unroll 8
  for (uint32_t i = 0; i < deg; ++i) {
    const uint32_t id = __ldg(ids + i);
    const double w = __ldg(ws + i);
    if (id != prev) total = __dadd_rn(total, w);
  }
  if (total <= 0.0) return false;
  const double target = __dmul_rn(u01, total);
  double cum = 0.0;
  for (uint32_t i = 0; i < deg; ++i) {
    const uint32_t id = __ldg(ids + i);
    if (id == prev) continue;
    const double w = __ldg(ws + i);
    cum = __dadd_rn(cum, w);
    next = id;
    ew = w;
    if (target < cum) break;
  }
  return true;
}

// One step at `cur` on the gathered slab head (shared memory). H rows with
// more than 4 entries fetch the slab tail here.
template <int C>
__device__ __forceinline__ bool walk_step(const DevGraph<C>& g, const uint4* head, uint32_t cur,
                                          uint32_t prev, double u01, uint32_t& next, double& ew,
                                          uint32_t& deg) {
  constexpr int NV = RowRegs<C>::kChunks;
  constexpr int NH = Gather<C>::kChunks;
  RowRegs<C> r;
#pragma unroll
  for (int i = 0; i < NH; ++i) r.v[i] = head[i];  // shared-memory reads (LDS.128)
  deg = r.s.deg;
  if (r.s.ext == kInline) {
    if (NH < NV && deg > 4) {
      const uint4* src = reinterpret_cast<const uint4*>(g.slab + cur);
#pragma unroll
      for (int i = NH; i < NV; ++i) r.v[i] = __ldg(src + i);
    }
    return sample_inline<C>(r.s, prev, u01, next, ew);
  }
  return sample_pool(g.pool_id + r.s.ext, g.pool_w + r.s.ext, deg, prev, u01, next, ew);
}

// The whole row of `x` straight into registers (the tail loop).
template <int C>
__device__ __forceinline__ void load_row(const DevGraph<C>& g, uint32_t x, RowRegs<C>& r) {
  const uint4* src = reinterpret_cast<const uint4*>(g.slab + x);
#pragma unroll
  for (int i = 0; i < RowRegs<C>::kChunks; ++i) r.v[i] = __ldg(src + i);
}

// Uniform draw from the SplitMix64 counter (rng.hpp:7-24): `ctr` already
// advanced by gamma for this draw.
__device__ __forceinline__ double u01_of(uint64_t ctr) {
  return __dmul_rn(static_cast<double>(hash_mix(ctr) >> 11), 0x1.0p-53);
}

// Per-lane counters are 32-bit (steps, and bytes in 32 B sectors: a lane
// takes ~10^3 steps per launch, far from 2^32); widened for the warp sum.
__device__ __forceinline__ void add_counters(WalkCounters* ctr, uint32_t steps32,
                                             uint32_t sectors, uint32_t tail_sectors) {
  unsigned long long steps = steps32, bytes = 32ull * sectors, tail = 32ull * tail_sectors;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    steps += __shfl_xor_sync(kFull, steps, off);
    bytes += __shfl_xor_sync(kFull, bytes, off);
    tail += __shfl_xor_sync(kFull, tail, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&ctr->steps, steps);
    atomicAdd(&ctr->row_bytes, bytes);
    atomicAdd(&ctr->tail_bytes, tail);
  }
}

// K1/K2 as persistent lane-refill kernels.
//
// Refill: walk lengths are long-tailed (most insertion walkers dead-end
// within a few steps, a few run to T), so a static lane<->walker mapping
// leaves most lanes idle (ncu: 6.4 of 32 lanes active). A lane that finishes
// a walker takes the next work item (query = w / s, walker = w % s) from a
// warp-local chunk of 32 items whose queries are prefetched with one
// coalesced load (one global atomic per 32 walkers). Latency is hidden by
// resident warps (24 / 16 per SM), not by several walker slots per lane:
// 2-3 slots with pipelined cp.async groups measured slower (DESIGN 4).
//
// Per-walker semantics are single_walk's (walk.cpp:41-80): cap at the loop
// top, then after each traversed edge budget before target. A walker whose
// step count reaches T after a non-terminal step ends as StepCap at once
// (exactly what the next loop-top check would decide, without a row fetch).
//
// Reach results (nbrw_reach, walk.cpp:82-98) are order-free reductions --
// reached = OR, steps = SUM, best = MIN -- so they are accumulated with
// atomics into outputs pre-set by k_reach_init. Min-path walkers keep their
// raw trace and (acc, terminal, steps) for K3.
struct Slot {
  uint32_t cur, prev, tgt, steps, widx, qi;
  bool has;
  uint64_t rng;
  double acc, wpq;
};

struct ChunkSmem {  // per warp: the current 32-item chunk
  uint2 pq[32];
  double w[32];
  unsigned long long seed[32];
  uint32_t qi[32];  // output slot of the item's query (reach)
  double u[32];  // this step's draw, stored before the fetch wait (see k_walk)
};

// Min-path walks: the last 8 trace entries of every lane (entry e in row
// e & 7, lane-minor: conflict-free whatever the lanes' step counts), written
// out a whole 32 B sector at a time. (A register shift register cost ~40
// moves per step.)
struct TraceRing {
  uint32_t e[8][32];
};

template <int C, int kWarps, bool kMinPath = false>
struct WalkLayout {
  static constexpr size_t kStageBytes = sizeof(uint4) * Gather<C>::kWarpWords;
  static constexpr size_t kWarpBytes =
      kStageBytes + sizeof(ChunkSmem) + (kMinPath ? sizeof(TraceRing) : 0);
  static constexpr size_t kBytes = kWarps * kWarpBytes;
};

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Issue (without waiting) the cooperative gather of the 32 rows `my_row`
// of one slot into `stage`, as one cp.async group.
template <int C>
__device__ __forceinline__ void issue_rows(const DevGraph<C>& g, uint32_t my_row, uint4* stage) {
  using Gt = Gather<C>;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t sub = lane / Gt::kLanesPerRow;
  const uint32_t chunk = lane % Gt::kLanesPerRow;
  if (__any_sync(kFull, my_row != kNoVertex)) {
#pragma unroll
    for (int j = 0; j < Gt::kRounds; ++j) {
      const uint32_t r = j * Gt::kRowsPerRound + sub;
      const uint32_t u = __shfl_sync(kFull, my_row, r);
      const bool live = u != kNoVertex;
      const uint4* src = reinterpret_cast<const uint4*>(g.slab + (live ? u : 0)) + chunk;
      if (C == kCapG)
        cp_async16_cg(stage + r * Gt::kStride + chunk, src, live ? 16u : 0u);
      else
        cp_async16(stage + r * Gt::kStride + chunk, src, live ? 16u : 0u);
    }
  }
  cp_async_commit();
}

template <int C, bool kMinPath, int kWarps, int kMinBlocks, bool kCount>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
    k_walk(DevGraph<C> g, const ReachQuery* __restrict__ rq, const MinQuery* __restrict__ mq,
           const uint32_t* __restrict__ nq_dev, WalkParams P, ReachOut rout, MinScratch S,
           WalkCounters* ctr, unsigned int* __restrict__ work) {
  using L = WalkLayout<C, kWarps, kMinPath>;
  // A drained warp with at most this many live walkers finishes them
  // lane by lane (the thin tail below).
  constexpr uint32_t kTailLanes = kMinPath ? 16u : 32u;
  // Min-path walks only: probing the reach walks' queue counter the same way
  // made K1 17 % slower (every warp leaves the cooperative gather as soon as
  // the last chunk is claimed, while most of its walkers are young).
  constexpr bool kProbeDrain = kMinPath;
  // A small min-path batch (fewer walkers than ~4 warps per SM: the memory
  // system is idle) gains nothing from the cooperative gather: its warps go
  // lane by lane as soon as the queue is drained.
  extern __shared__ __align__(16) unsigned char walk_smem[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  unsigned char* wbase = walk_smem + warp * L::kWarpBytes;
  uint4* stage0 = reinterpret_cast<uint4*>(wbase);
  ChunkSmem& cs = *reinterpret_cast<ChunkSmem*>(wbase + L::kStageBytes);
  uint32_t* ring = kMinPath
                       ? reinterpret_cast<TraceRing*>(wbase + L::kStageBytes + sizeof(ChunkSmem))->e[0] + lane
                       : nullptr;  // ring[32 * j] = trace entry j (mod 8) of this lane
  const uint32_t total_work = *nq_dev * P.s;
  const uint32_t tail_lanes = (kMinPath && total_work <= 4u * 32u * 148u) ? 32u : kTailLanes;
  if (threadIdx.x == 0) atomicMin(&ctr->t_start, global_ns());  // block start stamps
  uint32_t chunk_base = 0, chunk_pos = 32, chunk_end = 32;
  bool drained = false;
  uint32_t my_steps = 0, my_sectors = 0, my_tail = 0;  // add_counters

  // Give every lane of the warp whose slot is empty the next work item.
  auto refill = [&](Slot& w) {
    unsigned need = __ballot_sync(kFull, !w.has);
    while (need && !drained) {
      if (chunk_pos == chunk_end) {
        unsigned int base = 0;
        if (lane == 0) base = atomicAdd(work, 32u);
        base = __shfl_sync(kFull, base, 0);
        if (base >= total_work) {
          drained = true;
          if (lane == 0) atomicMin(&ctr->t_drain, global_ns());
          break;
        }
        __syncwarp();  // every lane has read the previous chunk
        chunk_base = base;
        chunk_pos = 0;
        chunk_end = min(32u, total_work - base);
        const uint32_t wi_all = base + lane;
        if (wi_all < total_work) {
          const uint32_t q = P.s_shift != kNoShift ? (wi_all >> P.s_shift) : wi_all / P.s;
          const uint32_t wi = wi_all - q * P.s;
          uint64_t qseed;
          if (kMinPath) {
            const MinQuery Q = mq[q];
            cs.pq[lane] = make_uint2(Q.p, Q.q);
            cs.w[lane] = 1.0;
            qseed = Q.qseed;
          } else {
            uint32_t qq = q;
            if (rout.nq_long) {
              const uint32_t nl = *rout.nq_long;
              if (q >= nl) qq = rout.cap - 1 - (q - nl);
            }
            const ReachQuery Q = rq[qq];
            cs.pq[lane] = make_uint2(Q.p, Q.q);
            cs.w[lane] = Q.w_pq;
            cs.qi[lane] = qq;
            qseed = Q.qseed;
          }
          cs.seed[lane] = walker_seed_from(qseed, wi);
        }
        __syncwarp();
      }
      const uint32_t rank = __popc(need & ((1u << lane) - 1u));
      const uint32_t take = min(static_cast<uint32_t>(__popc(need)), chunk_end - chunk_pos);
      if (((need >> lane) & 1u) && rank < take) {
        const uint32_t item = chunk_pos + rank;
        w.widx = chunk_base + item;
        const uint2 pq = cs.pq[item];
        w.cur = pq.x;
        w.tgt = pq.y;
        w.wpq = cs.w[item];
        w.rng = cs.seed[item];
        if (!kMinPath) w.qi = cs.qi[item];
        w.prev = kNoVertex;
        w.steps = 0;
        w.acc = 0.0;
        w.has = true;
        if (kMinPath) ring[0] = w.cur;  // trace entry 0
      }
      chunk_pos += take;
      need = __ballot_sync(kFull, !w.has);
    }
  };
  auto row_of = [&](const Slot& w) { return (w.has && w.steps < P.T) ? w.cur : kNoVertex; };
  // A walker ended with `term`: its outputs (walk.cpp:82-98 / :119-134).
  auto finish = [&](Slot& w, uint32_t term) {
    if (kCount) my_steps += w.steps;
    if (kMinPath) {
      // The trace's last, partial sector: entries steps-r+1 .. steps.
      const uint32_t r = (w.steps + 1) & 7u;
      uint32_t* tr = S.paths + static_cast<uint64_t>(w.widx) * trace_stride(P.T);
#pragma unroll
      for (int j = 1; j < 8; ++j)
        if (static_cast<uint32_t>(j) <= r) tr[w.steps + 1 - j] = ring[32 * (r - j)];
      S.acc[w.widx] = w.acc;
      S.term[w.widx] = term;
      S.steps[w.widx] = w.steps;
    } else {
      const uint32_t qi = w.qi;
      atomicAdd(&rout.steps[qi], static_cast<unsigned long long>(w.steps));
      if (term == kReached) {
        atomicOr(&rout.reached[qi], 1u);
        // best_estimate is run_batch's; a replay's commit reads `reached`
        // alone (sparsifier.cpp:228-233) and passes no best_bits.
        if (rout.best_bits)
          atomicMin(&rout.best_bits[qi],
                    static_cast<unsigned long long>(__double_as_longlong(w.acc)));
      }
    }
    w.has = false;
  };
  // A traversed edge (next, ew): accumulate, trace, and the budget / target
  // / cap checks in single_walk's order (walk.cpp:62-76).
  auto advance = [&](Slot& w, uint32_t next, double ew) -> uint32_t {
    w.acc = __dadd_rn(w.acc, __drcp_rn(ew));
    ++w.steps;
    w.prev = w.cur;
    w.cur = next;
    if (kMinPath) {
      // Trace entry `steps`; every 8th entry completes a 32 B sector,
      // written whole.
      ring[32 * (w.steps & 7u)] = next;
      if ((w.steps & 7u) == 7u) {
        uint4* dst = reinterpret_cast<uint4*>(
            S.paths + static_cast<uint64_t>(w.widx) * trace_stride(P.T) + (w.steps - 7));
        dst[0] = make_uint4(ring[0], ring[32], ring[64], ring[96]);
        dst[1] = make_uint4(ring[128], ring[160], ring[192], ring[224]);
      }
    }
    if (__dmul_rn(w.wpq, w.acc) > P.K) return kBudget;
    if (next == w.tgt) return kReached;
    if (w.steps >= P.T) return kStepCap;
    return 0xFFFFFFFFu;
  };

  Slot w;
  w.has = false;
  refill(w);
  issue_rows(g, row_of(w), stage0);
  for (;;) {
    // Thin tail: the queue is drained, so no lane takes new work, and at
    // most kTailLanes walkers are left in the warp. Every lane then runs its
    // walker to the end on its own, loading whole rows straight into
    // registers and requesting the next row right after sampling -- no
    // warp-wide gather, shuffles or shared staging on the dependent chain.
    // (With many live lanes the cooperative gather stays: lane-private row
    // loads cost one L1 wavefront per 16 B chunk.)
    if (drained && static_cast<uint32_t>(__popc(__ballot_sync(kFull, w.has))) <= tail_lanes)
      break;
    // This step's uniform draw (draw k = steps + 1) does not depend on the
    // row: computed while the fetch is in flight. The shared store pins it
    // before the wait (ptxas otherwise sinks the hash below the DEPBAR, onto
    // the dependent chain).
    const double u = u01_of(w.rng + kGamma);
    *reinterpret_cast<volatile double*>(&cs.u[lane]) = u;
    // A queue that ran dry without this warp asking (a one-wave min-path
    // batch: every warp took its one chunk at the start) is drained too, so
    // the next rows are requested before the advance arithmetic below. The
    // counter is read while the rows are in flight.
    unsigned int top = 0;
    const bool probe = kProbeDrain && !drained && chunk_pos == chunk_end;
    if (probe && lane == 0) top = *reinterpret_cast<volatile unsigned int*>(work);
    cp_async_wait<0>();
    __syncwarp();
    if (probe) {
      top = __shfl_sync(kFull, top, 0);
      if (top >= total_work) {
        drained = true;
        if (lane == 0) atomicMin(&ctr->t_drain, global_ns());
      }
    }
    // Once the queue is drained no refill follows, so the next row can be
    // requested right after sampling, before the reciprocal / budget
    // arithmetic: in the tail every walker is a chain of dependent steps
    // and this takes that arithmetic off the chain. A walker the budget
    // then ends wastes its fetch (the memory system is idle by then).
    const bool early = drained;
    uint32_t term = 0xFFFFFFFFu;
    uint32_t next = kNoVertex;
    double ew = 0.0;
    if (w.has) {
      if (w.steps >= P.T) {
        term = kStepCap;
      } else {
        w.rng += kGamma;  // draw k = steps + 1 (rng.hpp:7-13)
        uint32_t deg = 0;
        const bool ok =
            walk_step(g, stage0 + lane * Gather<C>::kStride, w.cur, w.prev, u, next, ew, deg);
        if (kCount) {
          my_sectors += step_sectors(deg);
          if (early) my_tail += step_sectors(deg);
        }
        if (!ok) term = kDeadEnd;
      }
    }
    if (early) {
      __syncwarp();  // every lane has read its staged row
      const bool cont = w.has && term == 0xFFFFFFFFu && next != w.tgt && w.steps + 1 < P.T;
      issue_rows(g, cont ? next : kNoVertex, stage0);
    }
    if (w.has) {
      if (term == 0xFFFFFFFFu) term = advance(w, next, ew);
      if (term != 0xFFFFFFFFu) finish(w, term);
    }
    if (!early) {
      __syncwarp();  // every lane has read its staged row before the slot is refilled
      refill(w);
      issue_rows(g, row_of(w), stage0);
    }
    if (!__any_sync(kFull, w.has)) break;
  }
  if (__any_sync(kFull, w.has)) {  // the thin-tail exit above
    cp_async_wait<0>();
    __syncwarp();
    if (w.has) {
      RowRegs<C> r;
      if (w.steps < P.T) {  // its current row is staged (head chunks)
        const uint4* st = stage0 + lane * Gather<C>::kStride;
#pragma unroll
        for (int i = 0; i < Gather<C>::kChunks; ++i) r.v[i] = st[i];
        const uint4* src = reinterpret_cast<const uint4*>(g.slab + w.cur);
#pragma unroll
        for (int i = Gather<C>::kChunks; i < RowRegs<C>::kChunks; ++i) r.v[i] = __ldg(src + i);
      }
      double u = u01_of(w.rng + kGamma);
      for (;;) {
        uint32_t term = 0xFFFFFFFFu;
        uint32_t next = kNoVertex;
        double ew = 0.0;
        if (w.steps >= P.T) {
          term = kStepCap;
        } else {
          w.rng += kGamma;
          const uint32_t deg = r.s.deg;
          const bool ok =
              r.s.ext == kInline
                  ? sample_inline<C>(r.s, w.prev, u, next, ew)
                  : sample_pool(g.pool_id + r.s.ext, g.pool_w + r.s.ext, deg, w.prev, u, next, ew);
          if (kCount) {
            my_sectors += step_sectors(deg);
            my_tail += step_sectors(deg);
          }
          if (!ok) term = kDeadEnd;
        }
        if (term == 0xFFFFFFFFu) {
          if (next != w.tgt && w.steps + 1 < P.T) load_row<C>(g, next, r);
          u = u01_of(w.rng + kGamma);  // the next draw, while the row is in flight
          term = advance(w, next, ew);
        }
        if (term != 0xFFFFFFFFu) {
          finish(w, term);
          break;
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  if (kCount) add_counters(ctr, my_steps, my_sectors, my_tail);
  if (lane == 0) {
    atomicMax(&ctr->t_end, global_ns());
  }
}

__global__ void k_reach_init(ReachOut out, uint32_t n, unsigned int* work) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *work = 0;
  if (i >= n) return;
  out.reached[i] = 0;
  out.steps[i] = 0;
  if (out.best_bits) out.best_bits[i] = 0x7FF0000000000000ull;
}

// Reach outputs of queries that found no walker keep +inf in best_bits;
// the reference leaves best_estimate = 0 when not reached (walk.hpp:31).
__global__ void k_reach_fix(ReachOut out, const uint32_t* __restrict__ nq_dev) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (out.best_bits && i < *nq_dev && !out.reached[i]) out.best_bits[i] = 0ull;
}

// K3: one warp per min-path query: winner, loop erasure, resistance. The
// winner's raw trace, the erased path and the per-edge 1/w live in shared
// memory (each erasure step is a ballot over the path so far: from global
// memory that was ~100 dependent L1/L2 round trips per query).
template <int C>
__global__ void __launch_bounds__(256) k_minpath_finish(DevGraph<C> g,
                                                        const uint32_t* __restrict__ nq_dev,
                                                        WalkParams P, MinScratch S, MinOut out) {
  extern __shared__ __align__(16) unsigned char fin_smem[];
  const uint32_t nq = *nq_dev;
  const uint32_t qi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t T1 = P.T + 1;
  unsigned char* wbase = fin_smem + static_cast<size_t>(threadIdx.x >> 5) * T1 * 16;
  double* rv = reinterpret_cast<double*>(wbase);
  uint32_t* trace = reinterpret_cast<uint32_t*>(wbase + T1 * 8);
  uint32_t* erased = trace + T1;
  if (qi >= nq) return;
  const uint64_t base = static_cast<uint64_t>(qi) * P.s;
  unsigned long long st = 0;
  double bacc = INFINITY;
  uint32_t bidx = 0xFFFFFFFFu;
  for (uint32_t j = lane; j < P.s; j += 32) {
    st += S.steps[base + j];
    if (S.term[base + j] == kReached) {
      const double a = S.acc[base + j];
      if (a < bacc || (a == bacc && j < bidx)) {
        bacc = a;
        bidx = j;
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    st += __shfl_xor_sync(kFull, st, off);
    const double oa = __shfl_xor_sync(kFull, bacc, off);
    const uint32_t oi = __shfl_xor_sync(kFull, bidx, off);
    if (oa < bacc || (oa == bacc && oi < bidx)) {
      bacc = oa;
      bidx = oi;
    }
  }
  if (lane == 0) out.steps[qi] = st;
  if (bidx == 0xFFFFFFFFu) {
    if (lane == 0) {
      out.has_path[qi] = 0;
      out.path_len[qi] = 0;
      if (out.resistance) out.resistance[qi] = 0.0;
      if (out.t_end) atomicMax(out.t_end, global_ns());
    }
    return;
  }
  const uint32_t* gtrace = S.paths + (base + bidx) * trace_stride(P.T);
  const uint32_t len = S.steps[base + bidx] + 1;
  for (uint32_t i = lane; i < len; i += 32) trace[i] = gtrace[i];
  __syncwarp();
  // loop_erase (walk.cpp:100-117): a revisit truncates back to the first
  // occurrence.
  uint32_t elen = 0;
  for (uint32_t i = 0; i < len; ++i) {
    const uint32_t v = trace[i];
    int pos = -1;
    for (uint32_t b = 0; b < elen && pos < 0; b += 32) {
      const uint32_t j = b + lane;
      const unsigned hit = __ballot_sync(kFull, j < elen && erased[j] == v);
      if (hit) pos = static_cast<int>(b + __ffs(hit) - 1);
    }
    if (pos >= 0) {
      elen = static_cast<uint32_t>(pos) + 1;
    } else {
      if (lane == 0) erased[elen] = v;
      ++elen;
    }
    __syncwarp();
  }
  uint32_t* gerased = out.paths + static_cast<uint64_t>(qi) * T1;
  for (uint32_t i = lane; i < elen; i += 32) gerased[i] = erased[i];
  // resistance = sum of 1/w over the erased path in path order
  // (walk.cpp:140-143) -- for run_batch's results; the replay's commit uses
  // only the path (sparsifier.cpp:503-514) and passes no resistance array.
  if (out.resistance) {
    for (uint32_t i = lane; i + 1 < elen; i += 32)
      rv[i] = __drcp_rn(edge_weight(g, erased[i], erased[i + 1]));
    __syncwarp();
  }
  if (lane == 0) {
    if (out.resistance) {
      double r = 0.0;
      for (uint32_t i = 0; i + 1 < elen; ++i) r = __dadd_rn(r, rv[i]);
      out.resistance[qi] = r;
    }
    out.has_path[qi] = 1;
    out.path_len[qi] = elen;
    if (out.t_end) atomicMax(out.t_end, global_ns());
  }
}

}  // namespace

template <typename K>
unsigned persistent_blocks(K kernel, uint64_t work, int threads, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  const unsigned b = static_cast<unsigned>(sms * (per_sm > 0 ? per_sm : 1));
  const unsigned need = blocks_for(work, static_cast<unsigned>(threads));
  return need < b ? need : b;
}

// Opt-in dynamic shared memory is a per-device function attribute: set it
// once per (kernel, device) and check the result (a second device in the
// same process needs its own opt-in).
template <typename K>
bool smem_opt_in(K kernel, size_t bytes) {
  // Keyed by (kernel, device): instantiations of one template share a type.
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const std::pair<const void*, int> key{reinterpret_cast<const void*>(kernel), dev};
  std::lock_guard<std::mutex> lock(mu);
  auto it = granted.find(key);
  if (it != granted.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(bytes)) != cudaSuccess)
    return false;
  granted[key] = bytes;
  return true;
}

// The walk kernel: 8 warps per block; reach walks run 4 blocks per SM
// (64 registers, a few counters spill to L1: measured 5 % faster than 3
// blocks of 79 registers -- more walkers in flight in the bulk phase),
// min-path walks 2 (111 registers; one wave of ~74 k walkers at C5 fills
// 2 x 8 x 32 x 148 lanes anyway).
template <int C, bool kMinPath>
void launch_walk(const DevGraph<C>& g, const ReachQuery* rq, const MinQuery* mq,
                 const uint32_t* nq_dev, uint64_t threads, const WalkParams& P, ReachOut ro,
                 MinScratch S, WalkCounters* ctr, unsigned int* work, cudaStream_t st) {
  constexpr int kWarps = 8;
  constexpr int kMinBlocks = kMinPath ? 2 : 4;
  auto k = P.count ? k_walk<C, kMinPath, kWarps, kMinBlocks, true>
                   : k_walk<C, kMinPath, kWarps, kMinBlocks, false>;
  constexpr size_t smem = WalkLayout<C, kWarps, kMinPath>::kBytes;
  smem_opt_in(k, smem);
  k<<<persistent_blocks(k, threads, kWarps * 32, smem), kWarps * 32, smem, st>>>(
      g, rq, mq, nq_dev, P, ro, S, ctr, work);
}

template <int C>
int launch_reach(const DevGraph<C>& g, const ReachQuery* q, const uint32_t* nq_dev,
                 uint32_t nq_max, const WalkParams& P, ReachOut out, WalkCounters* ctr,
                 unsigned int* work, cudaStream_t st, bool standalone) {
  if (nq_max == 0) return 0;
  int l = 1;
  if (standalone) {
    k_reach_init<<<blocks_for(nq_max, 256), 256, 0, st>>>(out, nq_max, work);
    ++l;
  }
  const uint64_t threads = static_cast<uint64_t>(nq_max) * P.s;
  launch_walk<C, false>(g, q, nullptr, nq_dev, threads, P, out, MinScratch{}, ctr, work, st);
  if (standalone) {
    k_reach_fix<<<blocks_for(nq_max, 256), 256, 0, st>>>(out, nq_dev);
    ++l;
  }
  return l;
}

__global__ void k_zero(unsigned int* work) { *work = 0; }

template <int C>
int launch_minpath(const DevGraph<C>& g, const MinQuery* q, const uint32_t* nq_dev,
                   uint32_t nq_max, const WalkParams& P, MinScratch scratch, MinOut out,
                   WalkCounters* ctr, unsigned int* work, cudaStream_t st, bool reset_work) {
  if (nq_max == 0) return 0;
  int l = 2;
  const uint64_t threads = static_cast<uint64_t>(nq_max) * P.s;
  if (reset_work) {
    k_zero<<<1, 1, 0, st>>>(work);
    ++l;
  }
  launch_walk<C, true>(g, nullptr, q, nq_dev, threads, P, ReachOut{}, scratch, ctr, work, st);
  // 16 B of shared memory per trace position per warp; long caps get one
  // warp per block (up to the opt-in shared-memory limit).
  const size_t per_warp = (static_cast<size_t>(P.T) + 1) * 16;
  const unsigned warps = per_warp * 8 <= 48 * 1024 ? 8u : 1u;
  if (per_warp * warps > 48 * 1024) smem_opt_in(k_minpath_finish<C>, per_warp * warps);
  k_minpath_finish<C><<<blocks_for(static_cast<uint64_t>(nq_max) * 32, 32 * warps), 32 * warps,
                        per_warp * warps, st>>>(g, nq_dev, P, scratch, out);
  return l;
}

template int launch_reach<kCapH>(const DevGraph<kCapH>&, const ReachQuery*, const uint32_t*,
                                 uint32_t, const WalkParams&, ReachOut, WalkCounters*,
                                 unsigned int*, cudaStream_t, bool);
template int launch_minpath<kCapG>(const DevGraph<kCapG>&, const MinQuery*, const uint32_t*,
                                   uint32_t, const WalkParams&, MinScratch, MinOut,
                                   WalkCounters*, unsigned int*, cudaStream_t, bool);


}  // namespace dyg
