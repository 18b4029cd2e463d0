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

#include "walk.cuh"

namespace dyg {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// One sample_neighbor call (walk.cpp:17-37) at `cur`. Loads the whole slab
// with 16-byte vector loads (one line), sums candidate weights in row order
// (pass 1), draws target = u01 * total with draw k, and selects the first
// candidate whose running sum exceeds target (pass 2), falling back to the
// last candidate. Returns false on a dead end (no draw consumed).
template <int C>
__device__ __forceinline__ bool walk_step(const DevGraph<C>& g, uint32_t cur, uint32_t prev,
                                          uint64_t wseed, uint32_t k, uint32_t& next,
                                          double& ew, uint32_t& deg) {
  constexpr int NV = static_cast<int>(sizeof(Slab<C>) / 16);
  union {
    uint4 v[NV];
    Slab<C> s;
  } r;
  const uint4* src = reinterpret_cast<const uint4*>(g.slab + cur);
#pragma unroll
  for (int i = 0; i < NV; ++i) r.v[i] = __ldg(src + i);
  deg = r.s.deg;
  if (r.s.ext == kInline) {
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i)
      if (i < static_cast<int>(deg) && r.s.id[i] != prev) total = __dadd_rn(total, r.s.w[i]);
    if (total <= 0.0) return false;
    const double target = __dmul_rn(draw_u01(wseed, k), total);
    double cum = 0.0;
    bool found = false;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      if (!found && i < static_cast<int>(deg) && r.s.id[i] != prev) {
        cum = __dadd_rn(cum, r.s.w[i]);
        next = r.s.id[i];
        ew = r.s.w[i];
        if (target < cum) found = true;
      }
    }
    return true;
  }
  const uint32_t* ids = g.pool_id + r.s.ext;
  const double* ws = g.pool_w + r.s.ext;
  double total = 0.0;
  for (uint32_t i = 0; i < deg; ++i)
    if (__ldg(ids + i) != prev) total = __dadd_rn(total, __ldg(ws + i));
  if (total <= 0.0) return false;
  const double target = __dmul_rn(draw_u01(wseed, k), total);
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

__device__ __forceinline__ void add_counters(WalkCounters* ctr, unsigned long long steps,
                                             unsigned long long bytes) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    steps += __shfl_xor_sync(kFull, steps, off);
    bytes += __shfl_xor_sync(kFull, bytes, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&ctr->steps, steps);
    atomicAdd(&ctr->row_bytes, bytes);
  }
}

// K1: lane = (query, walker); the s walkers of a query sit on s consecutive
// lanes. single_walk's check order (walk.cpp:54-78): cap at the loop top,
// then after each traversed edge budget before target.
template <int C>
__global__ void __launch_bounds__(256) k_reach(DevGraph<C> g, const ReachQuery* __restrict__ qs,
                                               const uint32_t* __restrict__ nq_dev, WalkParams P,
                                               ReachOut out, WalkCounters* ctr) {
  const uint32_t nq = *nq_dev;
  const uint64_t gt = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t qi = static_cast<uint32_t>(gt / P.s);
  const uint32_t wi = static_cast<uint32_t>(gt % P.s);
  const bool valid = qi < nq;
  if (__all_sync(kFull, !valid)) return;

  uint32_t steps = 0;
  double acc = 0.0;
  bool reached = false;
  unsigned long long bytes = 0;
  if (valid) {
    const ReachQuery Q = qs[qi];
    const uint64_t wseed = walker_seed(P.seed, Q.update_id, wi);
    uint32_t cur = Q.p, prev = kNoVertex;
    while (steps < P.T) {
      uint32_t next = kNoVertex, deg = 0;
      double ew = 0.0;
      const bool ok = walk_step(g, cur, prev, wseed, steps + 1, next, ew, deg);
      bytes += step_bytes(deg);
      if (!ok) break;
      acc = __dadd_rn(acc, __drcp_rn(ew));
      ++steps;
      prev = cur;
      cur = next;
      if (__dmul_rn(Q.w_pq, acc) > P.K) break;
      if (cur == Q.q) {
        reached = true;
        break;
      }
    }
  }
  add_counters(ctr, steps, bytes);

  // nbrw_reach (walk.cpp:82-98): reached = any; best = min; steps = sum.
  // All three reductions are order-free, so a tree reduction is exact.
  if (P.s <= 32 && (P.s & (P.s - 1)) == 0) {
    unsigned long long st = steps;
    uint32_t r = reached ? 1u : 0u;
    double best = reached ? acc : INFINITY;
    for (uint32_t off = 1; off < P.s; off <<= 1) {
      st += __shfl_xor_sync(kFull, st, off);
      r |= __shfl_xor_sync(kFull, r, off);
      best = fmin(best, __shfl_xor_sync(kFull, best, off));
    }
    if (valid && wi == 0) {
      out.reached[qi] = r;
      out.steps[qi] = st;
      out.best_bits[qi] = r ? static_cast<unsigned long long>(__double_as_longlong(best)) : 0ull;
    }
  } else if (valid) {
    // Outputs pre-set to {0, 0, +inf bits}; positive doubles order as u64.
    atomicAdd(&out.steps[qi], static_cast<unsigned long long>(steps));
    if (reached) {
      atomicOr(&out.reached[qi], 1u);
      atomicMin(&out.best_bits[qi], static_cast<unsigned long long>(__double_as_longlong(acc)));
    }
  }
}

__global__ void k_reach_init(ReachOut out, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out.reached[i] = 0;
  out.steps[i] = 0;
  out.best_bits[i] = 0x7FF0000000000000ull;
}

// K2: min-path walkers (w_pq = 1, budget from P.K = +inf for deletions),
// raw trace of each walker kept for K3.
template <int C>
__global__ void __launch_bounds__(256) k_minpath(DevGraph<C> g, const MinQuery* __restrict__ qs,
                                                 const uint32_t* __restrict__ nq_dev,
                                                 WalkParams P, MinScratch S, WalkCounters* ctr) {
  const uint32_t nq = *nq_dev;
  const uint64_t gt = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t qi = static_cast<uint32_t>(gt / P.s);
  const uint32_t wi = static_cast<uint32_t>(gt % P.s);
  const bool valid = qi < nq;
  if (__all_sync(kFull, !valid)) return;
  uint32_t steps = 0;
  unsigned long long bytes = 0;
  if (valid) {
    const MinQuery Q = qs[qi];
    const uint64_t wseed = walker_seed(P.seed, Q.update_id, wi);
    uint32_t* trace = S.paths + gt * (P.T + 1ull);
    uint32_t cur = Q.p, prev = kNoVertex;
    uint32_t term = kStepCap;
    double acc = 0.0;
    trace[0] = cur;
    while (true) {
      if (steps >= P.T) {
        term = kStepCap;
        break;
      }
      uint32_t next = kNoVertex, deg = 0;
      double ew = 0.0;
      const bool ok = walk_step(g, cur, prev, wseed, steps + 1, next, ew, deg);
      bytes += step_bytes(deg);
      if (!ok) {
        term = kDeadEnd;
        break;
      }
      acc = __dadd_rn(acc, __drcp_rn(ew));
      ++steps;
      prev = cur;
      cur = next;
      trace[steps] = cur;
      if (__dmul_rn(1.0, acc) > P.K) {
        term = kBudget;
        break;
      }
      if (cur == Q.q) {
        term = kReached;
        break;
      }
    }
    S.acc[gt] = acc;
    S.term[gt] = term;
    S.steps[gt] = steps;
  }
  add_counters(ctr, steps, bytes);
}

// K3: one warp per min-path query.
template <int C>
__global__ void __launch_bounds__(256) k_minpath_finish(DevGraph<C> g,
                                                        const uint32_t* __restrict__ nq_dev,
                                                        WalkParams P, MinScratch S, MinOut out) {
  const uint32_t nq = *nq_dev;
  const uint32_t qi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
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
      out.resistance[qi] = 0.0;
    }
    return;
  }
  const uint32_t* trace = S.paths + (base + bidx) * (P.T + 1ull);
  const uint32_t len = S.steps[base + bidx] + 1;
  uint32_t* erased = out.paths + static_cast<uint64_t>(qi) * (P.T + 1ull);
  // loop_erase: a revisit truncates back to the first occurrence.
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
  double* rv = S.rvals + static_cast<uint64_t>(qi) * (P.T + 1ull);
  for (uint32_t i = lane; i + 1 < elen; i += 32)
    rv[i] = __drcp_rn(edge_weight(g, erased[i], erased[i + 1]));
  __syncwarp();
  if (lane == 0) {
    double r = 0.0;
    for (uint32_t i = 0; i + 1 < elen; ++i) r = __dadd_rn(r, rv[i]);
    out.has_path[qi] = 1;
    out.path_len[qi] = elen;
    out.resistance[qi] = r;
  }
}

inline unsigned blocks_for(uint64_t threads, unsigned per_block) {
  return static_cast<unsigned>((threads + per_block - 1) / per_block);
}

}  // namespace

template <int C>
int launch_reach(const DevGraph<C>& g, const ReachQuery* q, const uint32_t* nq_dev,
                 uint32_t nq_max, const WalkParams& P, ReachOut out, WalkCounters* ctr,
                 cudaStream_t st) {
  if (nq_max == 0) return 0;
  int launches = 0;
  const bool seg = P.s <= 32 && (P.s & (P.s - 1)) == 0;
  if (!seg) {
    k_reach_init<<<blocks_for(nq_max, 256), 256, 0, st>>>(out, nq_max);
    ++launches;
  }
  const uint64_t threads = static_cast<uint64_t>(nq_max) * P.s;
  k_reach<C><<<blocks_for(threads, 256), 256, 0, st>>>(g, q, nq_dev, P, out, ctr);
  return launches + 1;
}

template <int C>
int launch_minpath(const DevGraph<C>& g, const MinQuery* q, const uint32_t* nq_dev,
                   uint32_t nq_max, const WalkParams& P, MinScratch scratch, MinOut out,
                   WalkCounters* ctr, cudaStream_t st) {
  if (nq_max == 0) return 0;
  const uint64_t threads = static_cast<uint64_t>(nq_max) * P.s;
  k_minpath<C><<<blocks_for(threads, 256), 256, 0, st>>>(g, q, nq_dev, P, scratch, ctr);
  k_minpath_finish<C><<<blocks_for(static_cast<uint64_t>(nq_max) * 32, 256), 256, 0, st>>>(
      g, nq_dev, P, scratch, out);
  return 2;
}

template int launch_reach<kCapH>(const DevGraph<kCapH>&, const ReachQuery*, const uint32_t*,
                                 uint32_t, const WalkParams&, ReachOut, WalkCounters*,
                                 cudaStream_t);
template int launch_reach<kCapG>(const DevGraph<kCapG>&, const ReachQuery*, const uint32_t*,
                                 uint32_t, const WalkParams&, ReachOut, WalkCounters*,
                                 cudaStream_t);
template int launch_minpath<kCapG>(const DevGraph<kCapG>&, const MinQuery*, const uint32_t*,
                                   uint32_t, const WalkParams&, MinScratch, MinOut,
                                   WalkCounters*, cudaStream_t);
template int launch_minpath<kCapH>(const DevGraph<kCapH>&, const MinQuery*, const uint32_t*,
                                   uint32_t, const WalkParams&, MinScratch, MinOut,
                                   WalkCounters*, cudaStream_t);

}  // namespace dyg
