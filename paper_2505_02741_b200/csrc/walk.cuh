// walk.cuh -- localized non-backtracking random walks on device rows.
//
// Bit-exact restatement of the reference walk engine
// (proj/src/walk.cpp:17-145) as SIMT lanes: one lane per walker, the s
// walkers of a query on s consecutive lanes. The RNG is the reference's own
// SplitMix64 stream in counter form, so a lane
// needs no generator state; fp64 sums run sequentially in row order with
// explicit _rn intrinsics (no FMA contraction).
#pragma once

#include "dyg_internal.cuh"

namespace dyg {

enum Terminal : uint32_t { kReached = 0, kBudget = 1, kStepCap = 2, kDeadEnd = 3 };  // walk.hpp:20

constexpr uint32_t kNoShift = 0xFFFFFFFFu;

struct WalkParams {
  double K;          // distortion threshold (budget)
  uint32_t T;        // step cap
  uint32_t s;        // walkers per query
  uint64_t seed;     // global seed
  uint32_t s_shift;  // log2(s) when s is a power of two, else kNoShift
  // Per-step statistics (walker steps, algorithmic bytes, tail bytes into
  // WalkCounters): an instrumented kernel variant, ~6 % slower (registers);
  // the stamps (start, drain, end) are always taken.
  uint32_t count;
};

inline WalkParams make_walk_params(double K, uint32_t T, uint32_t s, uint64_t seed) {
  uint32_t sh = kNoShift;
  if (s && (s & (s - 1)) == 0) {
    sh = 0;
    while ((1u << sh) != s) ++sh;
  }
  return WalkParams{K, T, s, seed, sh, 0};
}

// Entries per raw min-path trace: T + 1 rounded up to whole 32 B sectors, so
// the walkers write their traces in full sectors (a partial-sector store
// costs the HBM a read-modify-write).
__host__ __device__ inline uint64_t trace_stride(uint32_t T) {
  return (static_cast<uint64_t>(T) + 1 + 7) & ~7ull;
}

struct ReachQuery {   // WalkQuery Reach (walk.hpp:71-78)
  uint32_t p, q;
  double w_pq;
  uint64_t qseed;   // query_seed(global_seed, update_id)
};
struct MinQuery {     // WalkQuery MinPath
  uint32_t p, q;
  uint64_t qseed;
};

// Per-query outputs of the reach walk (ReachVerdict, walk.hpp:29-33).
struct ReachOut {
  uint32_t* reached;
  unsigned long long* steps;
  unsigned long long* best_bits;  // f64 bits of best_estimate
  // Optional walk-order split: queries [0, *nq_long) sit in slots 0.., the
  // rest in slots cap-1, cap-2, ... (nq_long null: walk order = slot order).
  const uint32_t* nq_long;
  uint32_t cap;
};
// Per-query outputs of the min-path walk (RecoveredPath, walk.hpp:35-39).
struct MinOut {
  uint32_t* has_path;
  uint32_t* path_len;
  unsigned long long* steps;
  double* resistance;
  uint32_t* paths;     // [q*(T+1)] loop-erased vertices
  unsigned long long* t_end;  // optional: %globaltimer at K3 end (max)
};
// Per-walker scratch of the min-path walk.
struct MinScratch {
  double* acc;
  uint32_t* term;
  uint32_t* steps;
  uint32_t* paths;     // [(q*s+i)*trace_stride(T)] raw traces
  double* rvals;       // [q*(T+1)] per-edge 1/w for the resistance sum
};

// Walk-phase counters (device), for the roofline accounting.
struct WalkCounters {
  unsigned long long steps;
  unsigned long long row_bytes;
  unsigned long long tail_bytes;  // row_bytes of steps taken after the warp found the queue drained
  // %globaltimer (ns): first warp start, first warp to find the work queue
  // drained, last warp exit -- the post-drain tail is drain..end.
  unsigned long long t_start;   // min
  unsigned long long t_drain;   // min
  unsigned long long t_end;     // max
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Host launchers (walk.cu). nq_dev: device count of queries (nq_max bounds
// the launch); work: a device u32 work counter. Standalone (run_batch) the
// launchers reset it and initialise / finalise the reach outputs; inside a
// session batch k_scatter does both and best_estimate is not needed.
// stream: session stream. Each returns the number of kernels launched.
template <int C>
int launch_reach(const DevGraph<C>& g, const ReachQuery* q, const uint32_t* nq_dev,
                 uint32_t nq_max, const WalkParams& P, ReachOut out,
                 WalkCounters* ctr, unsigned int* work, cudaStream_t st,
                 bool standalone = true);
template <int C>
int launch_minpath(const DevGraph<C>& g, const MinQuery* q, const uint32_t* nq_dev,
                   uint32_t nq_max, const WalkParams& P, MinScratch scratch, MinOut out,
                   WalkCounters* ctr, unsigned int* work, cudaStream_t st,
                   bool reset_work = true);

}  // namespace dyg
