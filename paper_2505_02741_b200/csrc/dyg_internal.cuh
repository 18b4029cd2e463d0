// dyg_internal.cuh -- device data layout and shared device helpers.
//
// Device-resident dynamic rows (reference
// DynamicGraph = vector<vector<Neighbor>>, proj/src/graph.hpp:65).
//
// Every vertex owns one fixed-size SLAB holding the row header and, while
// the row fits, the entries themselves:
//   G (C = 10, 128 B, one line):  { u32 deg; u32 ext; u32 id[10]; f64 w[10]; }
//   H (C = 7, 96 B, split):       bytes 0..63 = { deg, ext, id[0..3], w[0..3],
//                                 id[4..5] }, bytes 64..95 = { id[6], pad,
//                                 w[4..6] } -- the first 64 B are a complete
//                                 4-entry row (95% of H rows), the tail is
//                                 fetched only when deg > 4.
// A walker step therefore needs ONE dependent fetch (header + ids + weights
// in the same line) instead of the two a row_ptr CSR needs. A row that
// outgrows its slab moves to the overflow pool (SoA arrays pool_id /
// pool_w, block of cap[u] entries at index ext); the slab then only carries
// deg and ext. Per-row order is exactly the reference's: append =
// push_back (graph.cpp:80-81), delete = move the last entry into the hole
// (graph.cpp:97-108), coalesce in place (graph.cpp:74-79).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dyg {

constexpr uint32_t kNoVertex = 0xFFFFFFFFu;  // walk.cpp:12
constexpr uint32_t kInline = 0xFFFFFFFFu;    // slab.ext for inline rows
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr int kCapH = 7;   // inline entries per H slab (96 B, split 64 + 32)
constexpr int kCapG = 10;  // inline entries per G slab (128 B)
#ifndef DYG_H_SLAB_ALIGN
#define DYG_H_SLAB_ALIGN 32
#endif
constexpr int kHSlabAlign = DYG_H_SLAB_ALIGN;  // 32: 96 B slabs; 128: one line per slab

// rng.hpp:37-41
__host__ __device__ __forceinline__ uint64_t hash_mix(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// rng.hpp:45-50
__host__ __device__ __forceinline__ uint64_t walker_seed(uint64_t global_seed, uint64_t update_id,
                                                         uint64_t walker) {
  uint64_t h = hash_mix(global_seed + 0x9E3779B97F4A7C15ull);
  h = hash_mix(h ^ (update_id + 0xBF58476D1CE4E5B9ull));
  return hash_mix(h ^ (walker + 0x94D049BB133111EBull));
}
// walker_seed split at its query-level part: the first two mixes depend only
// on (global_seed, update_id) and are computed once per query.
__host__ __device__ __forceinline__ uint64_t query_seed(uint64_t global_seed, uint64_t update_id) {
  const uint64_t h = hash_mix(global_seed + 0x9E3779B97F4A7C15ull);
  return hash_mix(h ^ (update_id + 0xBF58476D1CE4E5B9ull));
}
__host__ __device__ __forceinline__ uint64_t walker_seed_from(uint64_t qseed, uint64_t walker) {
  return hash_mix(qseed ^ (walker + 0x94D049BB133111EBull));
}
// The k-th (1-based) SplitMix64 draw of a stream seeded `seed` is
// hash_mix(seed + k*gamma) (rng.hpp:7-13); next_double = (x >> 11) * 2^-53
// (rng.hpp:24). Counter form: a lane computes step t's draw (k = t + 1)
// without carrying generator state.
__device__ __forceinline__ double draw_u01(uint64_t seed, uint32_t k) {
  const uint64_t x = hash_mix(seed + static_cast<uint64_t>(k) * kGamma);
  return __dmul_rn(static_cast<double>(x >> 11), 0x1.0p-53);
}

template <int C>
struct Slab;

template <>
struct alignas(128) Slab<kCapG> {
  uint32_t deg;
  uint32_t ext;
  uint32_t id[kCapG];
  double w[kCapG];
  __host__ __device__ uint32_t& idr(uint32_t i) { return id[i]; }
  __host__ __device__ double& wr(uint32_t i) { return w[i]; }
};

template <>
struct alignas(kHSlabAlign) Slab<kCapH> {
  uint32_t deg;
  uint32_t ext;
  uint32_t id_lo[4];
  double w_lo[4];
  uint32_t id_hi[3];
  uint32_t pad;
  double w_hi[3];
  __host__ __device__ uint32_t& idr(uint32_t i) { return i < 4 ? id_lo[i] : id_hi[i - 4]; }
  __host__ __device__ double& wr(uint32_t i) { return i < 4 ? w_lo[i] : w_hi[i - 4]; }
};
static_assert(sizeof(Slab<kCapH>) == kHSlabAlign || kHSlabAlign == 32, "H slab size");
static_assert(sizeof(Slab<kCapG>) == 128, "G slab must be 128 B");

// A slab's entries as 16 B chunks, for whole-row vector loads into
// registers: H entries end at byte 96 whatever the slab padding.
template <int C>
struct RowRegs {
  static constexpr int kChunks = C == kCapH ? 6 : static_cast<int>(sizeof(Slab<C>) / 16);
  union {
    uint4 v[sizeof(Slab<C>) / 16];
    Slab<C> s;
  };
};

// POD view of one device graph, passed by value to kernels.
template <int C>
struct DevGraph {
  Slab<C>* slab;
  uint32_t* cap;                  // overflow block capacity (0 = inline)
  uint32_t* pool_id;
  double* pool_w;
  unsigned long long* pool_top;   // entries handed out (device counter)
  unsigned long long pool_cap;
  unsigned long long* edges;      // |E| (device counter)
  uint32_t n;
};

// ---------------------------------------------------------------- rows
// Index-based view of row u (inline slab or overflow block).
template <int C>
struct RowRef {
  Slab<C>* s;
  uint32_t* pid;  // nullptr when inline
  double* pw;
  __device__ __forceinline__ uint32_t deg() const { return s->deg; }
  __device__ __forceinline__ uint32_t id(uint32_t i) const { return pid ? pid[i] : s->idr(i); }
  __device__ __forceinline__ double w(uint32_t i) const { return pid ? pw[i] : s->wr(i); }
  __device__ __forceinline__ void set_w(uint32_t i, double x) const {
    if (pid) pw[i] = x;
    else s->wr(i) = x;
  }
  __device__ __forceinline__ void set(uint32_t i, uint32_t id, double x) const {
    if (pid) {
      pid[i] = id;
      pw[i] = x;
    } else {
      s->idr(i) = id;
      s->wr(i) = x;
    }
  }
};
template <int C>
__device__ __forceinline__ RowRef<C> row(const DevGraph<C>& g, uint32_t u) {
  Slab<C>* s = g.slab + u;
  if (s->ext == kInline) return RowRef<C>{s, nullptr, nullptr};
  return RowRef<C>{s, g.pool_id + s->ext, g.pool_w + s->ext};
}
// graph.cpp:34-46 find: index of the first entry of row u with id v, or -1.
template <int C>
__device__ __forceinline__ int row_find(const DevGraph<C>& g, uint32_t u, uint32_t v) {
  const RowRef<C> r = row(g, u);
  const uint32_t d = r.deg();
  for (uint32_t i = 0; i < d; ++i)
    if (r.id(i) == v) return static_cast<int>(i);
  return -1;
}
// graph.cpp:48-53 has_edge (scan the smaller row; symmetric result).
template <int C>
__device__ __forceinline__ bool has_edge(const DevGraph<C>& g, uint32_t u, uint32_t v) {
  if (g.slab[u].deg > g.slab[v].deg) { const uint32_t t = u; u = v; v = t; }
  return row_find(g, u, v) >= 0;
}
// graph.cpp:55-62 edge_weight (0.0 when absent).
template <int C>
__device__ __forceinline__ double edge_weight(const DevGraph<C>& g, uint32_t u, uint32_t v) {
  if (g.slab[u].deg > g.slab[v].deg) { const uint32_t t = u; u = v; v = t; }
  const int i = row_find(g, u, v);
  return i < 0 ? 0.0 : row(g, u).w(static_cast<uint32_t>(i));
}
// push_back with slab -> pool relocation. Returns false when the pool is
// exhausted (the host keeps enough headroom that this never happens).
template <int C>
__device__ __forceinline__ bool row_push(const DevGraph<C>& g, uint32_t u, uint32_t id,
                                         double w) {
  Slab<C>& s = g.slab[u];
  const uint32_t d = s.deg;
  if (s.ext == kInline) {
    if (d < C) {
      s.idr(d) = id;
      s.wr(d) = w;
      s.deg = d + 1;
      return true;
    }
    const uint32_t nc = 2 * C < 8 ? 8 : 2 * C;
    const unsigned long long b = atomicAdd(g.pool_top, static_cast<unsigned long long>(nc));
    if (b + nc > g.pool_cap) return false;
    for (uint32_t i = 0; i < d; ++i) {
      g.pool_id[b + i] = s.idr(i);
      g.pool_w[b + i] = s.wr(i);
    }
    s.ext = static_cast<uint32_t>(b);
    g.cap[u] = nc;
  } else if (d == g.cap[u]) {
    const uint32_t nc = 2 * g.cap[u];
    const unsigned long long b = atomicAdd(g.pool_top, static_cast<unsigned long long>(nc));
    if (b + nc > g.pool_cap) return false;
    for (uint32_t i = 0; i < d; ++i) {
      g.pool_id[b + i] = g.pool_id[s.ext + i];
      g.pool_w[b + i] = g.pool_w[s.ext + i];
    }
    s.ext = static_cast<uint32_t>(b);
    g.cap[u] = nc;
  }
  g.pool_id[s.ext + d] = id;
  g.pool_w[s.ext + d] = w;
  s.deg = d + 1;
  return true;
}
// graph.cpp:97-105 remove_from: the last entry moves into the hole.
template <int C>
__device__ __forceinline__ void row_remove_at(const DevGraph<C>& g, uint32_t u, uint32_t i) {
  const RowRef<C> r = row(g, u);
  const uint32_t last = r.deg() - 1;
  r.set(i, r.id(last), r.w(last));
  r.s->deg = last;
}

// graph.cpp:64-85 insert_edge on validated input. Returns 0 New,
// 1 Coalesced, -1 pool exhausted. |E| changes are accumulated into
// `dedges` by the caller (flushed once per warp, not one atomic per edge).
template <int C>
__device__ __forceinline__ int insert_edge(const DevGraph<C>& g, uint32_t u, uint32_t v,
                                           double w, long long& dedges) {
  const int i = row_find(g, u, v);
  if (i >= 0) {
    const RowRef<C> ru = row(g, u);
    const double nw = __dadd_rn(ru.w(static_cast<uint32_t>(i)), w);
    ru.set_w(static_cast<uint32_t>(i), nw);
    row(g, v).set_w(static_cast<uint32_t>(row_find(g, v, u)), nw);
    return 1;
  }
  if (!row_push(g, u, v, w)) return -1;
  if (!row_push(g, v, u, w)) return -1;
  ++dedges;
  return 0;
}
// graph.cpp:87-112 delete_edge. Returns false when absent (Data error).
template <int C>
__device__ __forceinline__ bool delete_edge(const DevGraph<C>& g, uint32_t u, uint32_t v,
                                            long long& dedges) {
  const int i = row_find(g, u, v);
  if (i < 0) return false;
  row_remove_at(g, u, static_cast<uint32_t>(i));
  row_remove_at(g, v, static_cast<uint32_t>(row_find(g, v, u)));
  --dedges;
  return true;
}

// Algorithmic bytes of one walker step at a row of degree d:
// the header plus d (u32 id, f64 w) pairs, rounded up to 32 B sectors.
__device__ __forceinline__ uint32_t step_sectors(uint32_t d) { return (8u + 12u * d + 31u) / 32u; }
__device__ __forceinline__ uint32_t step_bytes(uint32_t d) { return 32u * step_sectors(d); }

}  // namespace dyg
