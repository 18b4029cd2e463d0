// walk_image.cuh -- compact, read-only walk image of H for the reach walk K1.
//
// K1 (nbrw_reach, proj/src/walk.cpp:82-98) reads batch-start H only, and it
// is bound by random row fetches: ~60 G rows/s from HBM once the table is
// far beyond L2 (tools/gather_peak.cu), more the larger the share that hits
// the 126 MB L2. The authoritative H slabs are 96 B per vertex (403 MB at
// C5) for the commit engines' in-place edits; most rows need far less
// (average H degree 2.2-2.7). The image stores every row in ceil(deg/2)
// 32-byte blocks (181 MB at C5), each block holding two entries:
//
//   block 0   : u32 deg, u32 id0, u32 id1, u32 ext | f64 w0, f64 w1
//   block j>0 : u32 id(2j), u32 id(2j+1), 8 B pad   | f64 w(2j), f64 w(2j+1)
//
// in the reference's row order (graph.hpp:65), so a sampler reads the same
// entries in the same order as from the slab (bit-identical walks). Rows of
// degree > 8 keep only block 0 with `ext` pointing into H's overflow pool.
// loc[v] = (first block << 3) | blocks to fetch (1..4; 0 = pool row); the
// per-vertex loc table (16.8 MB at C5) stays L2-resident, so the walker's
// extra lookup is an L2 hit.
//
// Maintenance: H's mutators flag every row they touch (mark_dirty,
// dyg_internal.cuh); before a reach walk, k_img_sync rewrites the flagged
// rows in place, or in freshly allocated blocks when they outgrew their
// allocation (a bump allocator). When the blocks run out the same launch
// compacts the whole image in place from H's slabs; the host only keeps the
// pool larger than any compact image can be. Snapshots copy the image with H.
#pragma once

#include <stdint.h>

#include "graph_store.cuh"

namespace dyg {

constexpr uint32_t kImgMaxInline = 8;  // entries held in blocks; more -> H's pool

struct WalkImage {
  const uint32_t* loc;  // per vertex: (block << 3) | fetch blocks (0 = pool row)
  const uint4* rec;     // 32 B blocks as uint4 pairs
};

__host__ __device__ inline uint32_t image_blocks(uint32_t deg) {
  return deg > kImgMaxInline ? 1u : (deg < 2 ? 1u : (deg + 1) / 2);
}
__host__ __device__ inline uint32_t image_fetch(uint32_t deg) {
  return deg > kImgMaxInline ? 0u : image_blocks(deg);
}

class WalkImageStore {
 public:
  WalkImageStore() = default;
  ~WalkImageStore();
  WalkImageStore(const WalkImageStore&) = delete;
  WalkImageStore& operator=(const WalkImageStore&) = delete;

  // Full build from H (clears the change flags); allocates on first use.
  // Synchronises `st`.
  void build(const DevGraph<kCapH>& h, cudaStream_t st);
  // Rewrites the rows H's mutators flagged since the last sync (enqueued,
  // capturable; compacts in place when the block pool runs out). Returns
  // the number of kernels launched.
  int sync(const DevGraph<kCapH>& h, cudaStream_t st);
  // Before enqueueing work after which H may hold up to h_edges_bound
  // edges: guarantees a compaction always fits (grows and rebuilds
  // otherwise; never inside a capture).
  void ensure_capacity(const DevGraph<kCapH>& h, uint64_t h_edges_bound, cudaStream_t st);
  void copy_from(const WalkImageStore& o, cudaStream_t st);  // snapshot / restore

  WalkImage view() const { return WalkImage{loc_, rec_}; }
  uint8_t* dirty() const { return dirty_; }
  bool built() const { return built_; }
  uint64_t capacity_blocks() const { return cap_; }

 private:
  void allocate(uint32_t n, uint64_t cap_blocks);
  void release();
  uint32_t n_ = 0;
  uint32_t* loc_ = nullptr;
  uint8_t* alloc_ = nullptr;   // blocks allocated per vertex
  uint8_t* dirty_ = nullptr;
  uint4* rec_ = nullptr;
  unsigned long long* top_ = nullptr;  // device: [0] blocks handed out, [1] overflow flag
  unsigned long long* sums_ = nullptr; // compaction scan scratch (one per sync block)
  uint64_t cap_ = 0;                   // blocks
  int grid_ = 0;                       // sync blocks (all co-resident)
  bool built_ = false;
};

}  // namespace dyg
