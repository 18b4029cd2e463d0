// walk_image.cuh -- compact, read-only walk image of H for the reach walk K1.
//
// K1 (nbrw_reach, proj/src/walk.cpp:82-98) reads batch-start H only, one
// dependent row fetch per walker step. The authoritative H slabs are 96 B per
// vertex (403 MB at C5) so the commit engines can edit rows in place; most
// rows need far less (average H degree 2.2-2.7), and a 403 MB table hits the
// 126 MB L2 for ~26 % of the fetches. The image stores every row in
// ceil(deg / 2) 32-byte blocks (181 MB at C5: ~58 % L2 hits), two entries
// per block, in the reference's row order (graph.hpp:65) so a sampler reads
// the same entries in the same order as from the slab (bit-identical walks):
//
//   block j : u32 id(2j), u32 id(2j+1), u32 loc(2j), u32 loc(2j+1)
//             | f64 w(2j), f64 w(2j+1)
//
// loc(v) = (first block << 4) | deg(v) for deg <= 8, (block << 4) | 15 for a
// row kept in H's overflow pool (one block {deg, ext, 0, 0 | 0}). Every entry
// carries its neighbour's loc, so a walker steps from row to row with ONE
// dependent fetch -- the next row's address and size come with the sampled
// entry -- and only a walker's start vertex is looked up in the per-vertex
// loc table.
//
// Maintenance: H's mutators flag every row they touch (mark_dirty,
// dyg_internal.cuh). Before a reach walk, k_img_sync (one cooperative launch)
// (A) lists the flagged rows and gives each its new loc -- in place, or in
// freshly allocated blocks when it outgrew them (a bump allocator); (B)
// rewrites their records; (C) patches the copies of a changed loc held by
// unflagged neighbours (a flagged neighbour was rewritten in B); (D) clears
// the flags. Should the blocks run out, the same launch rebuilds the whole
// image contiguously from H's slabs; the host only keeps the pool larger than
// any compact image can be. Snapshots copy the image with H.
#pragma once

#include <stdint.h>

#include "graph_store.cuh"

namespace dyg {

constexpr uint32_t kImgMaxInline = 8;  // entries held in blocks; more -> H's pool
constexpr uint32_t kLocPool = 15;      // loc degree code of a pool row

struct WalkImage {
  const uint32_t* loc;  // per vertex (start vertices only)
  const uint4* rec;     // 32 B blocks as uint4 pairs
};

__host__ __device__ inline uint32_t image_blocks(uint32_t deg) {
  return deg > kImgMaxInline ? 1u : (deg < 2 ? 1u : (deg + 1) / 2);
}
__host__ __device__ inline uint32_t loc_code(uint32_t deg) {
  return deg > kImgMaxInline ? kLocPool : deg;
}
__host__ __device__ inline uint32_t make_loc(uint64_t block, uint32_t deg) {
  return static_cast<uint32_t>(block << 4) | loc_code(deg);
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
  // Brings the image up to date with H's flagged rows (enqueued, capturable;
  // rebuilds in place when the block pool runs out). Returns the number of
  // kernels launched.
  int sync(const DevGraph<kCapH>& h, cudaStream_t st);
  // Before enqueueing work after which H may hold up to h_edges_bound
  // edges: guarantees a rebuild always fits (grows and rebuilds otherwise;
  // never inside a capture).
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
  uint32_t* list_ = nullptr;   // flagged rows of the current sync
  uint4* rec_ = nullptr;
  unsigned long long* ctr_ = nullptr;  // device: [0] blocks handed out, [1] overflow, [2] listed
  unsigned long long* sums_ = nullptr; // rebuild scan scratch (one per sync block)
  uint64_t cap_ = 0;                   // blocks
  int grid_ = 0;                       // sync blocks (all co-resident)
  bool built_ = false;
};

}  // namespace dyg
