// walk_image.cu -- build, incremental sync and snapshots of the compact walk
// image of H (layout and rationale: walk_image.cuh).
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include <algorithm>

#include "walk_image.cuh"

namespace cg = cooperative_groups;

namespace dyg {

namespace {

unsigned grid_of(uint64_t n, unsigned bs = 256) {
  return static_cast<unsigned>(std::min<uint64_t>((n + bs - 1) / bs, 148ull * 64));
}

// Row v of H as image blocks at `block` (entries in row order).
__device__ void write_record(const DevGraph<kCapH>& h, uint32_t v, uint4* rec, uint64_t block) {
  const RowRef<kCapH> r = row(h, v);
  const uint32_t d = r.deg();
  uint4* out = rec + 2 * block;
  if (d > kImgMaxInline) {
    out[0] = make_uint4(d, 0u, 0u, r.s->ext);
    out[1] = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  const uint32_t nb = image_blocks(d);
  for (uint32_t j = 0; j < nb; ++j) {
    const uint32_t i0 = 2 * j, i1 = 2 * j + 1;
    const uint32_t id0 = i0 < d ? r.id(i0) : 0u, id1 = i1 < d ? r.id(i1) : 0u;
    const double w0 = i0 < d ? r.w(i0) : 0.0, w1 = i1 < d ? r.w(i1) : 0.0;
    const unsigned long long b0 = __double_as_longlong(w0), b1 = __double_as_longlong(w1);
    out[2 * j] = j == 0 ? make_uint4(d, id0, id1, 0u) : make_uint4(id0, id1, 0u, 0u);
    out[2 * j + 1] = make_uint4(static_cast<uint32_t>(b0), static_cast<uint32_t>(b0 >> 32),
                                static_cast<uint32_t>(b1), static_cast<uint32_t>(b1 >> 32));
  }
}

__global__ void k_img_blocks(DevGraph<kCapH> h, unsigned long long* blocks) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < h.n; v += gridDim.x * blockDim.x)
    blocks[v] = image_blocks(h.slab[v].deg);
}

__global__ void k_img_write_all(DevGraph<kCapH> h, const unsigned long long* __restrict__ base,
                                uint32_t* loc, uint8_t* alloc, uint8_t* dirty, uint4* rec) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < h.n; v += gridDim.x * blockDim.x) {
    const uint32_t d = h.slab[v].deg;
    write_record(h, v, rec, base[v]);
    loc[v] = static_cast<uint32_t>(base[v] << 3) | image_fetch(d);
    alloc[v] = static_cast<uint8_t>(image_blocks(d));
    dirty[v] = 0;
  }
}

struct ImgDev {
  uint32_t* loc;
  uint8_t* alloc;
  uint8_t* dirty;
  uint4* rec;
  unsigned long long* top;    // [0] blocks handed out, [1] overflow flag
  unsigned long long* sums;   // per-block scratch of the compaction scan
  unsigned long long cap;
};

// The flagged rows: rewritten in place, or in new blocks when they outgrew
// their allocation (one atomic per warp). Should the block pool run out, the
// whole image is compacted in the same launch: every row rewritten
// contiguously from H's slabs (a grid-wide scan of the block counts), so the
// image is always complete when the walk starts. Cooperative launch.
__global__ void __launch_bounds__(512) k_img_sync(DevGraph<kCapH> h, ImgDev d) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < h.n; base += stride) {
    const uint32_t v = base + threadIdx.x;
    const bool flagged = v < h.n && d.dirty[v] != 0;
    if (!__any_sync(0xFFFFFFFFu, flagged)) continue;
    uint32_t deg = 0, need = 0, grow = 0;
    if (flagged) {
      d.dirty[v] = 0;
      deg = h.slab[v].deg;
      need = image_blocks(deg);
      grow = need > d.alloc[v] ? need : 0;
    }
    uint32_t off = grow;  // inclusive warp prefix of the grown rows' blocks
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, off, o);
      if (lane >= static_cast<uint32_t>(o)) off += x;
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, off, 31);
    unsigned long long first = 0;
    if (lane == 31 && total) first = atomicAdd(d.top, static_cast<unsigned long long>(total));
    first = __shfl_sync(0xFFFFFFFFu, first, 31);
    if (!flagged) continue;
    if (grow && first + total > d.cap) {
      atomicOr(d.top + 1, 1ull);  // out of blocks: compacted below
      continue;
    }
    uint64_t block;
    if (grow) {
      block = first + off - grow;
      d.alloc[v] = static_cast<uint8_t>(need);
    } else {
      block = d.loc[v] >> 3;
    }
    write_record(h, v, d.rec, block);
    d.loc[v] = static_cast<uint32_t>(block << 3) | image_fetch(deg);
  }
  grid.sync();
  const bool overflow = *reinterpret_cast<volatile unsigned long long*>(d.top + 1) != 0;
  if (!overflow) return;  // uniform: read after the grid barrier
  // Compaction: block b owns vertices [lo, hi), thread t of it the
  // contiguous sub-range [tlo, thi).
  __shared__ unsigned long long s_scan[512];
  const uint32_t per_block = (h.n + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = min(h.n, blockIdx.x * per_block), hi = min(h.n, lo + per_block);
  const uint32_t per_thread = (hi - lo + blockDim.x - 1) / blockDim.x;
  const uint32_t tlo = min(hi, lo + threadIdx.x * per_thread), thi = min(hi, tlo + per_thread);
  unsigned long long mine = 0;
  for (uint32_t v = tlo; v < thi; ++v) mine += image_blocks(h.slab[v].deg);
  s_scan[threadIdx.x] = mine;
  __syncthreads();
  for (uint32_t o = 1; o < blockDim.x; o <<= 1) {  // inclusive block scan
    const unsigned long long x = threadIdx.x >= o ? s_scan[threadIdx.x - o] : 0ull;
    __syncthreads();
    s_scan[threadIdx.x] += x;
    __syncthreads();
  }
  if (threadIdx.x == blockDim.x - 1) d.sums[blockIdx.x] = s_scan[threadIdx.x];
  grid.sync();
  unsigned long long at = 0;
  for (uint32_t b = 0; b < blockIdx.x; ++b) at += d.sums[b];
  at += s_scan[threadIdx.x] - mine;
  for (uint32_t v = tlo; v < thi; ++v) {
    const uint32_t deg = h.slab[v].deg;
    write_record(h, v, d.rec, at);
    d.loc[v] = static_cast<uint32_t>(at << 3) | image_fetch(deg);
    d.alloc[v] = static_cast<uint8_t>(image_blocks(deg));
    d.dirty[v] = 0;
    at += image_blocks(deg);
  }
  grid.sync();
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) {
    unsigned long long total = 0;
    for (uint32_t b = 0; b < gridDim.x; ++b) total += d.sums[b];
    d.top[0] = total;  // the compact image's size
    d.top[1] = 0;
  }
}

__global__ void k_img_copy(const unsigned long long* __restrict__ top, const uint4* __restrict__ src,
                           uint4* dst) {
  const unsigned long long n = 2ull * *top;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

WalkImageStore::~WalkImageStore() { release(); }

void WalkImageStore::release() {
  cudaFree(loc_);
  cudaFree(alloc_);
  cudaFree(dirty_);
  cudaFree(rec_);
  cudaFree(top_);
  cudaFree(sums_);
  loc_ = nullptr;
  alloc_ = nullptr;
  dirty_ = nullptr;
  rec_ = nullptr;
  top_ = nullptr;
  sums_ = nullptr;
  n_ = 0;
  cap_ = 0;
  built_ = false;
}

void WalkImageStore::allocate(uint32_t n, uint64_t cap_blocks) {
  // The flag array is handed to H (GraphStore::set_dirty): it is kept when
  // only the block pool grows.
  if (n_ != n || dirty_ == nullptr) {
    release();
    n_ = n;
    const size_t m = std::max<size_t>(n, 1);
    cuda_check(cudaMalloc(&loc_, sizeof(uint32_t) * m), "image loc");
    cuda_check(cudaMalloc(&alloc_, m), "image alloc");
    cuda_check(cudaMalloc(&dirty_, m), "image flags");
    cuda_check(cudaMemset(dirty_, 0, m), "image flags");
    cuda_check(cudaMalloc(&top_, 2 * sizeof(unsigned long long)), "image top");
    cuda_check(cudaMemset(top_, 0, 2 * sizeof(unsigned long long)), "image top");
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_img_sync, 512, 0);
    grid_ = sms * (per_sm > 0 ? std::min(per_sm, 2) : 1);
    cuda_check(cudaMalloc(&sums_, sizeof(unsigned long long) * grid_), "image scan");
  }
  if (cap_blocks > cap_) {
    cudaFree(rec_);
    rec_ = nullptr;
    cuda_check(cudaMalloc(&rec_, 32ull * cap_blocks), "image blocks");
    cap_ = cap_blocks;
  }
}

void WalkImageStore::build(const DevGraph<kCapH>& h, cudaStream_t st) {
  const uint32_t n = h.n;
  unsigned long long* blocks = nullptr;
  unsigned long long* base = nullptr;
  cuda_check(cudaMalloc(&blocks, sizeof(unsigned long long) * (n + 1ull)), "image scan");
  cuda_check(cudaMalloc(&base, sizeof(unsigned long long) * (n + 1ull)), "image scan");
  cuda_check(cudaMemsetAsync(blocks + n, 0, sizeof(unsigned long long), st), "image scan");
  k_img_blocks<<<grid_of(n), 256, 0, st>>>(h, blocks);
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, blocks, base, n + 1, st);
  void* d_temp = nullptr;
  cuda_check(cudaMalloc(&d_temp, std::max<size_t>(temp, 1)), "image scan");
  cub::DeviceScan::ExclusiveSum(d_temp, temp, blocks, base, n + 1, st);
  unsigned long long total = 0;
  cuda_check(cudaMemcpyAsync(&total, base + n, sizeof total, cudaMemcpyDeviceToHost, st),
             "image size");
  cuda_check(cudaStreamSynchronize(st), "image size");
  // Room for rows that outgrow their blocks between compactions, and at
  // least what any compact image of this H can need (ensure_capacity).
  allocate(n, std::max<uint64_t>(cap_, total + std::max<uint64_t>(total, 2ull * n) + 64));
  k_img_write_all<<<grid_of(n), 256, 0, st>>>(h, base, loc_, alloc_, dirty_, rec_);
  const unsigned long long init[2] = {total, 0ull};
  cuda_check(cudaMemcpyAsync(top_, init, sizeof init, cudaMemcpyHostToDevice, st), "image top");
  cuda_check(cudaGetLastError(), "image build");
  cuda_check(cudaStreamSynchronize(st), "image build");
  cudaFree(d_temp);
  cudaFree(blocks);
  cudaFree(base);
  built_ = true;
}

int WalkImageStore::sync(const DevGraph<kCapH>& h, cudaStream_t st) {
  ImgDev d{loc_, alloc_, dirty_, rec_, top_, sums_, cap_};
  DevGraph<kCapH> hv = h;
  void* args[] = {&hv, &d};
  cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_img_sync), dim3(grid_),
                                         dim3(512), args, 0, st),
             "image sync");
  return 1;
}

void WalkImageStore::ensure_capacity(const DevGraph<kCapH>& h, uint64_t h_edges_bound,
                                     cudaStream_t st) {
  // A compact image needs sum(max(1, ceil(deg / 2))) <= |E_H| + n blocks
  // (2|E_H| entries, two per block, plus one block per row), so with that
  // much room k_img_sync can always compact in place.
  const uint64_t bound = h_edges_bound + n_ + 64;
  if (bound <= cap_) return;
  allocate(n_, 2 * bound);
  build(h, st);
}

void WalkImageStore::copy_from(const WalkImageStore& o, cudaStream_t st) {
  allocate(o.n_, o.cap_);
  const size_t n = o.n_;
  cuda_check(cudaMemcpyAsync(loc_, o.loc_, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st),
             "image copy");
  cuda_check(cudaMemcpyAsync(alloc_, o.alloc_, n, cudaMemcpyDeviceToDevice, st), "image copy");
  cuda_check(cudaMemcpyAsync(top_, o.top_, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToDevice, st), "image copy");
  cuda_check(cudaMemsetAsync(dirty_, 0, n, st), "image copy");
  k_img_copy<<<148 * 4, 256, 0, st>>>(o.top_, o.rec_, rec_);
  cuda_check(cudaGetLastError(), "image copy");
  built_ = o.built_;
}

}  // namespace dyg
