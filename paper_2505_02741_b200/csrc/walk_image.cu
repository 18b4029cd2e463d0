// walk_image.cu -- build, incremental sync and snapshots of the compact walk
// image of H (layout and rationale: walk_image.cuh).
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include <algorithm>

#include "walk_image.cuh"

namespace cg = cooperative_groups;

namespace dyg {

namespace {

constexpr unsigned kFullMask = 0xFFFFFFFFu;

unsigned grid_of(uint64_t n, unsigned bs = 256) {
  return static_cast<unsigned>(std::min<uint64_t>((n + bs - 1) / bs, 148ull * 64));
}

// Row v of H as image blocks at `block`: entries in row order, each with its
// neighbour's current loc.
__device__ void write_record(const DevGraph<kCapH>& h, uint32_t v, uint4* rec, uint64_t block,
                             const uint32_t* loc) {
  const RowRef<kCapH> r = row(h, v);
  const uint32_t d = r.deg();
  uint4* out = rec + 2 * block;
  if (d > kImgMaxInline) {
    out[0] = make_uint4(d, r.s->ext, 0u, 0u);
    out[1] = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  const uint32_t nb = image_blocks(d);
  for (uint32_t j = 0; j < nb; ++j) {
    const uint32_t i0 = 2 * j, i1 = 2 * j + 1;
    const uint32_t id0 = i0 < d ? r.id(i0) : 0u, id1 = i1 < d ? r.id(i1) : 0u;
    const uint32_t l0 = i0 < d ? loc[id0] : 0u, l1 = i1 < d ? loc[id1] : 0u;
    const double w0 = i0 < d ? r.w(i0) : 0.0, w1 = i1 < d ? r.w(i1) : 0.0;
    const unsigned long long b0 = __double_as_longlong(w0), b1 = __double_as_longlong(w1);
    out[2 * j] = make_uint4(id0, id1, l0, l1);
    out[2 * j + 1] = make_uint4(static_cast<uint32_t>(b0), static_cast<uint32_t>(b0 >> 32),
                                static_cast<uint32_t>(b1), static_cast<uint32_t>(b1 >> 32));
  }
}

__global__ void k_img_blocks(DevGraph<kCapH> h, unsigned long long* blocks) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < h.n; v += gridDim.x * blockDim.x)
    blocks[v] = image_blocks(h.slab[v].deg);
}

__global__ void k_img_loc_all(DevGraph<kCapH> h, const unsigned long long* __restrict__ base,
                              uint32_t* loc, uint8_t* alloc) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < h.n; v += gridDim.x * blockDim.x) {
    const uint32_t d = h.slab[v].deg;
    loc[v] = make_loc(base[v], d);
    alloc[v] = static_cast<uint8_t>(image_blocks(d));
  }
}

__global__ void k_img_write_all(DevGraph<kCapH> h, const uint32_t* __restrict__ loc,
                                uint8_t* dirty, uint4* rec) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < h.n; v += gridDim.x * blockDim.x) {
    write_record(h, v, rec, loc[v] >> 4, loc);
    dirty[v] = 0;
  }
}

struct ImgDev {
  uint32_t* loc;
  uint8_t* alloc;
  uint8_t* dirty;
  uint32_t* list;
  uint4* rec;
  unsigned long long* ctr;    // [0] blocks handed out, [1] overflow, [2] listed rows
  unsigned long long* sums;   // per-block scratch of the rebuild scan
  unsigned long long cap;
};

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// The whole image rebuilt contiguously from H's slabs (the block pool ran
// out). Block b owns vertices [lo, hi), thread t of it a contiguous
// sub-range; a grid-wide scan of the block counts places the rows.
__device__ void rebuild_all(const DevGraph<kCapH>& h, const ImgDev& d, cg::grid_group& grid) {
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
    d.loc[v] = make_loc(at, deg);
    d.alloc[v] = static_cast<uint8_t>(image_blocks(deg));
    at += image_blocks(deg);
  }
  grid.sync();
  for (uint32_t v = tlo; v < thi; ++v) {
    write_record(h, v, d.rec, d.loc[v] >> 4, d.loc);
    d.dirty[v] = 0;
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long total = 0;
    for (uint32_t b = 0; b < gridDim.x; ++b) total += d.sums[b];
    d.ctr[0] = total;
    d.ctr[1] = 0;
    d.ctr[2] = 0;
  }
}

// Block-wide exclusive sum of x (blockDim.x == 512); *total receives the sum.
__device__ __forceinline__ uint32_t block_exclusive(uint32_t x, uint32_t* total) {
  __shared__ uint32_t s_warp[16];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFullMask, inc, o);
    if (lane >= static_cast<uint32_t>(o)) inc += y;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  uint32_t before = 0, sum = 0;
  for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
    const uint32_t t = s_warp[w];
    before += w < wid ? t : 0u;
    sum += t;
  }
  __syncthreads();
  *total = sum;
  return before + inc - x;
}

// One cooperative launch: the passes A-D of walk_image.cuh. Flag values:
// 1 = row changed, 2 = row changed and its loc moved.
__global__ void __launch_bounds__(512) k_img_sync(DevGraph<kCapH> h, ImgDev d) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ unsigned long long s_first;
  // (A) new loc for every flagged row (and blocks when it outgrew its own;
  // one allocation per block and iteration).
  const uint32_t rounds = (h.n + stride - 1) / stride;
  for (uint32_t it = 0; it < rounds; ++it) {
    const uint32_t v = it * stride + gtid;
    const bool flagged = v < h.n && d.dirty[v] != 0;
    uint32_t deg = 0, grow = 0;
    if (flagged) {
      deg = h.slab[v].deg;
      const uint32_t need = image_blocks(deg);
      grow = need > d.alloc[v] ? need : 0;
    }
    uint32_t total;
    const uint32_t off = block_exclusive(grow, &total);
    if (threadIdx.x == 0)
      s_first = total ? atomicAdd(d.ctr, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    const unsigned long long first = s_first;
    __syncthreads();
    if (!flagged) continue;
    uint64_t block = d.loc[v] >> 4;
    if (grow) {
      if (first + total > d.cap) {
        atomicOr(d.ctr + 1, 1ull);  // out of blocks: rebuilt below
        continue;
      }
      block = first + off;
      d.alloc[v] = static_cast<uint8_t>(grow);
    }
    const uint32_t nl = make_loc(block, deg);
    if (nl != d.loc[v]) d.dirty[v] = 2;
    d.loc[v] = nl;
  }
  grid.sync();
  if (vload(d.ctr + 1) != 0) {  // uniform: read after the grid barrier
    rebuild_all(h, d, grid);
    return;
  }
  // (B) rewrite the flagged rows (their neighbours' locs are final now).
  for (uint32_t v = gtid; v < h.n; v += stride)
    if (d.dirty[v]) write_record(h, v, d.rec, d.loc[v] >> 4, d.loc);
  grid.sync();
  // (C) an unflagged neighbour y holds the old loc of a moved row v in its
  // record (its row is unchanged, so it has the entry): patch it.
  for (uint32_t v = gtid; v < h.n; v += stride) {
    if (d.dirty[v] != 2) continue;
    const uint32_t lv = d.loc[v];
    const RowRef<kCapH> r = row(h, v);
    const uint32_t deg = r.deg();
    for (uint32_t k = 0; k < deg; ++k) {
      const uint32_t y = r.id(k);
      if (d.dirty[y]) continue;
      const uint32_t ly = d.loc[y];
      const uint32_t dy = ly & 15u;
      if (dy == kLocPool) continue;  // pool rows hold ids only
      uint32_t* words = reinterpret_cast<uint32_t*>(d.rec + 2ull * (ly >> 4));
      for (uint32_t j = 0; j < dy; ++j)
        if (words[8 * (j >> 1) + (j & 1)] == v) {
          words[8 * (j >> 1) + 2 + (j & 1)] = lv;
          break;
        }
    }
  }
  grid.sync();
  // (D) clear the flags.
  for (uint32_t v = gtid; v < h.n; v += stride)
    if (d.dirty[v]) d.dirty[v] = 0;
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
  cudaFree(list_);
  cudaFree(rec_);
  cudaFree(ctr_);
  cudaFree(sums_);
  loc_ = nullptr;
  alloc_ = nullptr;
  dirty_ = nullptr;
  list_ = nullptr;
  rec_ = nullptr;
  ctr_ = nullptr;
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
    cuda_check(cudaMalloc(&list_, sizeof(uint32_t) * m), "image list");
    cuda_check(cudaMalloc(&ctr_, 3 * sizeof(unsigned long long)), "image counters");
    cuda_check(cudaMemset(ctr_, 0, 3 * sizeof(unsigned long long)), "image counters");
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_img_sync, 512, 0);
    grid_ = sms * (per_sm > 0 ? std::min(per_sm, 2) : 1);
    cuda_check(cudaMalloc(&sums_, sizeof(unsigned long long) * grid_), "image scan");
  }
  if (cap_blocks > cap_) {
    // The loc encoding holds 28 bits of block index.
    if (cap_blocks >= (1ull << 28)) throw DeviceError{4, "walk image too large"};
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
  // Room for rows that outgrow their blocks between rebuilds, and at least
  // what any compact image of this H can need (ensure_capacity).
  allocate(n, std::max<uint64_t>(cap_, total + std::max<uint64_t>(total, 2ull * n) + 64));
  k_img_loc_all<<<grid_of(n), 256, 0, st>>>(h, base, loc_, alloc_);
  k_img_write_all<<<grid_of(n), 256, 0, st>>>(h, loc_, dirty_, rec_);
  const unsigned long long init[3] = {total, 0ull, 0ull};
  cuda_check(cudaMemcpyAsync(ctr_, init, sizeof init, cudaMemcpyHostToDevice, st), "image top");
  cuda_check(cudaGetLastError(), "image build");
  cuda_check(cudaStreamSynchronize(st), "image build");
  cudaFree(d_temp);
  cudaFree(blocks);
  cudaFree(base);
  built_ = true;
}

int WalkImageStore::sync(const DevGraph<kCapH>& h, cudaStream_t st) {
  ImgDev d{loc_, alloc_, dirty_, list_, rec_, ctr_, sums_, cap_};
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
  // much room k_img_sync can always rebuild in place.
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
  cuda_check(cudaMemcpyAsync(ctr_, o.ctr_, 3 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToDevice, st), "image copy");
  cuda_check(cudaMemsetAsync(dirty_, 0, n, st), "image copy");
  k_img_copy<<<148 * 4, 256, 0, st>>>(o.ctr_, o.rec_, rec_);
  cuda_check(cudaGetLastError(), "image copy");
  built_ = o.built_;
}

}  // namespace dyg
