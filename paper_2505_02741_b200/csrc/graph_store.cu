// graph_store.cu -- device dynamic rows: build from a reference-order CSR,
// export back in row order, D2D copies (walk shadow / snapshots), pool growth.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "graph_store.cuh"

namespace dyg {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw DeviceError{4, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

namespace {

// Overflow-block capacity for a row of degree d > C at build time.
template <int C>
__host__ __device__ inline uint32_t initial_cap(uint64_t d) {
  uint64_t c = d + d / 2;
  c = (c + 7) & ~7ull;
  const uint64_t lo = 2 * C < 8 ? 8 : 2 * C;
  return static_cast<uint32_t>(c < lo ? lo : c);
}

template <int C>
__global__ void k_build(DevGraph<C> g, const uint64_t* __restrict__ rp,
                        const uint32_t* __restrict__ ids, const double* __restrict__ w) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= g.n) return;
  const uint64_t b = rp[u];
  const uint32_t d = static_cast<uint32_t>(rp[u + 1] - b);
  Slab<C>& s = g.slab[u];
  s.deg = d;
  if (d <= C) {
    s.ext = kInline;
    g.cap[u] = 0;
    for (uint32_t i = 0; i < d; ++i) {
      s.idr(i) = ids[b + i];
      s.wr(i) = w[b + i];
    }
    return;
  }
  const uint32_t c = initial_cap<C>(d);
  const unsigned long long at = atomicAdd(g.pool_top, static_cast<unsigned long long>(c));
  s.ext = static_cast<uint32_t>(at);
  g.cap[u] = c;
  for (uint32_t i = 0; i < d; ++i) {
    g.pool_id[at + i] = ids[b + i];
    g.pool_w[at + i] = w[b + i];
  }
}

template <int C>
__global__ void k_degrees(DevGraph<C> g, uint64_t* deg) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < g.n) deg[u] = g.slab[u].deg;
}

template <int C>
__global__ void k_gather(DevGraph<C> g, const uint64_t* __restrict__ rp, uint32_t* ids,
                         double* w) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= g.n) return;
  const RowRef<C> r = row(g, u);
  const uint32_t d = r.deg();
  const uint64_t b = rp[u];
  for (uint32_t i = 0; i < d; ++i) {
    ids[b + i] = r.id(i);
    w[b + i] = r.w(i);
  }
}

// Pool copy of [0, *top) with the bound read on the device.
__global__ void k_copy_pool(const unsigned long long* __restrict__ top,
                            const uint32_t* __restrict__ src_id,
                            const double* __restrict__ src_w, uint32_t* dst_id, double* dst_w) {
  const unsigned long long n = *top;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    dst_id[i] = src_id[i];
    dst_w[i] = src_w[i];
  }
}

unsigned grid_for(uint64_t n, unsigned bs = 256) {
  return static_cast<unsigned>((n + bs - 1) / bs);
}

}  // namespace

template <int C>
GraphStore<C>::~GraphStore() {
  release();
}

template <int C>
void GraphStore<C>::release() {
  cudaFree(v_.slab);
  cudaFree(v_.cap);
  cudaFree(v_.pool_id);
  cudaFree(v_.pool_w);
  cudaFree(counters_);
  v_ = DevGraph<C>{};
  counters_ = nullptr;
}

template <int C>
void GraphStore<C>::allocate(uint32_t n, uint64_t pool_cap) {
  release();
  v_.n = n;
  v_.pool_cap = pool_cap;
  cuda_check(cudaMalloc(&v_.slab, sizeof(Slab<C>) * static_cast<size_t>(n)), "alloc slabs");
  cuda_check(cudaMalloc(&v_.cap, sizeof(uint32_t) * static_cast<size_t>(n)), "alloc caps");
  cuda_check(cudaMalloc(&v_.pool_id, sizeof(uint32_t) * pool_cap), "alloc pool ids");
  cuda_check(cudaMalloc(&v_.pool_w, sizeof(double) * pool_cap), "alloc pool weights");
  cuda_check(cudaMalloc(&counters_, 2 * sizeof(unsigned long long)), "alloc counters");
  v_.pool_top = counters_;
  v_.edges = counters_ + 1;
}

template <int C>
void GraphStore<C>::upload(uint32_t n, const uint64_t* row_ptr, const uint32_t* ids,
                           const double* w, cudaStream_t st) {
  const uint64_t nnz = row_ptr[n];
  uint64_t ext = 0;
  for (uint32_t u = 0; u < n; ++u) {
    const uint64_t d = row_ptr[u + 1] - row_ptr[u];
    if (d > C) ext += initial_cap<C>(d);
  }
  const uint64_t pool_cap = ext + std::max<uint64_t>(nnz, 1ull << 20);
  allocate(n, pool_cap);
  uint64_t* d_rp = nullptr;
  uint32_t* d_ids = nullptr;
  double* d_w = nullptr;
  cuda_check(cudaMalloc(&d_rp, sizeof(uint64_t) * (n + 1ull)), "alloc staging");
  cuda_check(cudaMalloc(&d_ids, sizeof(uint32_t) * std::max<uint64_t>(nnz, 1)), "alloc staging");
  cuda_check(cudaMalloc(&d_w, sizeof(double) * std::max<uint64_t>(nnz, 1)), "alloc staging");
  cuda_check(cudaMemcpyAsync(d_rp, row_ptr, sizeof(uint64_t) * (n + 1ull),
                             cudaMemcpyHostToDevice, st), "upload row_ptr");
  if (nnz) {
    cuda_check(cudaMemcpyAsync(d_ids, ids, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, st),
               "upload ids");
    cuda_check(cudaMemcpyAsync(d_w, w, sizeof(double) * nnz, cudaMemcpyHostToDevice, st),
               "upload weights");
  }
  cuda_check(cudaMemsetAsync(v_.slab, 0, sizeof(Slab<C>) * static_cast<size_t>(n), st), "memset");
  const unsigned long long init[2] = {0ull, nnz / 2};
  cuda_check(cudaMemcpyAsync(counters_, init, sizeof(init), cudaMemcpyHostToDevice, st),
             "init counters");
  k_build<C><<<grid_for(n), 256, 0, st>>>(v_, d_rp, d_ids, d_w);
  cuda_check(cudaGetLastError(), "k_build");
  cuda_check(cudaStreamSynchronize(st), "build graph");
  cudaFree(d_rp);
  cudaFree(d_ids);
  cudaFree(d_w);
}

template <int C>
void GraphStore<C>::copy_from(const GraphStore& o, cudaStream_t st) {
  if (!allocated() || v_.n != o.v_.n || v_.pool_cap < o.v_.pool_cap) {
    allocate(o.v_.n, o.v_.pool_cap);
  }
  const size_t n = v_.n;
  cuda_check(cudaMemcpyAsync(v_.slab, o.v_.slab, sizeof(Slab<C>) * n, cudaMemcpyDeviceToDevice, st),
             "copy slabs");
  cuda_check(cudaMemcpyAsync(v_.cap, o.v_.cap, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st),
             "copy caps");
  cuda_check(cudaMemcpyAsync(counters_, o.counters_, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToDevice, st), "copy counters");
  k_copy_pool<<<148 * 4, 256, 0, st>>>(o.v_.pool_top, o.v_.pool_id, o.v_.pool_w, v_.pool_id,
                                       v_.pool_w);
  cuda_check(cudaGetLastError(), "k_copy_pool");
}

template <int C>
uint64_t GraphStore<C>::export_rows(uint64_t* row_ptr, uint32_t* ids, double* w,
                                    uint64_t capacity, cudaStream_t st) {
  const uint32_t n = v_.n;
  uint64_t* d_rp = nullptr;
  cuda_check(cudaMalloc(&d_rp, sizeof(uint64_t) * (n + 1ull)), "alloc export");
  cuda_check(cudaMemsetAsync(d_rp, 0, sizeof(uint64_t), st), "memset");
  uint64_t* d_deg = nullptr;
  cuda_check(cudaMalloc(&d_deg, sizeof(uint64_t) * n), "alloc export");
  k_degrees<C><<<grid_for(n), 256, 0, st>>>(v_, d_deg);
  size_t temp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, temp, d_deg, d_rp + 1, n, st);
  void* d_temp = nullptr;
  cuda_check(cudaMalloc(&d_temp, std::max<size_t>(temp, 1)), "alloc scan");
  cub::DeviceScan::InclusiveSum(d_temp, temp, d_deg, d_rp + 1, n, st);
  cuda_check(cudaMemcpyAsync(row_ptr, d_rp, sizeof(uint64_t) * (n + 1ull),
                             cudaMemcpyDeviceToHost, st), "download row_ptr");
  cuda_check(cudaStreamSynchronize(st), "export");
  const uint64_t nnz = row_ptr[n];
  if (nnz <= capacity && nnz > 0) {
    uint32_t* d_ids = nullptr;
    double* d_w = nullptr;
    cuda_check(cudaMalloc(&d_ids, sizeof(uint32_t) * nnz), "alloc export");
    cuda_check(cudaMalloc(&d_w, sizeof(double) * nnz), "alloc export");
    k_gather<C><<<grid_for(n), 256, 0, st>>>(v_, d_rp, d_ids, d_w);
    cuda_check(cudaMemcpyAsync(ids, d_ids, sizeof(uint32_t) * nnz, cudaMemcpyDeviceToHost, st),
               "download ids");
    cuda_check(cudaMemcpyAsync(w, d_w, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st),
               "download weights");
    cuda_check(cudaStreamSynchronize(st), "export");
    cudaFree(d_ids);
    cudaFree(d_w);
  }
  cudaFree(d_temp);
  cudaFree(d_deg);
  cudaFree(d_rp);
  return nnz;
}

template <int C>
void GraphStore<C>::ensure_pool(uint64_t top, uint64_t free_entries, cudaStream_t st) {
  if (v_.pool_cap >= top + free_entries) return;
  const uint64_t cap = std::max<uint64_t>(2 * v_.pool_cap, top + 2 * free_entries);
  uint32_t* nid = nullptr;
  double* nw = nullptr;
  cuda_check(cudaMalloc(&nid, sizeof(uint32_t) * cap), "grow pool");
  cuda_check(cudaMalloc(&nw, sizeof(double) * cap), "grow pool");
  // Copy the whole old capacity, not just `top`: batches already enqueued on
  // `st` may append past the host's last known top before this copy runs.
  (void)top;
  if (v_.pool_cap) {
    cuda_check(cudaMemcpyAsync(nid, v_.pool_id, sizeof(uint32_t) * v_.pool_cap,
                               cudaMemcpyDeviceToDevice, st), "grow pool");
    cuda_check(cudaMemcpyAsync(nw, v_.pool_w, sizeof(double) * v_.pool_cap,
                               cudaMemcpyDeviceToDevice, st), "grow pool");
  }
  cuda_check(cudaStreamSynchronize(st), "grow pool");
  cudaFree(v_.pool_id);
  cudaFree(v_.pool_w);
  v_.pool_id = nid;
  v_.pool_w = nw;
  v_.pool_cap = cap;
}

template class GraphStore<kCapH>;
template class GraphStore<kCapG>;

}  // namespace dyg
