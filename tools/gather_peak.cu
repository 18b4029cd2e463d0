// gather_peak.cu -- random-gather roofline of this B200 (the walk
// kernels are HBM random gathers). Measures (a) independent random row
// fetches of R bytes from a table of S bytes, cooperative cp.async like the
// walk kernels (R/16 lanes per row), and (b) a dependent pointer chase (one
// outstanding fetch per lane) -- the latency floor of one walker step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_peak gather_peak.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

// Each warp fetches `iters` rounds of 32 random rows of RB bytes (row
// stride RB), cooperatively, then consumes one word per row.
template <int RB>
__global__ void k_gather(const uint4* __restrict__ tab, uint64_t nrows, int iters,
                         unsigned long long* sink) {
  constexpr int LPR = RB / 16;             // lanes per row
  constexpr int RPR = 32 / LPR;            // rows per round
  __shared__ uint4 st[8][32 * LPR];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t h = mix(blockIdx.x * 1024ull + threadIdx.x + 12345);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    h = mix(h + 0x9E3779B97F4A7C15ull);
    const uint64_t my = h % nrows;
#pragma unroll
    for (int j = 0; j < 32 / RPR; ++j) {
      const int r = j * RPR + lane / LPR;
      const uint64_t u = __shfl_sync(0xffffffffu, my, r);
      cp16(&st[w][r * LPR + lane % LPR], tab + u * LPR + lane % LPR);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    acc += st[w][lane * LPR].x;
    __syncwarp();
  }
  if (acc == 0x1234567) *sink = acc;
}

// Pointer chase: next row index = word 0 of the current row.
__global__ void k_chase(const uint4* __restrict__ tab, int LPR, int steps, uint64_t nrows,
                        unsigned long long* sink) {
  uint64_t cur = mix(blockIdx.x * 1024ull + threadIdx.x + 99) % nrows;
  for (int s = 0; s < steps; ++s) cur = tab[cur * LPR].x;
  if (cur == 0x7fffffff) *sink = cur;
}
__global__ void k_fill(uint4* tab, uint64_t nrows, int LPR) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nrows;
       i += (uint64_t)gridDim.x * blockDim.x)
    tab[i * LPR] = make_uint4(static_cast<uint32_t>(mix(i + 7) % nrows), 0, 0, 0);
}

template <int RB>
void run_gather(uint4* tab, uint64_t bytes, int sms, unsigned long long* sink) {
  const uint64_t nrows = bytes / RB;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bps : {2, 4, 8}) {
    const int iters = 400, grid = sms * bps;
    k_gather<RB><<<grid, 256>>>(tab, nrows, 20, sink);
    cudaEventRecord(a);
    k_gather<RB><<<grid, 256>>>(tab, nrows, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double moved = double(grid) * 256 * iters * RB;
    printf("gather row=%3dB table=%5.0fMB blocks/SM=%d : %7.1f GB/s  (%.1f Grows/s)\n", RB,
           bytes / 1e6, bps, moved / ms / 1e6, moved / RB / ms / 1e6);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const uint64_t maxb = 2ull << 30;
  uint4* tab;
  cudaMalloc(&tab, maxb);
  cudaMemset(tab, 0, maxb);
  for (uint64_t mb : {32ull, 268ull, 537ull, 2048ull}) {
    const uint64_t bytes = mb << 20;
    run_gather<32>(tab, bytes, sms, sink);
    run_gather<64>(tab, bytes, sms, sink);
    run_gather<128>(tab, bytes, sms, sink);
  }
  // latency: one lane per warp... use 1 block of 32 threads, and a loaded chase
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (uint64_t mb : {32ull, 537ull}) {
    const uint64_t nrows = (mb << 20) / 64;
    k_fill<<<1024, 256>>>(tab, nrows, 4);
    for (int grid : {1, sms, sms * 8}) {
      const int steps = 2000;
      cudaEventRecord(a);
      k_chase<<<grid, 32>>>(tab, 4, steps, nrows, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("chase table=%4luMB lanes=%6d : %.0f ns per dependent fetch, %.1f GB/s (64B)\n", mb,
             grid * 32, ms * 1e6 / steps, double(grid) * 32 * steps * 64 / ms / 1e6);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
