// init_sparsifier.cu -- the initial sparsifier builder on the device
// (reference build_initial_sparsifier,
// proj/src/sparsifier.cpp:105-159 with TreeResistance :40-101), bit-identical
// to the reference:
//
//   1. G's edges (u < v) sorted by weight descending, then (u, v) ascending
//      (:115-118): two stable radix sorts (pair key, then weight key).
//   2. Kruskal's maximum spanning tree over that order (:120-129). Under a
//      strict total order the MST is unique, so Borůvka rounds (each
//      component takes its lowest-rank outgoing edge) give the same tree.
//   3. H's tree rows get their edges in Kruskal (rank) order, exactly the
//      order the reference's insert_edge calls append them.
//   4. TreeResistance: BFS from vertex 0, resistance_to_root accumulated
//      down each root path in path order (r[child] = r[parent] + 1/w, the
//      reference's left fold), one level per grid barrier of a cooperative
//      kernel; binary-lifting LCA tables as in :66-71 / :79-93.
//   5. Off-tree edges ranked by distortion w * (r[u] + r[v] - 2 r[lca])
//      descending, then hash_mix(seed ^ (u << 32 | v)) ascending (:137-148).
//   6. The fill count (:150-155) is evaluated on the host with the
//      reference's own density arithmetic; the selected edges are appended
//      to their rows in ranked order.
//
// Exactness: every floating-point value is produced by the same operations
// in the same order as the reference (correctly rounded 1.0 / w, the same
// additions along root paths, (a + b) - 2c, one multiply for the
// distortion); sorting keys are total orders on the same values.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "dyg_internal.cuh"
#include "graph_store.cuh"

namespace cg = cooperative_groups;

namespace dyg {

namespace {

unsigned blocks(uint64_t n, unsigned bs = 256) { return static_cast<unsigned>((n + bs - 1) / bs); }

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(uint64_t n) {
    cuda_check(cudaMalloc(&p, sizeof(T) * std::max<uint64_t>(n, 1)), "init sparsifier alloc");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Ascending key of a double's value (total order; -0 < +0 is irrelevant here).
__device__ __forceinline__ unsigned long long asc_key(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// 1. Upper-triangle edges in row order.
__global__ void k_upper_count(uint32_t n, const uint64_t* __restrict__ rp,
                              const uint32_t* __restrict__ ids, uint64_t* cnt) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint64_t c = 0;
  for (uint64_t i = rp[u]; i < rp[u + 1]; ++i) c += ids[i] > u;
  cnt[u] = c;
}

__global__ void k_upper_emit(uint32_t n, const uint64_t* __restrict__ rp,
                             const uint32_t* __restrict__ ids, const double* __restrict__ w,
                             const uint64_t* __restrict__ off, uint32_t* eu, uint32_t* ev,
                             double* ew, unsigned long long* key, uint32_t* idx) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint64_t o = off[u];
  for (uint64_t i = rp[u]; i < rp[u + 1]; ++i) {
    const uint32_t v = ids[i];
    if (v <= u) continue;
    eu[o] = u;
    ev[o] = v;
    ew[o] = w[i];
    key[o] = (static_cast<unsigned long long>(u) << 32) | v;  // (u, v) ascending
    idx[o] = static_cast<uint32_t>(o);
    ++o;
  }
}

__global__ void k_weight_key(uint64_t m, const uint32_t* __restrict__ idx,
                             const double* __restrict__ ew, unsigned long long* key) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < m) key[i] = ~asc_key(ew[idx[i]]);  // weight descending
}

// 2. Borůvka over ranks (rank = position in the sorted order).
__global__ void k_bv_best(uint64_t m, const uint32_t* __restrict__ order,
                          const uint32_t* __restrict__ eu, const uint32_t* __restrict__ ev,
                          const uint32_t* __restrict__ comp, uint32_t* best) {
  const uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  const uint32_t e = order[r];
  const uint32_t cu = comp[eu[e]], cv = comp[ev[e]];
  if (cu == cv) return;
  atomicMin(best + cu, static_cast<uint32_t>(r));
  atomicMin(best + cv, static_cast<uint32_t>(r));
}

__global__ void k_bv_hook(uint32_t n, const uint32_t* __restrict__ order,
                          const uint32_t* __restrict__ eu, const uint32_t* __restrict__ ev,
                          const uint32_t* __restrict__ comp, const uint32_t* __restrict__ best,
                          uint32_t* parent, uint8_t* in_tree, unsigned int* hooked) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n || comp[c] != c || best[c] == 0xFFFFFFFFu) return;
  const uint32_t r = best[c];
  const uint32_t e = order[r];
  const uint32_t cu = comp[eu[e]], cv = comp[ev[e]];
  const uint32_t other = cu == c ? cv : cu;
  in_tree[r] = 1;
  // Mutual choice (the same edge is both components' best): the lower id
  // stays a root.
  if (best[other] == r && c < other) return;
  parent[c] = other;
  atomicAdd(hooked, 1u);
}

__global__ void k_bv_jump(uint32_t n, uint32_t* comp, const uint32_t* __restrict__ parent,
                          unsigned int* changed) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  uint32_t c = parent[comp[v]];
  while (parent[c] != c) c = parent[c];
  if (c != comp[v]) {
    comp[v] = c;
    atomicAdd(changed, 1u);
  }
}

__global__ void k_compress(uint32_t n, uint32_t* parent) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  uint32_t c = parent[v];
  while (parent[c] != c) c = parent[c];
  parent[v] = c;
}

// 3 / 6. Row records (row << 32 | order) -> CSR.
__global__ void k_records(uint64_t m, const uint32_t* __restrict__ sel,
                          const uint32_t* __restrict__ sel_order, uint64_t nsel,
                          const uint32_t* __restrict__ eu, const uint32_t* __restrict__ ev,
                          unsigned long long* key, uint32_t* val) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nsel) return;
  const uint32_t e = sel[i];
  const uint32_t o = sel_order[i];
  key[2 * i] = (static_cast<unsigned long long>(eu[e]) << 32) | o;
  val[2 * i] = e;
  key[2 * i + 1] = (static_cast<unsigned long long>(ev[e]) << 32) | o;
  val[2 * i + 1] = e | 0x80000000u;  // the record lives in row v
  (void)m;
}

__global__ void k_csr_fill(uint64_t nrec, const unsigned long long* __restrict__ key,
                           const uint32_t* __restrict__ val, const uint32_t* __restrict__ eu,
                           const uint32_t* __restrict__ ev, const double* __restrict__ ew,
                           uint32_t* ids, double* w, uint64_t* deg) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nrec) return;
  const uint32_t x = val[i];
  const uint32_t e = x & 0x7FFFFFFFu;
  const bool in_v = (x >> 31) != 0;
  ids[i] = in_v ? eu[e] : ev[e];
  w[i] = ew[e];
  atomicAdd(reinterpret_cast<unsigned long long*>(deg) + (key[i] >> 32), 1ull);
}

// 4. BFS from 0 over the tree rows: one level per grid barrier.
__global__ void k_tree_bfs(uint32_t n, const uint64_t* __restrict__ rp,
                           const uint32_t* __restrict__ ids, const double* __restrict__ w,
                           uint32_t* parent, uint32_t* depth, double* rroot, uint8_t* visited,
                           uint32_t* fa, uint32_t* fb, unsigned int* sizes) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t tid = static_cast<uint32_t>(grid.thread_rank());
  const uint32_t nth = static_cast<uint32_t>(grid.size());
  uint32_t* cur = fa;
  uint32_t* nxt = fb;
  for (uint32_t level = 0;; ++level) {
    const uint32_t cn = sizes[level & 1];
    if (cn == 0) break;
    if (tid == 0) sizes[(level + 1) & 1] = 0;
    grid.sync();
    for (uint32_t i = tid; i < cn; i += nth) {
      const uint32_t u = cur[i];
      for (uint64_t j = rp[u]; j < rp[u + 1]; ++j) {
        const uint32_t v = ids[j];
        if (visited[v]) continue;  // a tree: v is u's child iff unvisited
        visited[v] = 1;
        parent[v] = u;
        depth[v] = depth[u] + 1;
        rroot[v] = __dadd_rn(rroot[u], __ddiv_rn(1.0, w[j]));  // :61
        nxt[atomicAdd(sizes + ((level + 1) & 1), 1u)] = v;
      }
    }
    grid.sync();
    uint32_t* t = cur;
    cur = nxt;
    nxt = t;
  }
}

__global__ void k_lift(uint32_t n, const uint32_t* __restrict__ prev, uint32_t* next) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) next[v] = prev[prev[v]];
}

// 5. Off-tree distortion and tiebreak.
__global__ void k_not(uint64_t m, const uint8_t* __restrict__ x, uint8_t* y) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < m) y[i] = x[i] ? 0 : 1;
}

__global__ void k_rank_keys(uint64_t k, const uint32_t* __restrict__ off_rank,
                            const uint32_t* __restrict__ order, const uint32_t* __restrict__ eu,
                            const uint32_t* __restrict__ ev, const double* __restrict__ ew,
                            const uint32_t* __restrict__ depth, const double* __restrict__ rroot,
                            const uint32_t* const* __restrict__ up, uint32_t levels,
                            uint64_t seed, unsigned long long* dist_key,
                            unsigned long long* tie_key) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= k) return;
  const uint32_t e = order[off_rank[i]];
  const uint32_t a = eu[e], b = ev[e];
  // lca (:79-93)
  uint32_t u = a, v = b;
  if (depth[u] < depth[v]) {
    const uint32_t t = u;
    u = v;
    v = t;
  }
  uint32_t gap = depth[u] - depth[v];
  for (uint32_t lv = 0; gap != 0; ++lv, gap >>= 1)
    if (gap & 1u) u = up[lv][u];
  uint32_t l = u;
  if (u != v) {
    for (uint32_t lv = levels; lv-- > 0;) {
      if (up[lv][u] != up[lv][v]) {
        u = up[lv][u];
        v = up[lv][v];
      }
    }
    l = up[0][u];
  }
  const double between = __dsub_rn(__dadd_rn(rroot[a], rroot[b]), __dmul_rn(2.0, rroot[l]));
  const double distortion = __dmul_rn(ew[e], between);
  dist_key[i] = ~asc_key(distortion);  // descending
  tie_key[i] = hash_mix(seed ^ ((static_cast<uint64_t>(a) << 32) | b));
}

__global__ void k_iota(uint64_t n, uint32_t* x) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = static_cast<uint32_t>(i);
}

__global__ void k_seq(uint64_t n, uint32_t base, uint32_t* x) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = base + static_cast<uint32_t>(i);
}

__global__ void k_gather_u64(uint64_t n, const unsigned long long* __restrict__ src,
                             const uint32_t* __restrict__ idx, unsigned long long* dst) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_gather_u32(uint64_t n, const uint32_t* __restrict__ src,
                             const uint32_t* __restrict__ idx, uint32_t* dst) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

template <typename K, typename V>
void radix_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int begin_bit,
                 int end_bit, cudaStream_t st) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, kin, kout, vin, vout, static_cast<int64_t>(n),
                                  begin_bit, end_bit, st);
  DevBuf<unsigned char> t(temp);
  cuda_check(cub::DeviceRadixSort::SortPairs(t.p, temp, kin, kout, vin, vout,
                                             static_cast<int64_t>(n), begin_bit, end_bit, st),
             "radix sort");
  cuda_check(cudaStreamSynchronize(st), "radix sort");
}

}  // namespace

// Host driver. out buffers: row_ptr[n + 1], ids / w with room for G's nnz.
void build_initial_sparsifier_device(uint32_t n, const uint64_t* h_rp, const uint32_t* h_ids,
                                     const double* h_w, double target_density, uint64_t seed,
                                     uint64_t* o_rp, uint32_t* o_ids, double* o_w) {
  if (target_density < 0.0) throw DeviceError{1, "target density must be nonnegative"};
  cudaStream_t st;
  cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{st};
  const uint64_t nnz = h_rp[n];
  DevBuf<uint64_t> rp(n + 1ull);
  DevBuf<uint32_t> ids(nnz);
  DevBuf<double> w(nnz);
  cuda_check(cudaMemcpyAsync(rp.p, h_rp, sizeof(uint64_t) * (n + 1ull), cudaMemcpyHostToDevice, st),
             "upload");
  cuda_check(cudaMemcpyAsync(ids.p, h_ids, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, st),
             "upload");
  cuda_check(cudaMemcpyAsync(w.p, h_w, sizeof(double) * nnz, cudaMemcpyHostToDevice, st), "upload");

  // 1. edges, sorted (weight desc, (u, v) asc)
  DevBuf<uint64_t> cnt(n), off(n);
  k_upper_count<<<blocks(n), 256, 0, st>>>(n, rp.p, ids.p, cnt.p);
  {
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, cnt.p, off.p, n, st);
    DevBuf<unsigned char> t(temp);
    cuda_check(cub::DeviceScan::ExclusiveSum(t.p, temp, cnt.p, off.p, n, st), "scan");
    cuda_check(cudaStreamSynchronize(st), "scan");
  }
  uint64_t last_off = 0, last_cnt = 0;
  cuda_check(cudaMemcpy(&last_off, off.p + (n - 1), 8, cudaMemcpyDeviceToHost), "m");
  cuda_check(cudaMemcpy(&last_cnt, cnt.p + (n - 1), 8, cudaMemcpyDeviceToHost), "m");
  const uint64_t m = last_off + last_cnt;
  if (m >= 0x7FFFFFFFull) throw DeviceError{1, "graph too large for the device builder"};
  DevBuf<uint32_t> eu(m), ev(m), idx_a(m), idx_b(m);
  DevBuf<double> ew(m);
  DevBuf<unsigned long long> key_a(m), key_b(m);
  k_upper_emit<<<blocks(n), 256, 0, st>>>(n, rp.p, ids.p, w.p, off.p, eu.p, ev.p, ew.p, key_a.p,
                                          idx_a.p);
  radix_pairs(key_a.p, key_b.p, idx_a.p, idx_b.p, m, 0, 64, st);  // (u, v) asc
  k_weight_key<<<blocks(m), 256, 0, st>>>(m, idx_b.p, ew.p, key_a.p);
  radix_pairs(key_a.p, key_b.p, idx_b.p, idx_a.p, m, 0, 64, st);  // stable: weight desc
  uint32_t* order = idx_a.p;  // rank -> edge

  // 2. Borůvka
  DevBuf<uint32_t> comp(n), parent(n), best(n);
  DevBuf<uint8_t> in_tree(m);
  DevBuf<unsigned int> flag(2);
  k_iota<<<blocks(n), 256, 0, st>>>(n, comp.p);
  k_iota<<<blocks(n), 256, 0, st>>>(n, parent.p);
  cuda_check(cudaMemsetAsync(in_tree.p, 0, m, st), "memset");
  for (int round = 0; round < 64; ++round) {
    cuda_check(cudaMemsetAsync(best.p, 0xFF, sizeof(uint32_t) * n, st), "memset");
    cuda_check(cudaMemsetAsync(flag.p, 0, sizeof(unsigned int) * 2, st), "memset");
    k_bv_best<<<blocks(m), 256, 0, st>>>(m, order, eu.p, ev.p, comp.p, best.p);
    k_bv_hook<<<blocks(n), 256, 0, st>>>(n, order, eu.p, ev.p, comp.p, best.p, parent.p,
                                         in_tree.p, flag.p);
    k_compress<<<blocks(n), 256, 0, st>>>(n, parent.p);
    k_bv_jump<<<blocks(n), 256, 0, st>>>(n, comp.p, parent.p, flag.p + 1);
    unsigned int hooked = 0;
    cuda_check(cudaMemcpyAsync(&hooked, flag.p, sizeof hooked, cudaMemcpyDeviceToHost, st), "bv");
    cuda_check(cudaStreamSynchronize(st), "boruvka");
    if (hooked == 0) break;
  }
  // tree edges in rank order
  DevBuf<uint32_t> tree_rank(n), off_rank(m);
  DevBuf<unsigned int> counts(2);
  cuda_check(cudaMemsetAsync(counts.p, 0, 8, st), "memset");
  {
    // selected ranks, compacted in rank order (cub flagged select keeps order)
    DevBuf<uint32_t> ranks(m);
    k_iota<<<blocks(m), 256, 0, st>>>(m, ranks.p);
    size_t temp = 0;
    cub::DeviceSelect::Flagged(nullptr, temp, ranks.p, in_tree.p, tree_rank.p, counts.p,
                               static_cast<int64_t>(m), st);
    DevBuf<unsigned char> t(temp);
    cuda_check(cub::DeviceSelect::Flagged(t.p, temp, ranks.p, in_tree.p, tree_rank.p, counts.p,
                                          static_cast<int64_t>(m), st), "select");
    cuda_check(cudaStreamSynchronize(st), "select");
  }
  unsigned int ntree = 0;
  cuda_check(cudaMemcpy(&ntree, counts.p, 4, cudaMemcpyDeviceToHost), "tree size");
  if (ntree != n - 1) throw DeviceError{2, "graph must be connected to build a sparsifier"};

  // 3. tree rows (for the BFS) in rank order
  auto build_rows = [&](const uint32_t* sel_rank, const uint32_t* sel_order, uint64_t nsel,
                        uint64_t* d_rp, uint32_t* d_ids, double* d_w) {
    const uint64_t nrec = 2 * nsel;
    DevBuf<uint32_t> sel(nsel);
    k_gather_u32<<<blocks(nsel), 256, 0, st>>>(nsel, order, sel_rank, sel.p);
    DevBuf<unsigned long long> k1(nrec), k2(nrec);
    DevBuf<uint32_t> v1(nrec), v2(nrec);
    DevBuf<uint64_t> deg(n);
    cuda_check(cudaMemsetAsync(deg.p, 0, sizeof(uint64_t) * n, st), "memset");
    k_records<<<blocks(nsel), 256, 0, st>>>(m, sel.p, sel_order, nsel, eu.p, ev.p, k1.p, v1.p);
    radix_pairs(k1.p, k2.p, v1.p, v2.p, nrec, 0, 64, st);
    k_csr_fill<<<blocks(nrec), 256, 0, st>>>(nrec, k2.p, v2.p, eu.p, ev.p, ew.p, d_ids, d_w,
                                             deg.p);
    cuda_check(cudaMemsetAsync(d_rp, 0, sizeof(uint64_t), st), "memset");
    size_t temp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, temp, deg.p, d_rp + 1, n, st);
    DevBuf<unsigned char> t(temp);
    cuda_check(cub::DeviceScan::InclusiveSum(t.p, temp, deg.p, d_rp + 1, n, st), "scan");
    cuda_check(cudaStreamSynchronize(st), "rows");
  };
  DevBuf<uint64_t> trp(n + 1ull);
  DevBuf<uint32_t> tids(2ull * (n - 1) + 1);
  DevBuf<double> tw(2ull * (n - 1) + 1);
  build_rows(tree_rank.p, tree_rank.p, ntree, trp.p, tids.p, tw.p);

  // 4. BFS from 0: parent, depth, resistance to the root
  DevBuf<uint32_t> tpar(n), depth(n), fa(n), fb(n);
  DevBuf<double> rroot(n);
  DevBuf<uint8_t> visited(n);
  DevBuf<unsigned int> sizes(2);
  cuda_check(cudaMemsetAsync(tpar.p, 0, sizeof(uint32_t) * n, st), "memset");  // parent(n, 0)
  cuda_check(cudaMemsetAsync(depth.p, 0, sizeof(uint32_t) * n, st), "memset");
  cuda_check(cudaMemsetAsync(rroot.p, 0, sizeof(double) * n, st), "memset");
  cuda_check(cudaMemsetAsync(visited.p, 0, n, st), "memset");
  {
    const uint8_t one = 1;
    const uint32_t zero = 0;
    const unsigned int sz[2] = {1u, 0u};
    cuda_check(cudaMemcpyAsync(visited.p, &one, 1, cudaMemcpyHostToDevice, st), "bfs");
    cuda_check(cudaMemcpyAsync(fa.p, &zero, 4, cudaMemcpyHostToDevice, st), "bfs");
    cuda_check(cudaMemcpyAsync(sizes.p, sz, 8, cudaMemcpyHostToDevice, st), "bfs");
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tree_bfs, 256, 0);
    uint32_t nn = n;
    uint64_t* a0 = trp.p;
    uint32_t* a1 = tids.p;
    double* a2 = tw.p;
    uint32_t* a3 = tpar.p;
    uint32_t* a4 = depth.p;
    double* a5 = rroot.p;
    uint8_t* a6 = visited.p;
    uint32_t* a7 = fa.p;
    uint32_t* a8 = fb.p;
    unsigned int* a9 = sizes.p;
    void* args[] = {&nn, &a0, &a1, &a2, &a3, &a4, &a5, &a6, &a7, &a8, &a9};
    cuda_check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_tree_bfs),
                                           dim3(sms * std::max(per_sm, 1)), dim3(256), args, 0, st),
               "tree bfs");
    cuda_check(cudaStreamSynchronize(st), "tree bfs");
  }
  // binary lifting: levels_ = ceil(log2 n), at least 1 (:63-65)
  uint32_t levels = 1;
  while ((1ull << levels) < n) ++levels;
  std::vector<DevBuf<uint32_t>*> up;
  std::vector<uint32_t*> up_ptrs;
  for (uint32_t k = 0; k < levels; ++k) {
    up.push_back(new DevBuf<uint32_t>(n));
    up_ptrs.push_back(up.back()->p);
  }
  struct UpGuard {
    std::vector<DevBuf<uint32_t>*>& v;
    ~UpGuard() {
      for (auto* b : v) delete b;
    }
  } up_guard{up};
  cuda_check(cudaMemcpyAsync(up_ptrs[0], tpar.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st),
             "lift");
  for (uint32_t k = 1; k < levels; ++k)
    k_lift<<<blocks(n), 256, 0, st>>>(n, up_ptrs[k - 1], up_ptrs[k]);
  DevBuf<uint32_t*> d_up(levels);
  cuda_check(cudaMemcpyAsync(d_up.p, up_ptrs.data(), sizeof(uint32_t*) * levels,
                             cudaMemcpyHostToDevice, st), "lift");

  // 5. off-tree ranking
  cuda_check(cudaMemsetAsync(counts.p, 0, 8, st), "memset");
  {
    DevBuf<uint32_t> ranks(m);
    k_iota<<<blocks(m), 256, 0, st>>>(m, ranks.p);
    DevBuf<uint8_t> nf(m);
    k_not<<<blocks(m), 256, 0, st>>>(m, in_tree.p, nf.p);
    size_t temp = 0;
    cub::DeviceSelect::Flagged(nullptr, temp, ranks.p, nf.p, off_rank.p, counts.p,
                               static_cast<int64_t>(m), st);
    DevBuf<unsigned char> t(temp);
    cuda_check(cub::DeviceSelect::Flagged(t.p, temp, ranks.p, nf.p, off_rank.p, counts.p,
                                          static_cast<int64_t>(m), st), "select");
    cuda_check(cudaStreamSynchronize(st), "select");
  }
  unsigned int noff = 0;
  cuda_check(cudaMemcpy(&noff, counts.p, 4, cudaMemcpyDeviceToHost), "off-tree size");
  // 6. fill count with the reference's density arithmetic (graph.cpp:114-116)
  uint64_t edges = n - 1ull, fill = 0;
  while (fill < noff) {
    const double density = static_cast<double>(edges) / static_cast<double>(n) - 1.0;
    if (std::max(density, 0.0) >= target_density) break;
    ++edges;
    ++fill;
  }
  DevBuf<uint32_t> all_rank(static_cast<uint64_t>(ntree) + fill + 1);
  DevBuf<uint32_t> all_order(static_cast<uint64_t>(ntree) + fill + 1);
  cuda_check(cudaMemcpyAsync(all_rank.p, tree_rank.p, sizeof(uint32_t) * ntree,
                             cudaMemcpyDeviceToDevice, st), "rows");
  k_seq<<<blocks(ntree), 256, 0, st>>>(ntree, 0u, all_order.p);
  if (fill > 0) {
    DevBuf<unsigned long long> dk(noff), tk(noff), kk(noff);
    DevBuf<uint32_t> p1(noff), p2(noff);
    k_rank_keys<<<blocks(noff), 256, 0, st>>>(noff, off_rank.p, order, eu.p, ev.p, ew.p, depth.p,
                                              rroot.p, d_up.p, levels, seed, dk.p, tk.p);
    k_iota<<<blocks(noff), 256, 0, st>>>(noff, p1.p);
    radix_pairs(tk.p, kk.p, p1.p, p2.p, noff, 0, 64, st);  // tiebreak asc
    // distortion keys in tiebreak order, then a stable sort by distortion
    // descending: p1 = positions (into off_rank) in ranked order.
    DevBuf<unsigned long long> dk2(noff);
    k_gather_u64<<<blocks(noff), 256, 0, st>>>(noff, dk.p, p2.p, dk2.p);
    radix_pairs(dk2.p, kk.p, p2.p, p1.p, noff, 0, 64, st);
    // selected off-tree ranks in ranked order: off_rank[p1[i]], i < fill
    DevBuf<uint32_t> sel_rank(fill);
    k_gather_u32<<<blocks(fill), 256, 0, st>>>(fill, off_rank.p, p1.p, sel_rank.p);
    cuda_check(cudaMemcpyAsync(all_rank.p + ntree, sel_rank.p, sizeof(uint32_t) * fill,
                               cudaMemcpyDeviceToDevice, st), "rows");
    k_seq<<<blocks(fill), 256, 0, st>>>(fill, ntree, all_order.p + ntree);
  }
  // H rows: tree edges in rank order, then the ranked fill
  const uint64_t nsel = ntree + fill;
  DevBuf<uint64_t> hrp(n + 1ull);
  DevBuf<uint32_t> hids(2 * nsel + 1);
  DevBuf<double> hw(2 * nsel + 1);
  build_rows(all_rank.p, all_order.p, nsel, hrp.p, hids.p, hw.p);
  cuda_check(cudaMemcpy(o_rp, hrp.p, sizeof(uint64_t) * (n + 1ull), cudaMemcpyDeviceToHost), "out");
  cuda_check(cudaMemcpy(o_ids, hids.p, sizeof(uint32_t) * 2 * nsel, cudaMemcpyDeviceToHost), "out");
  cuda_check(cudaMemcpy(o_w, hw.p, sizeof(double) * 2 * nsel, cudaMemcpyDeviceToHost), "out");
}

}  // namespace dyg
