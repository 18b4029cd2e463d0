// stream_gen.cu -- generate_update_stream (proj/src/stream.cpp:114-200) with
// its insertion sampling on the device, bit-identical to the reference.
//
// The reference draws insertion attempts from ONE SplitMix64 stream
// (rng.hpp:7-31): attempt = u = next_below(n), v = next_below(n) (locality
// 0), rejected when u == v, (u, v) is an edge of G, or the pair was already
// taken; an accepted attempt draws its weight next. SplitMix64 is
// counter-based -- draw j is hash_mix(state0 + j * gamma) -- so a whole run
// of attempts can be evaluated in parallel under the assumption that none of
// them is rejected: attempt i of a round then uses draws j0 + 3i + {1, 2, 3}.
// A round checks every candidate (self-loop, edge lookup in G, first
// occurrence of its key among everything accepted so far -- a device hash
// set keyed by the unordered pair, value = the event index that claimed it,
// atomicMin), finds the first rejected attempt k*, accepts [0, k*), undoes
// the hash-set claims of the attempts past k*, and the next round resumes
// after the rejected attempt's two draws. Random pairs in a sparse graph are
// almost never rejected (C5: ~2 rejections in 10^6 insertions), so a stream
// takes a few rounds; rounds shrink adaptively when rejections are frequent
// (dense graphs). Deletions -- a partial Fisher-Yates over G's edge list, a
// chain of dependent swaps -- stay on the host (O(deleted) swaps), as does
// the locality > 0 mode (its attempts consume a data-dependent number of
// draws; the host generator's BFS reuse already makes it 10-45x faster than
// the reference's).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_map>
#include <vector>

#include "graph_store.cuh"
#include "stream_gen.cuh"

namespace dyg {

namespace {

constexpr unsigned long long kGammaSM = 0x9E3779B97F4A7C15ull;
constexpr unsigned long long kEmptyKey = ~0ull;
constexpr unsigned long long kNoIndex = ~0ull;

__host__ __device__ inline unsigned long long mix64(unsigned long long x) {  // rng.hpp:37-41
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// Draw j (1-based) of the stream seeded with s0 (splitmix64_next: state +=
// gamma, then mix).
__host__ __device__ inline unsigned long long draw(unsigned long long s0, unsigned long long j) {
  return mix64(s0 + j * kGammaSM);
}
__device__ inline uint32_t below(unsigned long long x, uint32_t bound) {  // next_below
  return static_cast<uint32_t>(__umul64hi(x, static_cast<unsigned long long>(bound)));
}

struct GenArgs {
  const uint64_t* rp;    // G's CSR (reference row order)
  const uint32_t* ids;
  uint32_t n;
  unsigned long long s0;
  unsigned long long j0;     // draws consumed before this round
  unsigned long long k0;     // events accepted before this round
  uint32_t m;                // attempts in this round
  unsigned long long* key;   // hash set: unordered-pair keys
  unsigned long long* val;   // ... and the event index that claimed each
  unsigned long long mask;   // capacity - 1 (power of two)
  uint32_t* cu;              // per attempt: u, v, status
  uint32_t* cv;
  uint8_t* bad;
  unsigned long long* slot;  // hash slot the attempt claimed (kNoIndex: none)
  unsigned long long* first_bad;  // min rejected attempt of the round
};

__device__ bool has_edge_csr(const GenArgs& a, uint32_t u, uint32_t v) {
  const uint64_t du = a.rp[u + 1] - a.rp[u], dv = a.rp[v + 1] - a.rp[v];
  const uint32_t x = du <= dv ? u : v, y = du <= dv ? v : u;  // scan the smaller row
  for (uint64_t i = a.rp[x]; i < a.rp[x + 1]; ++i)
    if (a.ids[i] == y) return true;
  return false;
}

// Attempt i: draws, self-loop and edge checks, and the claim of its key.
__global__ void k_gen_attempts(GenArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.m) return;
  const unsigned long long j = a.j0 + 3ull * i;
  const uint32_t u = below(draw(a.s0, j + 1), a.n);
  const uint32_t v = below(draw(a.s0, j + 2), a.n);
  a.cu[i] = u;
  a.cv[i] = v;
  a.slot[i] = kNoIndex;
  uint8_t bad = 0;
  if (u == v || has_edge_csr(a, u, v)) {
    bad = 1;
  } else {
    const uint32_t lo = u < v ? u : v, hi = u < v ? v : u;
    const unsigned long long k = static_cast<unsigned long long>(lo) * a.n + hi;  // stream.cpp:159
    unsigned long long h = mix64(k) & a.mask;
    for (;;) {
      const unsigned long long prev = atomicCAS(a.key + h, kEmptyKey, k);
      if (prev == kEmptyKey || prev == k) break;
      h = (h + 1) & a.mask;
    }
    atomicMin(a.val + h, a.k0 + i);
    a.slot[i] = h;
  }
  a.bad[i] = bad;
}

// An attempt whose key was claimed by an earlier one (this round or before)
// is a repeat; the first rejected attempt bounds the round.
__global__ void k_gen_first_bad(GenArgs a) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.m) return;
  bool bad = a.bad[i] != 0;
  if (!bad) bad = a.val[a.slot[i]] != a.k0 + i;
  a.bad[i] = bad ? 1 : 0;
  if (bad) atomicMin(a.first_bad, static_cast<unsigned long long>(i));
}

// Accepted attempts become events; the claims of attempts at or past the
// first rejection are withdrawn (they are re-drawn in the next round).
__global__ void k_gen_emit(GenArgs a, unsigned long long n_ins, uint32_t batches, double lo,
                           double span, dyg_event* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.m) return;
  const unsigned long long kstar = *a.first_bad;
  if (i < kstar) {
    const uint32_t u = a.cu[i], v = a.cv[i];
    const unsigned long long k = a.k0 + i;
    const double u01 =
        __dmul_rn(static_cast<double>(draw(a.s0, a.j0 + 3ull * i + 3) >> 11), 0x1.0p-53);
    dyg_event e;
    e.kind = 0;
    e.u = u < v ? u : v;
    e.v = u < v ? v : u;
    e.weight = __dadd_rn(lo, __dmul_rn(u01, span));  // stream.cpp:174
    e.batch_index = static_cast<uint32_t>(k * batches / (n_ins > 0 ? n_ins : 1));
    out[k] = e;
  } else if (a.slot[i] != kNoIndex) {
    atomicCAS(a.val + a.slot[i], a.k0 + i, kNoIndex);
  }
}

// Rebuild the pair set from the accepted events alone (withdrawn claims of
// speculative attempts leave their keys behind and would fill the table).
__global__ void k_gen_rehash(const dyg_event* __restrict__ out, unsigned long long k, uint32_t n,
                             unsigned long long* key, unsigned long long* val,
                             unsigned long long mask) {
  const unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
  if (i >= k) return;
  const unsigned long long kk = static_cast<unsigned long long>(out[i].u) * n + out[i].v;
  unsigned long long h = mix64(kk) & mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(key + h, kEmptyKey, kk);
    if (prev == kEmptyKey || prev == kk) break;
    h = (h + 1) & mask;
  }
  val[h] = i;
}

inline unsigned blocks(uint64_t n) { return static_cast<unsigned>((n + 255) / 256); }

template <typename T>
T* dalloc(size_t n, const char* what) {
  T* p = nullptr;
  cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * std::max<size_t>(n, 1)), what);
  return p;
}

struct DevBufs {
  std::vector<void*> ptrs;
  template <typename T>
  T* get(size_t n, const char* what) {
    T* p = dalloc<T>(n, what);
    ptrs.push_back(p);
    return p;
  }
  ~DevBufs() {
    for (void* p : ptrs) cudaFree(p);
  }
};

}  // namespace

void generate_stream_device(const dyg_csr& g, double insert_fraction, double delete_fraction,
                            uint32_t batches, uint64_t seed, std::vector<dyg_event>& events,
                            uint32_t& batch_count, GenStats* stats) {
  // stream.cpp:115-127
  if (insert_fraction < 0.0 || delete_fraction < 0.0)
    throw GenError{1, "update fractions must be nonnegative"};
  if (batches == 0) throw GenError{1, "batch count must be positive"};
  const uint32_t n = g.n;
  const uint64_t nnz = g.row_ptr[n];
  const uint64_t m_edges = nnz / 2;
  const auto n_ins = static_cast<uint64_t>(std::llround(insert_fraction * static_cast<double>(n)));
  const auto n_del =
      static_cast<uint64_t>(std::llround(delete_fraction * static_cast<double>(m_edges)));
  // edges() -- (u, v) with u < v in row order (graph.cpp:118-127) -- is
  // not materialised: `upper[u]` counts row u's entries with v > u, so edge p
  // of the list is found by a binary search over their prefix sums. The
  // weight range of G (stream.cpp:129-134) in the same pass.
  std::vector<uint64_t> upper(n + 1ull, 0);
  double wmin = std::numeric_limits<double>::infinity(), wmax = 0.0;
  for (uint32_t u = 0; u < n; ++u) {
    uint64_t c = 0;
    for (uint64_t i = g.row_ptr[u]; i < g.row_ptr[u + 1]; ++i)
      if (u < g.ids[i]) {
        ++c;
        wmin = std::min(wmin, g.w[i]);
        wmax = std::max(wmax, g.w[i]);
      }
    upper[u + 1] = upper[u] + c;
  }
  const uint64_t ne = upper[n];
  auto edge_at = [&](uint64_t p, uint32_t& eu, uint32_t& ev) {
    eu = static_cast<uint32_t>(std::upper_bound(upper.begin(), upper.end(), p) - upper.begin() - 1);
    uint64_t r = p - upper[eu];
    for (uint64_t i = g.row_ptr[eu];; ++i)
      if (eu < g.ids[i] && r-- == 0) {
        ev = g.ids[i];
        return;
      }
  };
  if (n_ins > 0 && ne == 0)
    throw GenError{2, "cannot derive insertion weights from an edgeless graph"};
  const unsigned long long s0 = mix64(seed + 0x12345678ull);
  events.assign(n_ins, dyg_event{});
  unsigned long long j = 0;  // draws consumed
  GenStats st{};
  if (n_ins > 0) {
    DevBufs d;
    uint64_t* rp = d.get<uint64_t>(n + 1ull, "stream generator: graph");
    uint32_t* ids = d.get<uint32_t>(nnz, "stream generator: graph");
    cuda_check(cudaMemcpy(rp, g.row_ptr, sizeof(uint64_t) * (n + 1ull), cudaMemcpyHostToDevice),
               "stream generator: graph upload");
    if (nnz)
      cuda_check(cudaMemcpy(ids, g.ids, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice),
                 "stream generator: graph upload");
    const uint32_t chunk_max = static_cast<uint32_t>(std::min<uint64_t>(n_ins, 1u << 22));
    unsigned long long cap = 1024;
    while (cap < 2 * (n_ins + chunk_max)) cap <<= 1;
    GenArgs a{};
    a.rp = rp;
    a.ids = ids;
    a.n = n;
    a.s0 = s0;
    a.key = d.get<unsigned long long>(cap, "stream generator: pair set");
    a.val = d.get<unsigned long long>(cap, "stream generator: pair set");
    a.mask = cap - 1;
    a.cu = d.get<uint32_t>(chunk_max, "stream generator: attempts");
    a.cv = d.get<uint32_t>(chunk_max, "stream generator: attempts");
    a.bad = d.get<uint8_t>(chunk_max, "stream generator: attempts");
    a.slot = d.get<unsigned long long>(chunk_max, "stream generator: attempts");
    a.first_bad = d.get<unsigned long long>(1, "stream generator: attempts");
    dyg_event* out = d.get<dyg_event>(n_ins, "stream generator: events");
    cuda_check(cudaMemset(a.key, 0xFF, sizeof(unsigned long long) * cap), "pair set");
    cuda_check(cudaMemset(a.val, 0xFF, sizeof(unsigned long long) * cap), "pair set");
    // stream.cpp:143: attempts are capped for the whole insertion phase.
    const uint64_t attempt_cap = 200 * std::max<uint64_t>(n_ins, 1) + 10000;
    uint64_t attempts = 0, k = 0;
    uint64_t claimed = 0;  // keys ever placed in the set (accepted + withdrawn)
    uint32_t chunk = chunk_max;
    const double span = wmax - wmin;
    while (k < n_ins) {
      if (attempts >= attempt_cap)
        throw GenError{2, "could not sample enough non-edges (graph too dense?)"};
      const uint32_t m = static_cast<uint32_t>(
          std::min<uint64_t>({n_ins - k, static_cast<uint64_t>(chunk), attempt_cap - attempts}));
      if (claimed + m > cap / 2) {  // keep the set at most half full
        cuda_check(cudaMemset(a.key, 0xFF, sizeof(unsigned long long) * cap), "pair set");
        cuda_check(cudaMemset(a.val, 0xFF, sizeof(unsigned long long) * cap), "pair set");
        if (k) k_gen_rehash<<<blocks(k), 256>>>(out, k, n, a.key, a.val, a.mask);
        claimed = k;
        ++st.rehashes;
      }
      claimed += m;
      a.j0 = j;
      a.k0 = k;
      a.m = m;
      const unsigned long long none = m;
      cuda_check(cudaMemcpy(a.first_bad, &none, sizeof none, cudaMemcpyHostToDevice), "round");
      k_gen_attempts<<<blocks(m), 256>>>(a);
      k_gen_first_bad<<<blocks(m), 256>>>(a);
      k_gen_emit<<<blocks(m), 256>>>(a, n_ins, batches, wmin, span, out);
      cuda_check(cudaGetLastError(), "stream generator");
      unsigned long long kstar = 0;
      cuda_check(cudaMemcpy(&kstar, a.first_bad, sizeof kstar, cudaMemcpyDeviceToHost), "round");
      ++st.rounds;
      k += kstar;
      j += 3ull * kstar;
      attempts += kstar;
      if (kstar < m) {  // the rejected attempt: its two draws, one attempt
        j += 2;
        attempts += 1;
        ++st.rejections;
        // Frequent rejections: shorter speculative rounds.
        chunk = static_cast<uint32_t>(
            std::min<uint64_t>(chunk_max, std::max<uint64_t>(256, 4 * kstar)));
      } else {
        chunk = chunk_max;
      }
    }
    cuda_check(cudaMemcpy(events.data(), out, sizeof(dyg_event) * n_ins, cudaMemcpyDeviceToHost),
               "stream generator: events");
  }
  // Deletions (stream.cpp:180-196): partial Fisher-Yates over the edge list,
  // draws continuing after the insertion phase's. Only the positions the
  // swaps touched differ from the identity: they live in a small map.
  if (n_del > ne) throw GenError{2, "deletion fraction exceeds edge count"};
  const uint32_t deletion_base = n_ins > 0 ? batches : 0;
  events.reserve(n_ins + n_del);
  std::unordered_map<uint64_t, uint64_t> moved;  // position -> edge index now there
  moved.reserve(2 * n_del);
  auto at = [&](uint64_t p) {
    const auto it = moved.find(p);
    return it == moved.end() ? p : it->second;
  };
  for (uint64_t k = 0; k < n_del; ++k) {
    const unsigned long long x = draw(s0, ++j);
    const uint64_t pick =
        k + static_cast<uint64_t>((static_cast<unsigned __int128>(x) * (ne - k)) >> 64);
    const uint64_t ek = at(pick);  // std::swap(edges[k], edges[pick])
    moved[pick] = at(k);
    moved[k] = ek;
    dyg_event e{};
    e.kind = 1;
    edge_at(ek, e.u, e.v);
    e.batch_index =
        deletion_base + static_cast<uint32_t>(k * batches / std::max<uint64_t>(n_del, 1));
    events.push_back(e);
  }
  batch_count = events.empty() ? 0 : events.back().batch_index + 1;
  if (stats) *stats = st;
}

}  // namespace dyg
