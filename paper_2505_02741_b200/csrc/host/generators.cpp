// generators.cpp -- deterministic benchmark inputs: the mesh
// and grid graphs, the initial sparsifier (GRASS stand-in) and the update
// stream, each producing exactly the reference's edges, weights AND per-row
// order for the same seed, so GPU and CPU runs start from identical state.
//   make_mesh / make_random_connected  tests/support/generators.hpp:37-86
//   make_grid4                          SURVEY.md 8d C4 (mesh minus diagonals)
//   build_initial_sparsifier            proj/src/sparsifier.cpp:19-159
//   generate_update_stream              proj/src/stream.cpp:87-200
// Built with -ffp-contract=off: the reference's x86-64 build has no FMA.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <queue>
#include <unordered_set>

#include "../../../include/dyg_host.hpp"

namespace dyg {

namespace {

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;

std::uint64_t mix64(std::uint64_t x) {  // rng.hpp:37-41
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// SplitMix64 (rng.hpp:7-31).
struct Rng {
  std::uint64_t state;
  explicit Rng(std::uint64_t seed) : state(seed) {}
  std::uint64_t next() { return mix64(state += kGolden); }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  std::uint64_t next_below(std::uint64_t bound) {
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next()) * bound) >> 64);
  }
};

HostGraph lattice(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed, double w_min,
                  double w_max, bool diagonals) {
  HostGraph g(rows * cols);
  Rng rng(mix64(seed + 0x3E5Bull));
  const double span = w_max - w_min;
  auto draw = [&] { return w_min + rng.next_double() * span; };
  for (std::uint32_t r = 0; r < rows; ++r) {
    for (std::uint32_t c = 0; c < cols; ++c) {
      const VertexId at = r * cols + c;
      if (c + 1 < cols) g.insert_edge(at, at + 1, draw());
      if (r + 1 < rows) g.insert_edge(at, at + cols, draw());
      if (diagonals && r + 1 < rows && c + 1 < cols) {
        // One random diagonal per cell; the coin is drawn before its weight.
        if (rng.next() & 1u) {
          g.insert_edge(at, at + cols + 1, draw());
        } else {
          g.insert_edge(at + 1, at + cols, draw());
        }
      }
    }
  }
  return g;
}

// Tree-path resistance oracle of build_initial_sparsifier
// (sparsifier.cpp:42-101): BFS from vertex 0 over the spanning tree rows,
// resistance-to-root prefix sums, binary-lifting LCA.
class TreePaths {
 public:
  explicit TreePaths(const HostGraph& tree) {
    const std::uint32_t n = tree.vertex_count();
    depth_.assign(n, 0);
    to_root_.assign(n, 0.0);
    std::vector<VertexId> parent(n, 0);
    std::vector<std::uint8_t> seen(n, 0);
    std::vector<VertexId> queue;
    queue.reserve(n);
    seen[0] = 1;
    queue.push_back(0);
    for (std::size_t head = 0; head < queue.size(); ++head) {
      const VertexId u = queue[head];
      for (const Neighbor& nb : tree.neighbors(u)) {
        if (seen[nb.id]) continue;
        seen[nb.id] = 1;
        parent[nb.id] = u;
        depth_[nb.id] = depth_[u] + 1;
        to_root_[nb.id] = to_root_[u] + 1.0 / nb.weight;
        queue.push_back(nb.id);
      }
    }
    levels_ = 1;
    while ((1u << levels_) < n) ++levels_;
    jump_.assign(levels_, parent);
    for (std::uint32_t k = 1; k < levels_; ++k)
      for (std::uint32_t v = 0; v < n; ++v) jump_[k][v] = jump_[k - 1][jump_[k - 1][v]];
  }

  double between(VertexId u, VertexId v) const {
    return to_root_[u] + to_root_[v] - 2.0 * to_root_[ancestor(u, v)];
  }

 private:
  VertexId ancestor(VertexId u, VertexId v) const {
    if (depth_[u] < depth_[v]) std::swap(u, v);
    for (std::uint32_t k = 0, gap = depth_[u] - depth_[v]; gap != 0; ++k, gap >>= 1)
      if (gap & 1u) u = jump_[k][u];
    if (u == v) return u;
    for (std::uint32_t k = levels_; k-- > 0;) {
      if (jump_[k][u] != jump_[k][v]) {
        u = jump_[k][u];
        v = jump_[k][v];
      }
    }
    return jump_[0][u];
  }

  std::vector<std::uint32_t> depth_;
  std::vector<double> to_root_;
  std::vector<std::vector<VertexId>> jump_;
  std::uint32_t levels_ = 1;
};

}  // namespace

HostGraph make_mesh(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed, double w_min,
                    double w_max) {
  return lattice(rows, cols, seed, w_min, w_max, true);
}

HostGraph make_grid4(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed, double w_min,
                     double w_max) {
  return lattice(rows, cols, seed, w_min, w_max, false);
}

HostGraph make_random_connected(std::uint32_t n, std::uint32_t extra_edges, std::uint64_t seed,
                                double w_min, double w_max, bool with_pendant) {
  HostGraph g(n);
  Rng rng(mix64(seed + 0x57A77ull));
  auto draw = [&] { return w_min + rng.next_double() * (w_max - w_min); };
  const std::uint32_t core = with_pendant ? n - 1 : n;
  // The reference passes next_below(v) and weight() as arguments of one call
  // (generators.hpp:46); GCC evaluates them right to left: weight first.
  for (VertexId v = 1; v < core; ++v) {
    const double w = draw();
    const auto to = static_cast<VertexId>(rng.next_below(v));
    g.insert_edge(v, to, w);
  }
  std::uint32_t added = 0, tries = 0;
  while (added < extra_edges && tries < 100 * extra_edges + 100) {
    ++tries;
    const auto a = static_cast<VertexId>(rng.next_below(core));
    const auto b = static_cast<VertexId>(rng.next_below(core));
    if (a == b || g.has_edge(a, b)) continue;
    g.insert_edge(a, b, draw());
    ++added;
  }
  if (with_pendant) {
    const double w = draw();  // same right-to-left order (generators.hpp:58)
    const auto to = static_cast<VertexId>(rng.next_below(core));
    g.insert_edge(n - 1, to, w);
  }
  return g;
}

HostGraph build_initial_sparsifier(const HostGraph& g, double target_density,
                                   std::uint64_t seed) {
  if (target_density < 0.0) throw_error(ErrorKind::Usage, "target density must be nonnegative");
  if (!g.is_connected())
    throw_error(ErrorKind::Data, "graph must be connected to build a sparsifier");
  const std::uint32_t n = g.vertex_count();
  auto edges = g.edges();
  // Heaviest first, endpoints ascending on ties (total order).
  std::sort(edges.begin(), edges.end(), [](const auto& a, const auto& b) {
    return a.second != b.second ? a.second > b.second : a.first < b.first;
  });
  HostGraph h(n);
  std::vector<std::uint32_t> root(n);
  std::iota(root.begin(), root.end(), 0u);
  auto find = [&](std::uint32_t x) {
    while (root[x] != x) {
      root[x] = root[root[x]];
      x = root[x];
    }
    return x;
  };
  std::vector<std::size_t> rest;
  for (std::size_t i = 0; i < edges.size(); ++i) {
    const std::uint32_t a = find(edges[i].first.first), b = find(edges[i].first.second);
    if (a != b) {
      root[a] = b;
      h.insert_edge(edges[i].first.first, edges[i].first.second, edges[i].second);
    } else {
      rest.push_back(i);
    }
  }
  const TreePaths tree(h);
  struct Candidate {
    double distortion;
    std::uint64_t tiebreak;
    std::size_t edge;
  };
  std::vector<Candidate> cand;
  cand.reserve(rest.size());
  for (std::size_t i : rest) {
    const auto& e = edges[i];
    cand.push_back({e.second * tree.between(e.first.first, e.first.second),
                    mix64(seed ^ (static_cast<std::uint64_t>(e.first.first) << 32 | e.first.second)),
                    i});
  }
  std::sort(cand.begin(), cand.end(), [](const Candidate& a, const Candidate& b) {
    return a.distortion != b.distortion ? a.distortion > b.distortion : a.tiebreak < b.tiebreak;
  });
  for (const Candidate& c : cand) {
    if (std::max(h.density(), 0.0) >= target_density) break;
    const auto& e = edges[c.edge];
    h.insert_edge(e.first.first, e.first.second, e.second);
  }
  return h;
}

UpdateStream generate_update_stream(const HostGraph& g, const StreamGenOptions& o) {
  if (o.insert_fraction < 0.0 || o.delete_fraction < 0.0)
    throw_error(ErrorKind::Usage, "update fractions must be nonnegative");
  if (o.batches == 0) throw_error(ErrorKind::Usage, "batch count must be positive");
  const std::uint32_t n = g.vertex_count();
  const auto n_ins = static_cast<std::uint64_t>(std::llround(o.insert_fraction * static_cast<double>(n)));
  const auto n_del =
      static_cast<std::uint64_t>(std::llround(o.delete_fraction * static_cast<double>(g.edge_count())));
  auto edges = g.edges();
  double lo = std::numeric_limits<double>::infinity(), hi = 0.0;
  for (const auto& e : edges) {
    lo = std::min(lo, e.second);
    hi = std::max(hi, e.second);
  }
  if (n_ins > 0 && edges.empty())
    throw_error(ErrorKind::Data, "cannot derive insertion weights from an edgeless graph");
  Rng rng(mix64(o.seed + 0x12345678ull));
  UpdateStream s;
  s.events.reserve(n_ins + n_del);
  std::unordered_set<std::uint64_t> taken;
  const std::uint64_t max_tries = 200 * std::max<std::uint64_t>(n_ins, 1) + 10000;
  std::uint64_t tries = 0;
  std::vector<std::uint32_t> hop;
  std::vector<VertexId> nearby, frontier;
  for (std::uint64_t k = 0; k < n_ins; ++k) {
    VertexId u = 0, v = 0;
    bool ok = false;
    while (tries < max_tries) {
      ++tries;
      u = static_cast<VertexId>(rng.next_below(n));
      if (o.locality == 0) {
        v = static_cast<VertexId>(rng.next_below(n));
      } else {
        // Vertices within `locality` hops of u in BFS discovery order,
        // u excluded (stream.cpp:90-110). The reference allocates an n-sized
        // distance array per sample (O(n) each, unusable at C4/C5 with
        // locality); here one array is reused and only the visited entries
        // are reset afterwards -- the same BFS, hence the same ball and order.
        if (hop.size() != n) hop.assign(n, std::numeric_limits<std::uint32_t>::max());
        nearby.clear();
        frontier.clear();
        hop[u] = 0;
        frontier.push_back(u);
        for (std::size_t head = 0; head < frontier.size(); ++head) {
          const VertexId x = frontier[head];
          if (hop[x] == o.locality) continue;
          for (const Neighbor& nb : g.neighbors(x)) {
            if (hop[nb.id] != std::numeric_limits<std::uint32_t>::max()) continue;
            hop[nb.id] = hop[x] + 1;
            nearby.push_back(nb.id);
            frontier.push_back(nb.id);
          }
        }
        for (const VertexId x : frontier) hop[x] = std::numeric_limits<std::uint32_t>::max();
        if (nearby.empty()) continue;
        v = nearby[rng.next_below(nearby.size())];
      }
      if (u == v) continue;
      const std::uint64_t key = static_cast<std::uint64_t>(std::min(u, v)) * n + std::max(u, v);
      if (g.has_edge(u, v) || taken.count(key) != 0) continue;
      taken.insert(key);
      ok = true;
      break;
    }
    if (!ok) throw_error(ErrorKind::Data, "could not sample enough non-edges (graph too dense?)");
    EdgeEvent e;
    e.kind = EdgeEvent::Kind::Insertion;
    e.u = std::min(u, v);
    e.v = std::max(u, v);
    e.weight = lo + rng.next_double() * (hi - lo);
    e.batch_index = static_cast<std::uint32_t>(k * o.batches / std::max<std::uint64_t>(n_ins, 1));
    s.events.push_back(e);
  }
  if (n_del > g.edge_count()) throw_error(ErrorKind::Data, "deletion fraction exceeds edge count");
  const std::uint32_t base = n_ins > 0 ? o.batches : 0;
  for (std::uint64_t k = 0; k < n_del; ++k) {
    const std::uint64_t pick = k + rng.next_below(edges.size() - k);
    std::swap(edges[k], edges[pick]);
    EdgeEvent e;
    e.kind = EdgeEvent::Kind::Deletion;
    e.u = edges[k].first.first;
    e.v = edges[k].first.second;
    e.batch_index =
        base + static_cast<std::uint32_t>(k * o.batches / std::max<std::uint64_t>(n_del, 1));
    s.events.push_back(e);
  }
  s.batch_count = s.events.empty() ? 0 : s.events.back().batch_index + 1;
  return s;
}

}  // namespace dyg
