// adapter_test.cpp -- the drop-in boundary exercised from C++ the way a
// reference caller would use it: dysparse::SparsifierState (the UNMODIFIED
// reference, compiled from /root/reference/proj/src by oracle/ref/Makefile)
// and dyg::DysparseGpuSparsifierState (include/dyg_dysparse.hpp over
// libdyg.so) run side by side on the SAME dysparse::DynamicGraph /
// UpdateStream / SparsifierOptions objects. After every batch: identical
// BatchReports, identical per-event decisions (reference side derived and
// pinned by oracle/ref/decisions.cpp), identical G / H rows (ids, weight
// bits, order); errors surface as dysparse::Error with the reference's kind
// and message (error.hpp:11-32). Built into oracle/_ref/adapter_test (test
// infrastructure: it links the reference objects); run by
// tests/test_gpu_adapter.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "decisions.hpp"
#include "dyg_dysparse.hpp"
#include "graph.hpp"
#include "sparsifier.hpp"
#include "stream.hpp"
#include "support/generators.hpp"

using namespace dysparse;
using Gpu = dyg::DysparseGpuSparsifierState;

namespace {

int g_failures = 0;

#define EXPECT(cond, ...)                                      \
  do {                                                         \
    if (!(cond)) {                                             \
      std::fprintf(stderr, "FAIL %s:%d: %s: ", __FILE__, __LINE__, #cond); \
      std::fprintf(stderr, __VA_ARGS__);                       \
      std::fprintf(stderr, "\n");                              \
      ++g_failures;                                            \
    }                                                          \
  } while (0)

bool same_report(const BatchReport& a, const BatchReport& b) {
  return a.batch_index == b.batch_index && a.insertions_seen == b.insertions_seen &&
         a.insertions_kept == b.insertions_kept && a.insertions_pruned == b.insertions_pruned &&
         a.deletions_seen == b.deletions_seen &&
         a.deletions_in_sparsifier == b.deletions_in_sparsifier &&
         a.paths_recovered == b.paths_recovered && a.edges_recovered == b.edges_recovered &&
         a.fallback_activations == b.fallback_activations && a.walker_steps == b.walker_steps &&
         a.max_event_steps == b.max_event_steps && a.density_graph == b.density_graph &&
         a.density_sparsifier == b.density_sparsifier;
}

// Device rows vs the reference's rows: ids, weight bits, order.
bool same_rows(const Gpu::Rows& r, const DynamicGraph& g) {
  if (r.row_ptr.size() != g.vertex_count() + 1ull) return false;
  for (VertexId u = 0; u < g.vertex_count(); ++u) {
    const auto nb = g.neighbors(u);
    if (r.row_ptr[u + 1] - r.row_ptr[u] != nb.size()) return false;
    for (std::size_t i = 0; i < nb.size(); ++i) {
      const std::uint64_t at = r.row_ptr[u] + i;
      if (r.ids[at] != nb[i].id || std::memcmp(&r.w[at], &nb[i].weight, sizeof(double)) != 0)
        return false;
    }
  }
  return true;
}

bool same_edges(const DynamicGraph& a, const DynamicGraph& b) {
  const auto ea = a.edges(), eb = b.edges();
  if (ea.size() != eb.size()) return false;
  for (std::size_t i = 0; i < ea.size(); ++i)
    if (ea[i].first != eb[i].first || std::memcmp(&ea[i].second, &eb[i].second, 8) != 0)
      return false;
  return true;
}

bool is_kind(const UpdateStream& s, std::uint32_t b, EdgeEvent::Kind k) {
  bool any = false;
  for (const EdgeEvent& e : s.events)
    if (e.batch_index == b) {
      if (e.kind != k) return false;
      any = true;
    }
  return any;
}

// Replays every batch on both; dyGRASS.incremental()/decremental() for pure
// batches, replay_batch for mixed ones.
void side_by_side(const char* name, const DynamicGraph& g, const DynamicGraph& h,
                  const UpdateStream& s, SparsifierOptions o) {
  SparsifierState ref(g, h, o);
  Gpu gpu(g, h, o);
  std::size_t n_events = 0, n_dec = 0;
  for (std::uint32_t b = 0; b < s.batch_count; ++b) {
    std::vector<std::uint8_t> rdec, ddec;
    std::string rerr, derr;
    int rkind = 0, dkind = 0;
    BatchReport rr{}, dr{};
    try {
      rr = dyg_oracle::replay_batch_with_decisions(ref, s, b, rdec);
    } catch (const Error& e) {
      rerr = e.what();
      rkind = static_cast<int>(e.kind());
    }
    try {
      if (is_kind(s, b, EdgeEvent::Kind::Insertion)) dr = gpu.incremental(s, b, &ddec);
      else if (is_kind(s, b, EdgeEvent::Kind::Deletion)) dr = gpu.decremental(s, b, &ddec);
      else dr = gpu.replay_batch(s, b, &ddec);
    } catch (const Error& e) {
      derr = e.what();
      dkind = static_cast<int>(e.kind());
    }
    EXPECT(rerr == derr && rkind == dkind, "%s batch %u: error '%s'(%d) vs '%s'(%d)", name, b,
           rerr.c_str(), rkind, derr.c_str(), dkind);
    if (rerr.empty()) EXPECT(same_report(rr, dr), "%s batch %u: reports differ", name, b);
    EXPECT(rdec == ddec, "%s batch %u: decisions differ", name, b);
    EXPECT(same_rows(gpu.rows(0), ref.graph()), "%s batch %u: G rows differ", name, b);
    EXPECT(same_rows(gpu.rows(1), ref.sparsifier()), "%s batch %u: H rows differ", name, b);
    EXPECT(gpu.update_counter() == ref.update_counter(), "%s batch %u: counters", name, b);
    n_events += rdec.size();
    for (std::uint8_t d : rdec) n_dec += d != dyg_oracle::kNone;
    if (!rerr.empty()) break;
  }
  // graph() / sparsifier() hand back the caller's own type.
  EXPECT(same_edges(gpu.graph(), ref.graph()), "%s: graph() edge sets differ", name);
  EXPECT(same_edges(gpu.sparsifier(), ref.sparsifier()), "%s: sparsifier() edge sets differ", name);
  std::printf("%s: %u batches, %zu events, %zu decisions compared\n", name, s.batch_count,
              n_events, n_dec);
}

// A random valid mixed stream (coalescing, re-insertions, deletions of
// edges inserted earlier in the batch) from the reference's own RNG.
UpdateStream mixed_stream(const DynamicGraph& g, std::uint64_t seed, std::uint32_t batches,
                          std::uint32_t per_batch) {
  SplitMix64 rng(seed);
  DynamicGraph live = g;
  UpdateStream s;
  s.batch_count = batches;
  const std::uint32_t n = g.vertex_count();
  for (std::uint32_t b = 0; b < batches; ++b)
    for (std::uint32_t i = 0; i < per_batch; ++i) {
      const VertexId u = static_cast<VertexId>(rng.next() % n);
      if (rng.next_double() < 0.4 && live.degree(u) > 0) {
        const auto nb = live.neighbors(u);
        const VertexId v = nb[rng.next() % nb.size()].id;
        live.delete_edge(u, v);
        s.events.push_back({EdgeEvent::Kind::Deletion, u, v, 0.0, b});
      } else {
        const VertexId v = static_cast<VertexId>(rng.next() % n);
        if (u == v) continue;
        const double w = 0.3 + 2.7 * rng.next_double();
        live.insert_edge(u, v, w);
        s.events.push_back({EdgeEvent::Kind::Insertion, u, v, w, b});
      }
    }
  return s;
}

}  // namespace

int main() {
  SparsifierOptions o;
  o.walk.distortion_threshold = 100.0;
  o.walk.step_cap = 100;
  o.walk.walker_count = 16;
  o.walk.global_seed = 42;
  o.batched = true;

  // C2: fe_4elt-shaped mesh, 10 incremental + 10 decremental.
  {
    const DynamicGraph g = testing::make_mesh(100, 110, 1);
    const DynamicGraph h = build_initial_sparsifier(g, 0.10, 1);
    StreamGenOptions so;
    so.insert_fraction = 0.25;
    so.delete_fraction = 0.01;
    so.batches = 10;
    so.seed = 7;
    so.locality = 3;
    side_by_side("C2", g, h, generate_update_stream(g, so), o);
  }
  // Mixed batches, small budgets (pruning and budget stops), fallbacks.
  for (std::uint64_t seed : {3ull, 4ull}) {
    const DynamicGraph g = testing::make_mesh(14, 15, seed);
    const DynamicGraph h = build_initial_sparsifier(g, 0.10, seed);
    SparsifierOptions m = o;
    m.walk.distortion_threshold = 3.0;
    m.walk.step_cap = 12;
    m.walk.walker_count = 4;
    side_by_side("mixed", g, h, mixed_stream(g, seed, 6, 50), m);
  }
  // A failing batch: deleting an absent edge (sparsifier.cpp:491).
  {
    const DynamicGraph g = testing::make_mesh(9, 9, 2);
    const DynamicGraph h = build_initial_sparsifier(g, 0.10, 2);
    const auto edges = g.edges();
    UpdateStream s;
    s.batch_count = 2;
    s.events.push_back({EdgeEvent::Kind::Insertion, 0, 40, 1.0, 0});
    for (int i = 0; i < 8; ++i)
      s.events.push_back({EdgeEvent::Kind::Deletion, edges[i].first.first,
                          edges[i].first.second, 0.0, 1});
    s.events.push_back({EdgeEvent::Kind::Deletion, edges[2].first.first, edges[2].first.second,
                        0.0, 1});
    side_by_side("failing", g, h, s, o);
  }
  // Usage errors: the reference's message for an out-of-range batch; a
  // deletion batch given to incremental().
  {
    const DynamicGraph g = testing::make_mesh(6, 6, 1);
    const DynamicGraph h = build_initial_sparsifier(g, 0.10, 1);
    UpdateStream s;
    s.batch_count = 1;
    const auto e0 = g.edges()[0].first;
    s.events.push_back({EdgeEvent::Kind::Deletion, e0.first, e0.second, 0.0, 0});
    SparsifierState ref(g, h, o);
    Gpu gpu(g, h, o);
    std::string rmsg, dmsg;
    try { ref.replay_batch(s, 5); } catch (const Error& e) { rmsg = e.what(); }
    try { gpu.replay_batch(s, 5); } catch (const Error& e) { dmsg = e.what(); }
    EXPECT(!rmsg.empty() && rmsg == dmsg, "usage: '%s' vs '%s'", rmsg.c_str(), dmsg.c_str());
    bool usage = false;
    try { gpu.incremental(s, 0); } catch (const Error& e) { usage = e.kind() == ErrorKind::Usage; }
    EXPECT(usage, "incremental() accepted a deletion batch");
    // Immediate mode: apply_insertion / apply_deletion return values.
    SparsifierOptions im = o;
    im.batched = false;
    SparsifierState ri(g, h, im);
    Gpu di(g, h, im);
    EXPECT(ri.apply_insertion(0, 35, 1.5) == di.apply_insertion(0, 35, 1.5), "apply_insertion");
    const auto a = ri.apply_deletion(e0.first, e0.second);
    const auto b = di.apply_deletion(e0.first, e0.second);
    EXPECT(a.kind == b.kind && a.edges_added == b.edges_added, "apply_deletion");
    EXPECT(ri.last_event_steps() == di.last_event_steps(), "last_event_steps");
    EXPECT(same_rows(di.rows(1), ri.sparsifier()), "immediate H rows");
    std::string m1, m2;
    int k1 = 0, k2 = 0;
    try { ri.apply_deletion(e0.first, e0.second); } catch (const Error& e) { m1 = e.what(); k1 = (int)e.kind(); }
    try { di.apply_deletion(e0.first, e0.second); } catch (const Error& e) { m2 = e.what(); k2 = (int)e.kind(); }
    EXPECT(!m1.empty() && m1 == m2 && k1 == k2, "absent deletion: '%s' vs '%s'", m1.c_str(), m2.c_str());
  }
  if (g_failures) {
    std::fprintf(stderr, "adapter_test: %d failures\n", g_failures);
    return 1;
  }
  std::printf("adapter_test ok\n");
  return 0;
}
