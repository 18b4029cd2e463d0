// ref_harness.cpp -- extern "C" driver over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY (see oracle/oracle_abi.h). Built by
// oracle/ref/Makefile into oracle/_ref/libdyg_ref.so together with
// /root/reference/proj/src/{graph,walk,stream,matrix_market,sparsifier}.cpp,
// compiled in place with the reference's own flags (RelWithDebInfo: -O2 -g,
// no -march; /root/reference/proj/CMakeLists.txt:8-9). No reference source
// is copied; this file only marshals plain C arguments into the reference's
// C++ API and catches its exceptions.
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

#include "../oracle_abi.h"
#include "decisions.hpp"
#include "graph.hpp"
#include "matrix_market.hpp"
#include "rng.hpp"
#include "sparsifier.hpp"
#include "stream.hpp"
#include "support/generators.hpp"  // /root/reference/proj/tests/support
#include "walk.hpp"

using namespace dysparse;

namespace {

thread_local std::string g_error;
thread_local int g_kind = 0;

int fail(const Error& e) {
  g_error = e.what();
  g_kind = static_cast<int>(e.kind());
  return g_kind;
}
int fail_other(const std::exception& e) {
  g_error = e.what();
  g_kind = 2;
  return 2;
}

DynamicGraph* G(void* p) { return static_cast<DynamicGraph*>(p); }
const DynamicGraph* G(const void* p) { return static_cast<const DynamicGraph*>(p); }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_other(e);
  }
}

template <typename F>
void* guarded_ptr(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    fail(e);
  } catch (const std::exception& e) {
    fail_other(e);
  }
  return nullptr;
}

struct State {
  SparsifierState state;
};

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_error.c_str(); }
int orc_last_error_kind(void) { return g_kind; }
const char* orc_impl_name(void) { return "reference"; }

void* orc_graph_new(uint32_t n) {
  return guarded_ptr([&] { return static_cast<void*>(new DynamicGraph(n)); });
}
void* orc_graph_clone(const void* g) { return new DynamicGraph(*G(g)); }
void orc_graph_free(void* g) { delete G(g); }
uint32_t orc_graph_n(const void* g) { return G(g)->vertex_count(); }
uint64_t orc_graph_edges(const void* g) { return G(g)->edge_count(); }
double orc_graph_density(const void* g) { return G(g)->density(); }
int orc_graph_insert(void* g, uint32_t u, uint32_t v, double w) {
  return guarded([&] { G(g)->insert_edge(u, v, w); });
}
int orc_graph_delete(void* g, uint32_t u, uint32_t v) {
  return guarded([&] { G(g)->delete_edge(u, v); });
}
double orc_graph_edge_weight(const void* g, uint32_t u, uint32_t v) {
  return G(g)->edge_weight(u, v);
}
void orc_graph_export(const void* g, uint64_t* row_ptr, uint32_t* ids, double* w) {
  const DynamicGraph& graph = *G(g);
  uint64_t at = 0;
  for (uint32_t u = 0; u < graph.vertex_count(); ++u) {
    row_ptr[u] = at;
    for (const Neighbor& nb : graph.neighbors(u)) {
      ids[at] = nb.id;
      w[at] = nb.weight;
      ++at;
    }
  }
  row_ptr[graph.vertex_count()] = at;
}

void* orc_make_mesh(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max) {
  return guarded_ptr([&] {
    return static_cast<void*>(
        new DynamicGraph(testing::make_mesh(rows, cols, seed, w_min, w_max)));
  });
}

// SURVEY.md 8(d) C4 "grid4": make_mesh's loop minus the diagonal draw.
void* orc_make_grid4(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max) {
  return guarded_ptr([&] {
    auto* g = new DynamicGraph(rows * cols);
    SplitMix64 rng(hash_mix(seed + 0x3E5Bull));
    auto weight = [&] { return w_min + rng.next_double() * (w_max - w_min); };
    for (uint32_t r = 0; r < rows; ++r) {
      for (uint32_t c = 0; c < cols; ++c) {
        if (c + 1 < cols) g->insert_edge(r * cols + c, r * cols + c + 1, weight());
        if (r + 1 < rows) g->insert_edge(r * cols + c, (r + 1) * cols + c, weight());
      }
    }
    return static_cast<void*>(g);
  });
}

void* orc_make_random_connected(uint32_t n, uint32_t extra, uint64_t seed, double w_min,
                                double w_max, int with_pendant) {
  return guarded_ptr([&] {
    return static_cast<void*>(new DynamicGraph(
        testing::make_random_connected(n, extra, seed, w_min, w_max, with_pendant != 0)));
  });
}

void* orc_build_initial_sparsifier(const void* g, double target_density, uint64_t seed) {
  return guarded_ptr([&] {
    return static_cast<void*>(
        new DynamicGraph(build_initial_sparsifier(*G(g), target_density, seed)));
  });
}

void* orc_stream_generate(const void* g, double insert_fraction, double delete_fraction,
                          uint32_t batches, uint64_t seed, uint32_t locality) {
  return guarded_ptr([&] {
    StreamGenOptions o;
    o.insert_fraction = insert_fraction;
    o.delete_fraction = delete_fraction;
    o.batches = batches;
    o.seed = seed;
    o.locality = locality;
    return static_cast<void*>(new UpdateStream(generate_update_stream(*G(g), o)));
  });
}

void* orc_stream_from_events(const orc_event* ev, size_t n, uint32_t batch_count) {
  auto* s = new UpdateStream;
  s->events.resize(n);
  for (size_t i = 0; i < n; ++i) {
    EdgeEvent& e = s->events[i];
    e.kind = ev[i].kind == 0 ? EdgeEvent::Kind::Insertion : EdgeEvent::Kind::Deletion;
    e.u = ev[i].u;
    e.v = ev[i].v;
    e.weight = ev[i].weight;
    e.batch_index = ev[i].batch_index;
  }
  s->batch_count = batch_count;
  return s;
}
size_t orc_stream_size(const void* s) { return static_cast<const UpdateStream*>(s)->events.size(); }
uint32_t orc_stream_batches(const void* s) {
  return static_cast<const UpdateStream*>(s)->batch_count;
}
void orc_stream_copy(const void* s, orc_event* out) {
  const auto& events = static_cast<const UpdateStream*>(s)->events;
  for (size_t i = 0; i < events.size(); ++i) {
    out[i].kind = events[i].kind == EdgeEvent::Kind::Insertion ? 0u : 1u;
    out[i].u = events[i].u;
    out[i].v = events[i].v;
    out[i].batch_index = events[i].batch_index;
    out[i].weight = events[i].weight;
  }
}
void orc_stream_free(void* s) { delete static_cast<UpdateStream*>(s); }

uint64_t orc_walker_seed(uint64_t global_seed, uint64_t update_id, uint64_t walker) {
  return walker_seed(global_seed, update_id, walker);
}

int orc_single_walk(const void* g, uint32_t p, uint32_t q, double w_pq, double budget,
                    uint32_t cap, uint64_t rng_seed, uint32_t* terminal, uint32_t* steps,
                    double* acc, uint32_t* path, uint32_t path_cap, uint32_t* path_len) {
  return guarded([&] {
    SplitMix64 rng(rng_seed);
    WalkTrace t = single_walk(*G(g), p, q, w_pq, budget, cap, rng);
    *terminal = static_cast<uint32_t>(t.terminal);
    *steps = t.steps;
    *acc = t.accumulated_resistance;
    *path_len = static_cast<uint32_t>(t.path.size());
    for (size_t i = 0; i < t.path.size() && i < path_cap; ++i) path[i] = t.path[i];
  });
}

size_t orc_loop_erase(const uint32_t* path, size_t n, uint32_t* out) {
  auto erased = loop_erase(std::span<const VertexId>(path, n));
  std::memcpy(out, erased.data(), erased.size() * sizeof(uint32_t));
  return erased.size();
}

int orc_run_batch(const void* g, const orc_query* q, size_t nq, const orc_walk_config* cfg,
                  unsigned workers, orc_result* out, uint32_t* path_buf) {
  return guarded([&] {
    WalkConfig c;
    c.distortion_threshold = cfg->distortion_threshold;
    c.step_cap = cfg->step_cap;
    c.walker_count = cfg->walker_count;
    c.global_seed = cfg->global_seed;
    std::vector<WalkQuery> queries(nq);
    for (size_t i = 0; i < nq; ++i) {
      queries[i].kind = q[i].kind == 0 ? WalkQuery::Kind::Reach : WalkQuery::Kind::MinPath;
      queries[i].p = q[i].p;
      queries[i].q = q[i].q;
      queries[i].w_pq = q[i].w_pq;
      queries[i].update_id = q[i].update_id;
    }
    auto results = run_batch(*G(g), queries, c, workers);
    const size_t stride = static_cast<size_t>(c.step_cap) + 1;
    for (size_t i = 0; i < nq; ++i) {
      orc_result& r = out[i];
      std::memset(&r, 0, sizeof(r));
      r.steps_used = results[i].steps_used;
      if (queries[i].kind == WalkQuery::Kind::Reach) {
        r.reached = results[i].verdict.reached ? 1 : 0;
        r.best_estimate = results[i].verdict.best_estimate;
      } else if (results[i].path) {
        r.reached = 1;
        r.path_len = static_cast<uint32_t>(results[i].path->vertices.size());
        r.resistance = results[i].path->resistance;
        if (path_buf != nullptr) {
          std::memcpy(path_buf + i * stride, results[i].path->vertices.data(),
                      results[i].path->vertices.size() * sizeof(uint32_t));
        }
      }
    }
  });
}

void* orc_state_new(const void* g, const void* h, const orc_walk_config* cfg, int batched,
                    int freeze) {
  return guarded_ptr([&] {
    SparsifierOptions o;
    o.walk.distortion_threshold = cfg->distortion_threshold;
    o.walk.step_cap = cfg->step_cap;
    o.walk.walker_count = cfg->walker_count;
    o.walk.global_seed = cfg->global_seed;
    o.batched = batched != 0;
    o.freeze_sparsifier = freeze != 0;
    return static_cast<void*>(new State{SparsifierState(*G(g), *G(h), o)});
  });
}
void orc_state_free(void* st) { delete static_cast<State*>(st); }

int orc_state_replay_batch(void* st, const void* stream, uint32_t batch_index, orc_report* out) {
  return guarded([&] {
    BatchReport r = static_cast<State*>(st)->state.replay_batch(
        *static_cast<const UpdateStream*>(stream), batch_index);
    std::memset(out, 0, sizeof(*out));
    out->batch_index = r.batch_index;
    out->insertions_seen = r.insertions_seen;
    out->insertions_kept = r.insertions_kept;
    out->insertions_pruned = r.insertions_pruned;
    out->deletions_seen = r.deletions_seen;
    out->deletions_in_sparsifier = r.deletions_in_sparsifier;
    out->paths_recovered = r.paths_recovered;
    out->edges_recovered = r.edges_recovered;
    out->fallback_activations = r.fallback_activations;
    out->walker_steps = r.walker_steps;
    out->max_event_steps = r.max_event_steps;
    out->wall_ms = r.wall_ms;
    out->density_graph = r.density_graph;
    out->density_sparsifier = r.density_sparsifier;
  });
}
// replay_batch plus each event's decision (DYG_DECISION_* codes), derived
// from the reference's own pieces and pinned to its replay (decisions.hpp).
int orc_state_replay_batch_decisions(void* st, const void* stream, uint32_t batch_index,
                                     orc_report* out, uint8_t* decisions) {
  std::vector<uint8_t> dec;
  const int rc = guarded([&] {
    BatchReport r = dyg_oracle::replay_batch_with_decisions(
        static_cast<State*>(st)->state, *static_cast<const UpdateStream*>(stream), batch_index,
        dec);
    std::memset(out, 0, sizeof(*out));
    out->batch_index = r.batch_index;
    out->insertions_seen = r.insertions_seen;
    out->insertions_kept = r.insertions_kept;
    out->insertions_pruned = r.insertions_pruned;
    out->deletions_seen = r.deletions_seen;
    out->deletions_in_sparsifier = r.deletions_in_sparsifier;
    out->paths_recovered = r.paths_recovered;
    out->edges_recovered = r.edges_recovered;
    out->fallback_activations = r.fallback_activations;
    out->walker_steps = r.walker_steps;
    out->max_event_steps = r.max_event_steps;
    out->wall_ms = r.wall_ms;
    out->density_graph = r.density_graph;
    out->density_sparsifier = r.density_sparsifier;
  });
  if (!dec.empty()) std::memcpy(decisions, dec.data(), dec.size());
  return rc;
}
const void* orc_state_graph(const void* st) {
  return &static_cast<const State*>(st)->state.graph();
}
const void* orc_state_sparsifier(const void* st) {
  return &static_cast<const State*>(st)->state.sparsifier();
}
uint64_t orc_state_update_counter(const void* st) {
  return static_cast<const State*>(st)->state.update_counter();
}

void* orc_load_matrix_market(const char* path) {
  return guarded_ptr(
      [&] { return static_cast<void*>(new DynamicGraph(load_matrix_market(path))); });
}
int orc_save_matrix_market(const void* g, const char* path) {
  return guarded([&] { save_matrix_market(*G(g), path); });
}
void* orc_stream_load(const char* path) {
  return guarded_ptr([&] { return static_cast<void*>(new UpdateStream(load_update_stream(path))); });
}
int orc_stream_save(const void* s, const char* path) {
  return guarded([&] { save_update_stream(*static_cast<const UpdateStream*>(s), path); });
}

}  // extern "C"
