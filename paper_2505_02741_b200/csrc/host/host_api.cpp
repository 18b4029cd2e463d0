// host_api.cpp -- C wrappers (include/dyg_host.h) over the host input
// pipeline, for bindings (the Python package uses them through ctypes).
#include <cstring>
#include <memory>
#include <string>

#include "../../../include/dyg_host.h"
#include "../../../include/dyg_host.hpp"

struct dygh_graph {
  dyg::HostGraph g;
  dyg::HostGraph::Csr csr;
  bool csr_valid = false;
};

struct dygh_stream {
  dyg::UpdateStream s;
  std::vector<dyg_event> flat;
};

namespace {

thread_local std::string g_host_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return DYG_OK;
  } catch (const dyg::Error& e) {
    g_host_error = e.what();
    return static_cast<int>(e.kind());
  } catch (const std::bad_alloc&) {
    g_host_error = "host allocation failed";
    return DYG_ERR_DEVICE;
  } catch (const std::exception& e) {
    g_host_error = e.what();
    return DYG_ERR_DATA;
  }
}

dygh_graph* wrap(dyg::HostGraph&& g) { return new dygh_graph{std::move(g), {}, false}; }

void flatten(dygh_stream* s) {
  s->flat.resize(s->s.events.size());
  for (std::size_t i = 0; i < s->flat.size(); ++i) {
    const dyg::EdgeEvent& e = s->s.events[i];
    s->flat[i] = dyg_event{e.kind == dyg::EdgeEvent::Kind::Insertion ? 0u : 1u, e.u, e.v,
                           e.batch_index, e.weight};
  }
}

dygh_stream* wrap(dyg::UpdateStream&& us) {
  auto* s = new dygh_stream{std::move(us), {}};
  flatten(s);
  return s;
}

}  // namespace

extern "C" {

const char* dygh_last_error(void) { return g_host_error.c_str(); }

int dygh_graph_new(uint32_t n, dygh_graph** out) {
  return guard([&] { *out = wrap(dyg::HostGraph(n)); });
}
int dygh_graph_from_csr(const dyg_csr* csr, dygh_graph** out) {
  return guard([&] {
    if (csr == nullptr || csr->row_ptr == nullptr)
      dyg::throw_error(dyg::ErrorKind::Usage, "null csr");
    *out = wrap(dyg::HostGraph::from_csr(*csr));
  });
}
void dygh_graph_free(dygh_graph* g) { delete g; }
uint32_t dygh_graph_n(const dygh_graph* g) { return g->g.vertex_count(); }
uint64_t dygh_graph_edges(const dygh_graph* g) { return g->g.edge_count(); }
double dygh_graph_density(const dygh_graph* g) { return g->g.density(); }
int dygh_graph_insert(dygh_graph* g, uint32_t u, uint32_t v, double w) {
  return guard([&] {
    g->csr_valid = false;
    g->g.insert_edge(u, v, w);
  });
}
int dygh_graph_delete(dygh_graph* g, uint32_t u, uint32_t v) {
  return guard([&] {
    g->csr_valid = false;
    g->g.delete_edge(u, v);
  });
}
double dygh_graph_edge_weight(const dygh_graph* g, uint32_t u, uint32_t v) {
  double w = 0.0;
  if (guard([&] { w = g->g.edge_weight(u, v); }) != DYG_OK) return 0.0;
  return w;
}
int dygh_graph_csr(dygh_graph* g, dyg_csr* out) {
  return guard([&] {
    if (!g->csr_valid) {
      g->csr = g->g.to_csr();
      g->csr_valid = true;
    }
    *out = g->csr.view();
  });
}

int dygh_make_mesh(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max,
                   dygh_graph** out) {
  return guard([&] { *out = wrap(dyg::make_mesh(rows, cols, seed, w_min, w_max)); });
}
int dygh_make_grid4(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max,
                    dygh_graph** out) {
  return guard([&] { *out = wrap(dyg::make_grid4(rows, cols, seed, w_min, w_max)); });
}
int dygh_make_random_connected(uint32_t n, uint32_t extra, uint64_t seed, double w_min,
                               double w_max, int with_pendant, dygh_graph** out) {
  return guard([&] {
    *out = wrap(dyg::make_random_connected(n, extra, seed, w_min, w_max, with_pendant != 0));
  });
}
int dygh_build_initial_sparsifier(const dygh_graph* g, double target_density, uint64_t seed,
                                  dygh_graph** out) {
  return guard([&] { *out = wrap(dyg::build_initial_sparsifier(g->g, target_density, seed)); });
}
int dygh_generate_stream(const dygh_graph* g, double insert_fraction, double delete_fraction,
                         uint32_t batches, uint64_t seed, uint32_t locality, dygh_stream** out) {
  return guard([&] {
    dyg::StreamGenOptions o;
    o.insert_fraction = insert_fraction;
    o.delete_fraction = delete_fraction;
    o.batches = batches;
    o.seed = seed;
    o.locality = locality;
    *out = wrap(dyg::generate_update_stream(g->g, o));
  });
}

int dygh_load_matrix_market(const char* path, dygh_graph** out) {
  return guard([&] { *out = wrap(dyg::load_matrix_market(path)); });
}
int dygh_save_matrix_market(const dygh_graph* g, const char* path) {
  return guard([&] { dyg::save_matrix_market(g->g, path); });
}
int dygh_load_stream(const char* path, dygh_stream** out) {
  return guard([&] { *out = wrap(dyg::load_update_stream(path)); });
}
int dygh_save_stream(const dygh_stream* s, const char* path) {
  return guard([&] { dyg::save_update_stream(s->s, path); });
}

int dygh_stream_from_events(const dyg_event* events, size_t n, uint32_t batch_count,
                            dygh_stream** out) {
  return guard([&] {
    dyg::UpdateStream us;
    us.events.resize(n);
    for (size_t i = 0; i < n; ++i) {
      dyg::EdgeEvent& e = us.events[i];
      e.kind = events[i].kind == 0 ? dyg::EdgeEvent::Kind::Insertion
                                   : dyg::EdgeEvent::Kind::Deletion;
      e.u = events[i].u;
      e.v = events[i].v;
      e.weight = events[i].weight;
      e.batch_index = events[i].batch_index;
    }
    us.batch_count = batch_count;
    *out = wrap(std::move(us));
  });
}
void dygh_stream_free(dygh_stream* s) { delete s; }
size_t dygh_stream_size(const dygh_stream* s) { return s->flat.size(); }
uint32_t dygh_stream_batches(const dygh_stream* s) { return s->s.batch_count; }
const dyg_event* dygh_stream_events(const dygh_stream* s) { return s->flat.data(); }

}  // extern "C"
