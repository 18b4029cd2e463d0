// dyg_adapter.hpp -- header-only C++ drop-in for dysparse::SparsifierState.
//
// SparsifierStateAdapter<Traits> has the public surface of the reference's
// SparsifierState (proj/src/sparsifier.hpp:71-112) over the C-ABI of
// include/dyg.h, for ANY caller-side graph / stream / options / error types
// with the reference's shape. It touches the caller's types only through:
//
//   Graph      g.vertex_count(), g.neighbors(u) -> range of {id, weight}
//              (graph.hpp:14-17, 27-38); Traits::make_graph builds one back.
//   Stream     .events (each {kind, u, v, weight, batch_index}, kind an enum
//              with ::Insertion / ::Deletion) and .batch_count
//              (stream.hpp:11-23).
//   Options    .walk.{distortion_threshold, step_cap, walker_count,
//              global_seed}, .batched, .freeze_sparsifier (sparsifier.hpp:
//              25-34, walk.hpp:13-18).
//   InsertionDecision {Kept, Pruned}; DeletionOutcome {kind, edges_added}
//              with Kind {GraphOnly, PathRecovered, LocalFallback};
//              BatchReport / UpdateReport with the reference's field names
//              (sparsifier.hpp:36-65).
//   Errors     Traits::raise(int kind, const std::string& message) --
//              the caller's exception (dysparse::Error(ErrorKind(kind), ...)
//              for the reference, error.hpp:11-20); kind 4 is a device
//              failure, which has no reference ErrorKind.
//
// So a reference caller keeps its own DynamicGraph / UpdateStream /
// SparsifierOptions / Error types and swaps only the state class
// (include/dyg_dysparse.hpp gives the Traits for the dysparse namespace;
// include/dyg_host.hpp instantiates it for this library's host types).
// Neighbour order inside a row is not part of the reference's contract
// (graph.hpp:19-22): graph() / sparsifier() rebuild the caller's graph with
// Traits::make_graph, and rows() exports the device rows in their exact
// order for bit-level comparisons.
#pragma once

#include <cstdint>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "dyg.h"

namespace dyg {

template <class Traits>
class SparsifierStateAdapter {
 public:
  using Graph = typename Traits::Graph;
  using Stream = typename Traits::Stream;
  using Options = typename Traits::Options;
  using InsertionDecision = typename Traits::InsertionDecision;
  using DeletionOutcome = typename Traits::DeletionOutcome;
  using BatchReport = typename Traits::BatchReport;
  using UpdateReport = typename Traits::UpdateReport;
  using Event = typename std::decay_t<decltype(std::declval<const Stream&>().events)>::value_type;

  // Device rows in their exact order (row_ptr[n + 1], ids / w [2|E|]).
  struct Rows {
    std::vector<std::uint64_t> row_ptr;
    std::vector<std::uint32_t> ids;
    std::vector<double> w;
  };

  // SparsifierState(G, H, options) (sparsifier.cpp:183-203): the same
  // validation and messages, then G and H are uploaded to `device`.
  SparsifierStateAdapter(const Graph& graph, const Graph& sparsifier, Options options,
                         int device = 0)
      : options_(std::move(options)) {
    const Csr g = flatten(graph), h = flatten(sparsifier);
    const dyg_csr gv = g.view(), hv = h.view();
    dyg_options o{};
    o.walk.distortion_threshold = options_.walk.distortion_threshold;
    o.walk.step_cap = options_.walk.step_cap;
    o.walk.walker_count = options_.walk.walker_count;
    o.walk.global_seed = options_.walk.global_seed;
    o.batched = options_.batched ? 1 : 0;
    o.freeze_sparsifier = options_.freeze_sparsifier ? 1 : 0;
    check(dyg_session_create(&gv, &hv, &o, device, &session_));
  }
  ~SparsifierStateAdapter() { dyg_session_destroy(session_); }
  SparsifierStateAdapter(const SparsifierStateAdapter&) = delete;
  SparsifierStateAdapter& operator=(const SparsifierStateAdapter&) = delete;

  // graph() / sparsifier() (sparsifier.hpp:76-77): the reference returns a
  // const reference to host rows; here G and H live on the device, so these
  // build the caller's graph from an export.
  Graph graph() const { return export_graph(0); }
  Graph sparsifier() const { return export_graph(1); }
  Rows rows(int which) const {
    std::uint32_t n = 0;
    std::uint64_t edges = 0;
    check(dyg_graph_info(session_, which, &n, &edges, nullptr));
    Rows r;
    r.row_ptr.resize(n + 1ull);
    r.ids.resize(2 * edges);
    r.w.resize(2 * edges);
    check(dyg_export_rows(session_, which, r.row_ptr.data(), r.ids.data(), r.w.data(),
                          2 * edges));
    return r;
  }
  const Options& options() const { return options_; }
  std::uint64_t update_counter() const { return dyg_update_counter(session_); }

  // apply_insertion / apply_deletion / last_event_steps (sparsifier.cpp:243-317).
  InsertionDecision apply_insertion(std::uint32_t u, std::uint32_t v, double weight) {
    int d = 0;
    check(dyg_apply_insertion(session_, u, v, weight, &d));
    return d == 0 ? InsertionDecision::Kept : InsertionDecision::Pruned;
  }
  DeletionOutcome apply_deletion(std::uint32_t u, std::uint32_t v) {
    int kind = 0;
    std::uint32_t added = 0;
    check(dyg_apply_deletion(session_, u, v, &kind, &added));
    DeletionOutcome out;
    out.kind = static_cast<typename DeletionOutcome::Kind>(kind);
    out.edges_added = added;
    return out;
  }
  std::uint64_t last_event_steps() const { return dyg_last_event_steps(session_); }

  // replay_batch(stream, b) (sparsifier.cpp:541-548). Only the batch's events
  // are converted (one pass over the stream selects them, as the reference's
  // own scan does, :401-404). `decisions` (optional) receives one
  // DYG_DECISION_* per event of the batch, in stream order.
  BatchReport replay_batch(const Stream& stream, std::uint32_t batch_index,
                           std::vector<std::uint8_t>* decisions = nullptr) {
    if (batch_index >= stream.batch_count && stream.batch_count > 0)
      Traits::raise(DYG_ERR_USAGE, "batch index out of range");
    std::vector<dyg_event> ev;
    std::vector<std::uint64_t> pos;
    for (std::size_t i = 0; i < stream.events.size(); ++i)
      if (stream.events[i].batch_index == batch_index) {
        ev.push_back(to_event(stream.events[i]));
        pos.push_back(i);
      }
    if (decisions) decisions->assign(ev.size(), DYG_DECISION_NONE);
    dyg_batch_report r{};
    check(dyg_replay_events(session_, ev.data(), pos.data(), ev.size(), batch_index, &r,
                            decisions ? decisions->data() : nullptr));
    return to_report(r);
  }

  // replay(stream) (sparsifier.cpp:550-559) in one library call (the upload
  // of later batches overlaps the work on earlier ones). `decisions`: one per
  // stream event, indexed by stream position.
  UpdateReport replay(const Stream& stream, std::vector<std::uint8_t>* decisions = nullptr) {
    std::vector<dyg_event> ev(stream.events.size());
    for (std::size_t i = 0; i < ev.size(); ++i) ev[i] = to_event(stream.events[i]);
    std::vector<dyg_batch_report> reps(stream.batch_count);
    if (decisions) decisions->assign(ev.size(), DYG_DECISION_NONE);
    if (stream.batch_count)
      check(dyg_replay_stream(session_, ev.data(), ev.size(), nullptr, stream.batch_count,
                              reps.data(), decisions ? decisions->data() : nullptr));
    UpdateReport out;
    for (const dyg_batch_report& r : reps) out.batches.push_back(to_report(r));
    check(dyg_graph_info(session_, 0, nullptr, nullptr, &out.final_density_graph));
    check(dyg_graph_info(session_, 1, nullptr, nullptr, &out.final_density_sparsifier));
    return out;
  }

  // dyGRASS.incremental() / .decremental(): a deferred
  // batch that must contain only insertions / only deletions (Usage error
  // otherwise; mixed batches go through replay_batch).
  BatchReport incremental(const Stream& stream, std::uint32_t batch_index,
                          std::vector<std::uint8_t>* decisions = nullptr) {
    require_kind(stream, batch_index, true);
    return replay_batch(stream, batch_index, decisions);
  }
  BatchReport decremental(const Stream& stream, std::uint32_t batch_index,
                          std::vector<std::uint8_t>* decisions = nullptr) {
    require_kind(stream, batch_index, false);
    return replay_batch(stream, batch_index, decisions);
  }

  dyg_session* session() const { return session_; }

 private:
  struct Csr {
    std::vector<std::uint64_t> row_ptr;
    std::vector<std::uint32_t> ids;
    std::vector<double> w;
    dyg_csr view() const {
      return dyg_csr{static_cast<std::uint32_t>(row_ptr.size() - 1), 0, row_ptr.data(),
                     ids.data(), w.data()};
    }
  };

  static Csr flatten(const Graph& g) {
    Csr c;
    const std::uint32_t n = g.vertex_count();
    c.row_ptr.assign(n + 1ull, 0);
    for (std::uint32_t u = 0; u < n; ++u) {
      for (const auto& nb : g.neighbors(u)) {
        c.ids.push_back(nb.id);
        c.w.push_back(nb.weight);
      }
      c.row_ptr[u + 1] = c.ids.size();
    }
    return c;
  }

  static dyg_event to_event(const Event& e) {
    return dyg_event{e.kind == Event::Kind::Insertion ? 0u : 1u, e.u, e.v, e.batch_index,
                     e.kind == Event::Kind::Insertion ? e.weight : 0.0};
  }

  static BatchReport to_report(const dyg_batch_report& r) {
    BatchReport o{};
    o.batch_index = r.batch_index;
    o.insertions_seen = r.insertions_seen;
    o.insertions_kept = r.insertions_kept;
    o.insertions_pruned = r.insertions_pruned;
    o.deletions_seen = r.deletions_seen;
    o.deletions_in_sparsifier = r.deletions_in_sparsifier;
    o.paths_recovered = r.paths_recovered;
    o.edges_recovered = r.edges_recovered;
    o.fallback_activations = r.fallback_activations;
    o.walker_steps = r.walker_steps;
    o.max_event_steps = r.max_event_steps;
    o.wall_ms = r.wall_ms;
    o.density_graph = r.density_graph;
    o.density_sparsifier = r.density_sparsifier;
    return o;
  }

  Graph export_graph(int which) const {
    const Rows r = rows(which);
    return Traits::make_graph(static_cast<std::uint32_t>(r.row_ptr.size() - 1), r.row_ptr.data(),
                              r.ids.data(), r.w.data());
  }

  static void require_kind(const Stream& stream, std::uint32_t batch_index, bool insertions) {
    for (const Event& e : stream.events)
      if (e.batch_index == batch_index &&
          (e.kind == Event::Kind::Insertion) != insertions)
        Traits::raise(DYG_ERR_USAGE, insertions ? "incremental(): the batch contains deletions"
                                                : "decremental(): the batch contains insertions");
  }

  void check(int status) const {
    if (status != DYG_OK) Traits::raise(status, dyg_last_error());
  }

  dyg_session* session_ = nullptr;
  Options options_;
};

}  // namespace dyg
