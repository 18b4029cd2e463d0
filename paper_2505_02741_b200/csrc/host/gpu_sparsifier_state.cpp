// gpu_sparsifier_state.cpp -- dyg::GpuSparsifierState, the C++ drop-in for
// dysparse::SparsifierState (proj/src/sparsifier.hpp:71-112) over the C-ABI.
// Status codes from dyg.h become dyg::Error of the same ErrorKind, like the
// reference's exceptions (error.hpp:11-32).
#include <vector>

#include "../../../include/dyg_host.hpp"

namespace dyg {

namespace {

void raise(int status) {
  if (status == DYG_OK) return;
  throw Error(static_cast<ErrorKind>(status), dyg_last_error());
}

std::vector<dyg_event> flatten(const UpdateStream& s) {
  std::vector<dyg_event> out(s.events.size());
  for (std::size_t i = 0; i < out.size(); ++i) {
    const EdgeEvent& e = s.events[i];
    out[i] = dyg_event{e.kind == EdgeEvent::Kind::Insertion ? 0u : 1u, e.u, e.v, e.batch_index,
                       e.weight};
  }
  return out;
}

}  // namespace

GpuSparsifierState::GpuSparsifierState(const HostGraph& graph, const HostGraph& sparsifier,
                                       SparsifierOptions options, int device)
    : options_(options) {
  const HostGraph::Csr g = graph.to_csr();
  const HostGraph::Csr h = sparsifier.to_csr();
  const dyg_csr gv = g.view(), hv = h.view();
  dyg_options o{};
  o.walk.distortion_threshold = options.walk.distortion_threshold;
  o.walk.step_cap = options.walk.step_cap;
  o.walk.walker_count = options.walk.walker_count;
  o.walk.global_seed = options.walk.global_seed;
  o.batched = options.batched ? 1 : 0;
  o.freeze_sparsifier = options.freeze_sparsifier ? 1 : 0;
  raise(dyg_session_create(&gv, &hv, &o, device, &session_));
}

GpuSparsifierState::~GpuSparsifierState() { dyg_session_destroy(session_); }

HostGraph GpuSparsifierState::export_graph(int which) const {
  std::uint32_t n = 0;
  std::uint64_t edges = 0;
  raise(dyg_graph_info(session_, which, &n, &edges, nullptr));
  HostGraph::Csr c;
  c.row_ptr.resize(n + 1ull);
  c.ids.resize(2 * edges);
  c.w.resize(2 * edges);
  raise(dyg_export_rows(session_, which, c.row_ptr.data(), c.ids.data(), c.w.data(), 2 * edges));
  return HostGraph::from_csr(c.view());
}

HostGraph GpuSparsifierState::graph() const { return export_graph(0); }
HostGraph GpuSparsifierState::sparsifier() const { return export_graph(1); }
std::uint64_t GpuSparsifierState::update_counter() const { return dyg_update_counter(session_); }
std::uint64_t GpuSparsifierState::last_event_steps() const {
  return dyg_last_event_steps(session_);
}

InsertionDecision GpuSparsifierState::apply_insertion(VertexId u, VertexId v, double weight) {
  int decision = 0;
  raise(dyg_apply_insertion(session_, u, v, weight, &decision));
  return decision == 0 ? InsertionDecision::Kept : InsertionDecision::Pruned;
}

DeletionOutcome GpuSparsifierState::apply_deletion(VertexId u, VertexId v) {
  int kind = 0;
  std::uint32_t added = 0;
  raise(dyg_apply_deletion(session_, u, v, &kind, &added));
  DeletionOutcome out;
  out.kind = static_cast<DeletionOutcome::Kind>(kind);
  out.edges_added = added;
  return out;
}

BatchReport GpuSparsifierState::replay_batch(const UpdateStream& stream,
                                             std::uint32_t batch_index) {
  const std::vector<dyg_event> ev = flatten(stream);
  BatchReport r{};
  raise(dyg_replay_batch(session_, ev.data(), ev.size(), stream.batch_count, batch_index, &r));
  return r;
}

// sparsifier.cpp:550-559, one library call: dyg_replay_stream pipelines the
// upload of later batches with the work on earlier ones (events grouped by
// batch; an ungrouped stream replays batch by batch inside the library).
UpdateReport GpuSparsifierState::replay(const UpdateStream& stream) {
  const std::vector<dyg_event> ev = flatten(stream);
  UpdateReport report;
  report.batches.resize(stream.batch_count);
  if (stream.batch_count)
    raise(dyg_replay_stream(session_, ev.data(), ev.size(), nullptr, stream.batch_count,
                            report.batches.data()));
  double dg = 0.0, dh = 0.0;
  raise(dyg_graph_info(session_, 0, nullptr, nullptr, &dg));
  raise(dyg_graph_info(session_, 1, nullptr, nullptr, &dh));
  report.final_density_graph = dg;
  report.final_density_sparsifier = dh;
  return report;
}

}  // namespace dyg
