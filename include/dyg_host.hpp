// dyg_host.hpp -- C++ host API of the B200 dyGRASS update path.
//
// Mirrors the reference's public C++ surface (proj/src/{graph,stream,
// sparsifier}.hpp) so a caller of dysparse::SparsifierState can switch to
// dyg::GpuSparsifierState with the same calls, argument meanings and error
// behaviour (exceptions of kind Usage / Data / Numeric, error.hpp:9-32).
// Behind it, G and H live on the GPU (include/dyg.h); the host keeps no
// copy of them.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dyg.h"
#include "dyg_adapter.hpp"

namespace dyg {

using VertexId = std::uint32_t;

// error.hpp:9 (Device = 4 has no reference analogue: CUDA failures).
enum class ErrorKind { Usage = 1, Data = 2, Numeric = 3, Device = 4 };

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& message) : std::runtime_error(message), kind_(kind) {}
  ErrorKind kind() const { return kind_; }

 private:
  ErrorKind kind_;
};

[[noreturn]] void throw_error(ErrorKind kind, const std::string& message);

struct Neighbor {  // graph.hpp:14-17
  VertexId id;
  double weight;
};

// Host adjacency rows with DynamicGraph's semantics (graph.hpp:23-68). Used
// for inputs (file loading, generators) and for exported device state.
class HostGraph {
 public:
  enum class InsertOutcome { New, Coalesced };
  explicit HostGraph(std::uint32_t vertex_count);
  static HostGraph from_csr(const dyg_csr& csr);

  std::uint32_t vertex_count() const { return static_cast<std::uint32_t>(rows_.size()); }
  std::uint64_t edge_count() const { return edge_count_; }
  double total_weight() const { return total_weight_; }
  std::uint32_t degree(VertexId u) const;
  std::span<const Neighbor> neighbors(VertexId u) const;
  bool has_edge(VertexId u, VertexId v) const;
  double edge_weight(VertexId u, VertexId v) const;
  InsertOutcome insert_edge(VertexId u, VertexId v, double weight);
  double delete_edge(VertexId u, VertexId v);
  double density() const;
  std::vector<std::pair<std::pair<VertexId, VertexId>, double>> edges() const;
  bool is_connected() const;

  // Flattened rows in row order (row_ptr / ids / w) for dyg_session_create.
  struct Csr {
    std::vector<std::uint64_t> row_ptr;
    std::vector<std::uint32_t> ids;
    std::vector<double> w;
    dyg_csr view() const;
  };
  Csr to_csr() const;

 private:
  void check_vertex(VertexId u) const;
  Neighbor* find(VertexId u, VertexId v);
  const Neighbor* find(VertexId u, VertexId v) const;
  std::vector<std::vector<Neighbor>> rows_;
  std::uint64_t edge_count_ = 0;
  double total_weight_ = 0.0;
};

// stream.hpp:11-23
struct EdgeEvent {
  enum class Kind { Insertion, Deletion };
  Kind kind = Kind::Insertion;
  VertexId u = 0;
  VertexId v = 0;
  double weight = 0.0;
  std::uint32_t batch_index = 0;
};
struct UpdateStream {
  std::vector<EdgeEvent> events;
  std::uint32_t batch_count = 0;
};
struct StreamGenOptions {  // stream.hpp:33-42
  double insert_fraction = 0.0;
  double delete_fraction = 0.0;
  std::uint32_t batches = 1;
  std::uint64_t seed = 0;
  std::uint32_t locality = 0;
};

UpdateStream load_update_stream(const std::string& path);
void save_update_stream(const UpdateStream& stream, const std::string& path);
UpdateStream generate_update_stream(const HostGraph& g, const StreamGenOptions& options);
HostGraph load_matrix_market(const std::string& path);
void save_matrix_market(const HostGraph& g, const std::string& path);

// Benchmark-input generators.
HostGraph make_mesh(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed,
                    double w_min = 0.5, double w_max = 2.0);
HostGraph make_grid4(std::uint32_t rows, std::uint32_t cols, std::uint64_t seed,
                     double w_min = 0.5, double w_max = 2.0);
HostGraph make_random_connected(std::uint32_t n, std::uint32_t extra_edges, std::uint64_t seed,
                                double w_min = 0.1, double w_max = 10.0,
                                bool with_pendant = false);
HostGraph build_initial_sparsifier(const HostGraph& g, double target_density, std::uint64_t seed);

struct WalkConfig {  // walk.hpp:13-18
  double distortion_threshold = 10.0;
  std::uint32_t step_cap = 100;
  std::uint32_t walker_count = 16;
  std::uint64_t global_seed = 0;
};
struct SparsifierOptions {  // sparsifier.hpp:25-34
  WalkConfig walk;
  bool batched = false;
  bool freeze_sparsifier = false;
};
enum class InsertionDecision { Kept, Pruned };
struct DeletionOutcome {
  enum class Kind { GraphOnly, PathRecovered, LocalFallback };
  Kind kind = Kind::GraphOnly;
  std::uint32_t edges_added = 0;
};
using BatchReport = dyg_batch_report;  // same fields as sparsifier.hpp:44-59
struct UpdateReport {
  std::vector<BatchReport> batches;
  double final_density_graph = 0.0;
  double final_density_sparsifier = 0.0;
};

// SparsifierState (sparsifier.hpp:71-112) with G and H device-resident, on
// this library's host types: the header-only adapter (dyg_adapter.hpp)
// instantiated with them. (A caller of the reference keeps its own types:
// dyg_dysparse.hpp.)
struct HostTraits {
  using Graph = HostGraph;
  using Stream = UpdateStream;
  using Options = SparsifierOptions;
  using InsertionDecision = dyg::InsertionDecision;
  using DeletionOutcome = dyg::DeletionOutcome;
  using BatchReport = dyg::BatchReport;
  using UpdateReport = dyg::UpdateReport;
  static Graph make_graph(std::uint32_t n, const std::uint64_t* row_ptr,
                          const std::uint32_t* ids, const double* w) {
    return HostGraph::from_csr(dyg_csr{n, 0, row_ptr, ids, w});  // exact row order
  }
  [[noreturn]] static void raise(int kind, const std::string& message) {
    throw Error(static_cast<ErrorKind>(kind), message);
  }
};
using GpuSparsifierState = SparsifierStateAdapter<HostTraits>;

}  // namespace dyg
