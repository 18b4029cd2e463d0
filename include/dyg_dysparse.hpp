// dyg_dysparse.hpp -- the reference's own types bound to the device update
// path: dyg::DysparseGpuSparsifierState is a drop-in for
// dysparse::SparsifierState (proj/src/sparsifier.hpp:71-112) that takes and
// returns dysparse::DynamicGraph / UpdateStream / SparsifierOptions /
// BatchReport / UpdateReport and throws dysparse::Error (error.hpp:11-20).
//
// Include it from a translation unit that already sees the reference's
// headers (graph.hpp, stream.hpp, sparsifier.hpp) and link libdyg.so; see
// INTEGRATION.md §2. A device failure (status 4, no reference ErrorKind)
// throws std::runtime_error.
#pragma once

#include <stdexcept>
#include <string>

#include "dyg_adapter.hpp"

namespace dyg {

struct DysparseTraits {
  using Graph = dysparse::DynamicGraph;
  using Stream = dysparse::UpdateStream;
  using Options = dysparse::SparsifierOptions;
  using InsertionDecision = dysparse::InsertionDecision;
  using DeletionOutcome = dysparse::DeletionOutcome;
  using BatchReport = dysparse::BatchReport;
  using UpdateReport = dysparse::UpdateReport;

  // Neighbour order is not part of DynamicGraph's contract (graph.hpp:19-22):
  // the edge set is rebuilt with insert_edge, once per edge (u < v).
  static Graph make_graph(std::uint32_t n, const std::uint64_t* row_ptr,
                          const std::uint32_t* ids, const double* w) {
    Graph g(n);
    for (std::uint32_t u = 0; u < n; ++u)
      for (std::uint64_t i = row_ptr[u]; i < row_ptr[u + 1]; ++i)
        if (u < ids[i]) g.insert_edge(u, ids[i], w[i]);
    return g;
  }

  [[noreturn]] static void raise(int kind, const std::string& message) {
    if (kind >= 1 && kind <= 3)
      throw dysparse::Error(static_cast<dysparse::ErrorKind>(kind), message);
    throw std::runtime_error(message);
  }
};

using DysparseGpuSparsifierState = SparsifierStateAdapter<DysparseTraits>;

}  // namespace dyg
