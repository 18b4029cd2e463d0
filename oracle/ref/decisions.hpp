// decisions.hpp -- per-event decisions of the reference's replay_batch
// (TEST INFRASTRUCTURE ONLY, like the rest of oracle/).
//
// The reference reports batch counters only; its per-event verdicts live
// inside replay_batch_deferred (sparsifier.cpp:466-533) / apply_* (:220-317).
// replay_batch_with_decisions derives them from the reference's own public
// pieces and then pins the derivation to the reference itself: it runs the
// REAL state.replay_batch afterwards and throws std::logic_error unless the
// derivation's G and H equal the reference's, row for row and bit for bit.
#pragma once

#include <cstdint>
#include <vector>

#include "sparsifier.hpp"
#include "stream.hpp"

namespace dyg_oracle {

// Codes as DYG_DECISION_* in include/dyg.h.
enum : std::uint8_t { kKept = 0, kPruned = 1, kGraphOnly = 2, kPathRecovered = 3,
                      kLocalFallback = 4, kNone = 255 };

// decisions[k] for the k-th event of batch `batch_index` (stream order).
// Rethrows the reference's dysparse::Error after filling the decisions of
// the events that committed (the rest stay kNone).
dysparse::BatchReport replay_batch_with_decisions(dysparse::SparsifierState& state,
                                                  const dysparse::UpdateStream& stream,
                                                  std::uint32_t batch_index,
                                                  std::vector<std::uint8_t>& decisions);

bool same_rows(const dysparse::DynamicGraph& a, const dysparse::DynamicGraph& b);

}  // namespace dyg_oracle
