// decisions.cpp -- see decisions.hpp. TEST INFRASTRUCTURE ONLY.
//
// Deferred mode restates replay_batch_deferred (sparsifier.cpp:395-539) on
// COPIES of the state's G and H with the reference's own DynamicGraph
// operations and run_batch; immediate mode calls the reference's public
// apply_insertion / apply_deletion (:243-317) on a copy of the state. Either
// way the real replay_batch then runs and must produce the same G and H.
#include "decisions.hpp"

#include <cmath>
#include <cstring>
#include <limits>
#include <optional>
#include <stdexcept>

#include "walk.hpp"

using namespace dysparse;

namespace dyg_oracle {

bool same_rows(const DynamicGraph& a, const DynamicGraph& b) {
  if (a.vertex_count() != b.vertex_count() || a.edge_count() != b.edge_count()) return false;
  for (VertexId u = 0; u < a.vertex_count(); ++u) {
    const auto ra = a.neighbors(u), rb = b.neighbors(u);
    if (ra.size() != rb.size()) return false;
    for (std::size_t i = 0; i < ra.size(); ++i)
      if (ra[i].id != rb[i].id || std::memcmp(&ra[i].weight, &rb[i].weight, sizeof(double)) != 0)
        return false;
  }
  return true;
}

namespace {

// validate_event_shape (sparsifier.cpp:321-337): a failing batch commits
// nothing.
bool shape_ok(const EdgeEvent& e, std::uint32_t n) {
  if (e.u >= n || e.v >= n || e.u == e.v) return false;
  return e.kind != EdgeEvent::Kind::Insertion || (e.weight > 0.0 && std::isfinite(e.weight));
}

// set_edge_weight (sparsifier.cpp:207-216).
void set_weight(DynamicGraph& h, VertexId u, VertexId v, double target) {
  const double current = h.edge_weight(u, v);
  if (target > current) {
    h.insert_edge(u, v, target - current);
  } else if (target < current) {
    h.delete_edge(u, v);
    h.insert_edge(u, v, target);
  }
}

// run_local_fallback (sparsifier.cpp:264-280); returns edges added.
std::uint32_t local_fallback(const DynamicGraph& g, DynamicGraph& h, VertexId u, VertexId v) {
  std::uint32_t added = 0;
  for (const VertexId x : {u, v}) {
    if (h.degree(x) != 0 || g.degree(x) == 0) continue;
    const Neighbor* best = nullptr;
    for (const Neighbor& nb : g.neighbors(x))
      if (best == nullptr || nb.weight > best->weight ||
          (nb.weight == best->weight && nb.id < best->id))
        best = &nb;
    h.insert_edge(x, best->id, best->weight);
    ++added;
  }
  return added;
}

// Fills dec and leaves the derived G / H (after the batch, or after its
// partial commit) in g / h, which start as copies of the state's.
void derive_deferred(const SparsifierState& state, const UpdateStream& stream,
                     std::uint32_t b, std::vector<std::uint8_t>& dec, DynamicGraph& g,
                     DynamicGraph& h) {
  const SparsifierOptions& opt = state.options();
  const std::uint64_t counter = state.update_counter();
  std::vector<std::size_t> pos;
  for (std::size_t i = 0; i < stream.events.size(); ++i)
    if (stream.events[i].batch_index == b) pos.push_back(i);
  dec.assign(pos.size(), kNone);
  for (std::size_t p : pos)
    if (!shape_ok(stream.events[p], g.vertex_count())) return;
  const bool filtering = opt.walk.distortion_threshold != 0.0 && !opt.freeze_sparsifier;
  // :415-423
  const DynamicGraph h0 = h;
  DynamicGraph shadow = g;
  for (std::size_t p : pos) {
    const EdgeEvent& e = stream.events[p];
    if (e.kind == EdgeEvent::Kind::Deletion && shadow.has_edge(e.u, e.v))
      shadow.delete_edge(e.u, e.v);
  }
  // :425-457
  constexpr std::size_t kNoSlot = static_cast<std::size_t>(-1);
  std::vector<std::size_t> slot(pos.size(), kNoSlot);
  std::vector<WalkQuery> ins, del;
  for (std::size_t k = 0; k < pos.size(); ++k) {
    const EdgeEvent& e = stream.events[pos[k]];
    WalkQuery q;
    q.p = e.u;
    q.q = e.v;
    q.update_id = counter + k;
    if (e.kind == EdgeEvent::Kind::Insertion) {
      if (!filtering || h0.degree(e.u) == 0 || h0.degree(e.v) == 0) continue;
      q.kind = WalkQuery::Kind::Reach;
      q.w_pq = g.edge_weight(e.u, e.v) + e.weight;
      slot[k] = ins.size();
      ins.push_back(q);
    } else {
      if (opt.freeze_sparsifier || !h0.has_edge(e.u, e.v)) continue;
      if (shadow.degree(e.u) == 0 || shadow.degree(e.v) == 0) continue;
      q.kind = WalkQuery::Kind::MinPath;
      slot[k] = del.size();
      del.push_back(q);
    }
  }
  WalkConfig dcfg = opt.walk;
  dcfg.distortion_threshold = std::numeric_limits<double>::infinity();
  const auto ri = run_batch(h0, ins, opt.walk);
  const auto rd = run_batch(shadow, del, dcfg);
  // :466-533, in event order on the live copies.
  for (std::size_t k = 0; k < pos.size(); ++k) {
    const EdgeEvent& e = stream.events[pos[k]];
    try {
      if (e.kind == EdgeEvent::Kind::Insertion) {
        g.insert_edge(e.u, e.v, e.weight);
        const bool have = slot[k] != kNoSlot;
        const bool reached = have && ri[slot[k]].verdict.reached;
        std::uint8_t d = kKept;
        if (opt.freeze_sparsifier) {
          d = kPruned;
        } else {
          if (opt.walk.distortion_threshold != 0.0 && have && reached) d = kPruned;
          const double total = g.edge_weight(e.u, e.v);
          if (h.has_edge(e.u, e.v)) set_weight(h, e.u, e.v, total);
          else if (d == kKept) h.insert_edge(e.u, e.v, total);
        }
        dec[k] = d;
      } else {
        g.delete_edge(e.u, e.v);
        std::uint8_t d = kGraphOnly;
        if (h.has_edge(e.u, e.v)) {
          h.delete_edge(e.u, e.v);
          d = kLocalFallback;
          if (!opt.freeze_sparsifier) {
            const RecoveredPath* path =
                slot[k] != kNoSlot && rd[slot[k]].path ? &*rd[slot[k]].path : nullptr;
            if (path) {
              for (std::size_t i = 0; i + 1 < path->vertices.size(); ++i) {
                const VertexId a = path->vertices[i], c = path->vertices[i + 1];
                if (!h.has_edge(a, c)) h.insert_edge(a, c, g.edge_weight(a, c));
              }
              d = kPathRecovered;
            } else {
              local_fallback(g, h, e.u, e.v);
            }
          }
        }
        dec[k] = d;
      }
    } catch (const Error&) {
      return;  // this event and the later ones did not commit (:525-529)
    }
  }
}

}  // namespace

BatchReport replay_batch_with_decisions(SparsifierState& state, const UpdateStream& stream,
                                        std::uint32_t b, std::vector<std::uint8_t>& dec) {
  const std::uint32_t n = state.graph().vertex_count();
  if (!state.options().batched) {
    // Immediate mode: the reference's own apply_* on a copy of the state.
    SparsifierState sim = state;
    dec.clear();
    for (const EdgeEvent& e : stream.events) {
      if (e.batch_index != b) continue;
      dec.push_back(kNone);
      if (!shape_ok(e, n)) break;
      try {
        if (e.kind == EdgeEvent::Kind::Insertion) {
          dec.back() = sim.apply_insertion(e.u, e.v, e.weight) == InsertionDecision::Kept
                           ? kKept : kPruned;
        } else {
          dec.back() = static_cast<std::uint8_t>(
              kGraphOnly + static_cast<int>(sim.apply_deletion(e.u, e.v).kind));
        }
      } catch (const Error&) {
        break;
      }
    }
    std::size_t nb = 0;
    for (const EdgeEvent& e : stream.events) nb += e.batch_index == b;
    dec.resize(nb, kNone);
    auto pinned = [&] {
      if (!same_rows(sim.graph(), state.graph()) ||
          !same_rows(sim.sparsifier(), state.sparsifier()))
        throw std::logic_error("decision derivation diverged from the reference (immediate)");
    };
    BatchReport r;
    try {
      r = state.replay_batch(stream, b);
    } catch (const Error&) {
      pinned();
      throw;
    }
    pinned();
    return r;
  }
  DynamicGraph g = state.graph();
  DynamicGraph h = state.sparsifier();
  derive_deferred(state, stream, b, dec, g, h);
  auto pinned = [&] {
    if (!same_rows(g, state.graph()) || !same_rows(h, state.sparsifier()))
      throw std::logic_error("decision derivation diverged from the reference (deferred)");
  };
  BatchReport r;
  try {
    r = state.replay_batch(stream, b);
  } catch (const Error&) {
    pinned();  // the partial commit (:525-529) must match too
    throw;
  }
  pinned();
  return r;
}

}  // namespace dyg_oracle
