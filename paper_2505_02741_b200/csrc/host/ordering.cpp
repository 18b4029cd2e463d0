// ordering.cpp -- see ordering.hpp.
//
// Each piece (a vertex set of the induced subgraph) is split by the middle
// level of a breadth-first level structure rooted at a pseudo-peripheral
// vertex: levels below the middle form one half, levels above the other, and
// the middle level -- trimmed to the vertices that touch the upper half --
// is the separator, ordered after both halves. Disconnected pieces are split
// into their components first; pieces of at most kLeaf vertices are emitted
// in breadth-first order. On 2-D meshes the separators are O(sqrt n) level
// lines, the classic nested-dissection fill O(n log n); the whole ordering
// is a few breadth-first sweeps per recursion level, O(n log n) time.
#include "ordering.hpp"

#include <algorithm>

namespace dyg {

namespace {

constexpr int kLeaf = 64;

struct Nd {
  int m;
  const int* rp;
  const int* ci;
  std::vector<int> mark;   // piece label of each vertex (-1: emitted)
  std::vector<int> level;  // BFS level within the current piece
  std::vector<int> queue;
  std::vector<int> out;
  int next_label = 1;

  // BFS over the piece labelled `lab` from `root`; fills queue[0..n) in
  // visit order and level[]. Returns the number reached.
  int bfs(int root, int lab) {
    int head = 0, tail = 0;
    queue[tail++] = root;
    level[root] = 0;
    mark[root] = -2 - lab;  // "seen" while this sweep runs
    while (head < tail) {
      const int u = queue[head++];
      for (int i = rp[u]; i < rp[u + 1]; ++i) {
        const int v = ci[i];
        if (mark[v] == lab) {
          mark[v] = -2 - lab;
          level[v] = level[u] + 1;
          queue[tail++] = v;
        }
      }
    }
    for (int i = 0; i < tail; ++i) mark[queue[i]] = lab;
    return tail;
  }

  // Order the piece whose vertices are `verts` (all marked `lab`).
  void order(std::vector<int> verts, int lab) {
    const int n = static_cast<int>(verts.size());
    if (n == 0) return;
    if (n <= kLeaf) {
      const int got = bfs(verts[0], lab);
      if (got == n) {
        for (int i = 0; i < n; ++i) emit(queue[i]);
        return;
      }
    }
    // Components: the first one reached from verts[0]; the rest later.
    int got = bfs(verts[0], lab);
    if (got < n) {
      std::vector<int> comp(queue.begin(), queue.begin() + got);
      const int lc = next_label++;
      for (int v : comp) mark[v] = lc;
      std::vector<int> rest;
      rest.reserve(n - got);
      for (int v : verts)
        if (mark[v] == lab) rest.push_back(v);
      verts.clear();
      verts.shrink_to_fit();
      order(std::move(comp), lc);
      order(std::move(rest), lab);
      return;
    }
    if (n <= kLeaf) {  // connected small piece (bfs above already covered it)
      for (int i = 0; i < n; ++i) emit(queue[i]);
      return;
    }
    // Pseudo-peripheral root: two sweeps from the farthest vertex.
    int root = queue[n - 1];
    for (int sweep = 0; sweep < 2; ++sweep) {
      bfs(root, lab);
      root = queue[n - 1];
    }
    bfs(root, lab);
    const int depth = level[queue[n - 1]] + 1;
    if (depth < 3) {  // no useful separator (a near-clique): emit as is
      for (int i = 0; i < n; ++i) emit(queue[i]);
      return;
    }
    // Middle level: the first whose cumulative count reaches n / 2.
    std::vector<int> count(depth, 0);
    for (int i = 0; i < n; ++i) ++count[level[queue[i]]];
    int mid = 1, acc = 0;
    for (int l = 0; l < depth; ++l) {
      acc += count[l];
      if (acc >= n / 2) {
        mid = std::min(std::max(l, 1), depth - 2);
        break;
      }
    }
    const int la = next_label++, lb = next_label++;
    std::vector<int> a, b, sep;
    for (int i = 0; i < n; ++i) {
      const int v = queue[i];
      const int l = level[v];
      if (l < mid) {
        a.push_back(v);
      } else if (l > mid) {
        b.push_back(v);
      } else {
        bool touches_upper = false;
        for (int k = rp[v]; k < rp[v + 1] && !touches_upper; ++k) {
          const int w = ci[k];
          touches_upper = mark[w] == lab && level[w] == mid + 1;
        }
        (touches_upper ? sep : a).push_back(v);
      }
    }
    for (int v : a) mark[v] = la;
    for (int v : b) mark[v] = lb;
    for (int v : sep) mark[v] = -1;  // ordered last, out of both halves
    verts.clear();
    verts.shrink_to_fit();
    order(std::move(a), la);
    order(std::move(b), lb);
    for (int v : sep) out.push_back(v);
  }

  void emit(int v) {
    mark[v] = -1;
    out.push_back(v);
  }
};

}  // namespace

std::vector<int> nested_dissection_order(int m, const int* row_ptr, const int* cols) {
  Nd nd;
  nd.m = m;
  nd.rp = row_ptr;
  nd.ci = cols;
  nd.mark.assign(m, 0);
  nd.level.assign(m, 0);
  nd.queue.assign(m, 0);
  nd.out.reserve(m);
  std::vector<int> all(m);
  for (int i = 0; i < m; ++i) all[i] = i;
  nd.order(std::move(all), 0);
  return nd.out;
}

}  // namespace dyg
