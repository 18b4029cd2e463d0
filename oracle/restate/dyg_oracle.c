/*
 * dyg_oracle.c -- plain-C restatement of the dyGRASS batched update path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/oracle_abi.h). This is the CPU
 * oracle the GPU product is checked against; it is never linked into or
 * called by paper_2505_02741_b200/. It restates, single-threaded, the
 * reference's algorithm for the hot path plus the input
 * generators the benchmark configs need. Every function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/). It is pinned by tests/test_oracle.py against
 * oracle/_ref (the reference compiled unmodified) and the committed golden
 * vectors in tests/golden/.
 *
 * Not restated (reference-only in the oracle ABI): MatrixMarket and stream
 * file I/O (host formats; the product's C++ host loader is checked against
 * oracle/_ref directly).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../oracle_abi.h"

/* ---------------------------------------------------------------- errors */
/* error.hpp:9 ErrorKind { Usage = 1, Data = 2, Numeric = 3 } */
enum { E_OK = 0, E_USAGE = 1, E_DATA = 2, E_NUMERIC = 3 };
static __thread char g_err[512];
static __thread int g_err_kind;

static int set_err(int kind, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  g_err_kind = kind;
  return kind;
}
const char* orc_last_error(void) { return g_err; }
int orc_last_error_kind(void) { return g_err_kind; }
const char* orc_impl_name(void) { return "restate"; }

/* ------------------------------------------------------------------- rng */
#define GAMMA 0x9E3779B97F4A7C15ull
/* rng.hpp:37-41 hash_mix */
static uint64_t hash_mix(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
/* rng.hpp:7-13 splitmix64_next: state += gamma; return mix(state) */
typedef struct { uint64_t state; } rng_t;
static uint64_t rng_next(rng_t* r) {
  r->state += GAMMA;
  return hash_mix(r->state);
}
/* rng.hpp:24 next_double: (next() >> 11) * 2^-53 */
static double rng_next_double(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:28-31 next_below: Lemire multiply-shift */
static uint64_t rng_next_below(rng_t* r, uint64_t bound) {
  return (uint64_t)(((unsigned __int128)rng_next(r) * bound) >> 64);
}
/* rng.hpp:45-50 walker_seed */
uint64_t orc_walker_seed(uint64_t global_seed, uint64_t update_id, uint64_t walker) {
  uint64_t h = hash_mix(global_seed + 0x9E3779B97F4A7C15ull);
  h = hash_mix(h ^ (update_id + 0xBF58476D1CE4E5B9ull));
  return hash_mix(h ^ (walker + 0x94D049BB133111EBull));
}

/* ----------------------------------------------------------------- graph */
/* graph.hpp:14-17 Neighbor; graph.hpp:65 vector<vector<Neighbor>> */
typedef struct { uint32_t id; double w; } nb_t;
typedef struct { nb_t* a; uint32_t n, cap; } row_t;
typedef struct {
  uint32_t n;
  row_t* rows;
  uint64_t edge_count;
  double total_weight;
} graph_t;

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  return p;
}

void* orc_graph_new(uint32_t n) {
  if (n == 0) { set_err(E_USAGE, "graph must have at least one vertex"); return NULL; }
  graph_t* g = xmalloc(sizeof *g);
  g->n = n;
  g->rows = calloc(n, sizeof(row_t));
  g->edge_count = 0;
  g->total_weight = 0.0;
  return g;
}
void* orc_graph_clone(const void* gp) {
  const graph_t* g = gp;
  graph_t* c = xmalloc(sizeof *c);
  *c = *g;
  c->rows = xmalloc((size_t)g->n * sizeof(row_t));
  for (uint32_t u = 0; u < g->n; ++u) {
    c->rows[u].n = g->rows[u].n;
    c->rows[u].cap = g->rows[u].n;
    c->rows[u].a = g->rows[u].n ? xmalloc(g->rows[u].n * sizeof(nb_t)) : NULL;
    if (g->rows[u].n) memcpy(c->rows[u].a, g->rows[u].a, g->rows[u].n * sizeof(nb_t));
  }
  return c;
}
void orc_graph_free(void* gp) {
  graph_t* g = gp;
  if (!g) return;
  for (uint32_t u = 0; u < g->n; ++u) free(g->rows[u].a);
  free(g->rows);
  free(g);
}
uint32_t orc_graph_n(const void* g) { return ((const graph_t*)g)->n; }
uint64_t orc_graph_edges(const void* g) { return ((const graph_t*)g)->edge_count; }
/* graph.cpp:114-116 density = |E|/|V| - 1 */
static double g_density(const graph_t* g) {
  return (double)g->edge_count / (double)g->n - 1.0;
}
double orc_graph_density(const void* g) { return g_density(g); }

static int check_vertex(const graph_t* g, uint32_t u) {
  if (u >= g->n) return set_err(E_USAGE, "vertex id %u out of range (n = %u)", u, g->n);
  return 0;
}
/* graph.cpp:34-46 find: first entry of row u with id v */
static nb_t* g_find(const graph_t* g, uint32_t u, uint32_t v) {
  row_t* r = &g->rows[u];
  for (uint32_t i = 0; i < r->n; ++i)
    if (r->a[i].id == v) return &r->a[i];
  return NULL;
}
/* graph.cpp:48-53 has_edge scans the smaller row */
static int g_has_edge(const graph_t* g, uint32_t u, uint32_t v) {
  if (g->rows[u].n > g->rows[v].n) { uint32_t t = u; u = v; v = t; }
  return g_find(g, u, v) != NULL;
}
/* graph.cpp:55-62 edge_weight (0.0 when absent) */
static double g_edge_weight(const graph_t* g, uint32_t u, uint32_t v) {
  if (g->rows[u].n > g->rows[v].n) { uint32_t t = u; u = v; v = t; }
  const nb_t* nb = g_find(g, u, v);
  return nb ? nb->w : 0.0;
}
double orc_graph_edge_weight(const void* g, uint32_t u, uint32_t v) {
  return g_edge_weight(g, u, v);
}
static void row_push(row_t* r, uint32_t id, double w) {
  if (r->n == r->cap) {
    r->cap = r->cap ? r->cap * 2 : 4;
    nb_t* a = xmalloc(r->cap * sizeof(nb_t));
    if (r->n) memcpy(a, r->a, r->n * sizeof(nb_t));
    free(r->a);
    r->a = a;
  }
  r->a[r->n].id = id;
  r->a[r->n].w = w;
  r->n++;
}
/* graph.cpp:64-85 insert_edge: validate; coalesce in place (row u entry
 * += w, mirror = same) or push_back to row u then row v. Returns 0 New,
 * 1 Coalesced, or -kind on error. */
static int g_insert(graph_t* g, uint32_t u, uint32_t v, double w) {
  int e;
  if ((e = check_vertex(g, u)) || (e = check_vertex(g, v))) return -e;
  if (u == v) return -set_err(E_USAGE, "self-loops are not allowed");
  if (!(w > 0.0) || !isfinite(w))
    return -set_err(E_USAGE, "edge weight must be a positive finite number");
  nb_t* nb = g_find(g, u, v);
  if (nb) {
    nb->w += w;
    g_find(g, v, u)->w = nb->w;
    g->total_weight += w;
    return 1;
  }
  row_push(&g->rows[u], v, w);
  row_push(&g->rows[v], u, w);
  g->edge_count++;
  g->total_weight += w;
  return 0;
}
/* graph.cpp:87-112 delete_edge: find in row u, swap-with-last + pop in row
 * u, then in row v. Data error when absent. */
static void row_remove(row_t* r, uint32_t b) {
  for (uint32_t i = 0; i < r->n; ++i) {
    if (r->a[i].id == b) {
      r->a[i] = r->a[r->n - 1];
      r->n--;
      return;
    }
  }
}
static int g_delete(graph_t* g, uint32_t u, uint32_t v, double* removed) {
  int e;
  if ((e = check_vertex(g, u)) || (e = check_vertex(g, v))) return e;
  nb_t* nb = g_find(g, u, v);
  if (!nb) return set_err(E_DATA, "edge (%u, %u) does not exist", u, v);
  double w = nb->w;
  row_remove(&g->rows[u], v);
  row_remove(&g->rows[v], u);
  g->edge_count--;
  g->total_weight -= w;
  if (removed) *removed = w;
  return 0;
}
int orc_graph_insert(void* g, uint32_t u, uint32_t v, double w) {
  int r = g_insert(g, u, v, w);
  return r < 0 ? -r : 0;
}
int orc_graph_delete(void* g, uint32_t u, uint32_t v) { return g_delete(g, u, v, NULL); }
void orc_graph_export(const void* gp, uint64_t* row_ptr, uint32_t* ids, double* w) {
  const graph_t* g = gp;
  uint64_t at = 0;
  for (uint32_t u = 0; u < g->n; ++u) {
    row_ptr[u] = at;
    for (uint32_t i = 0; i < g->rows[u].n; ++i, ++at) {
      ids[at] = g->rows[u].a[i].id;
      w[at] = g->rows[u].a[i].w;
    }
  }
  row_ptr[g->n] = at;
}

/* graph.cpp:118-126 edges(): u < v, vertex order then row order */
typedef struct { uint32_t u, v; double w; } edge_t;
static edge_t* g_edges(const graph_t* g, size_t* count) {
  edge_t* out = xmalloc(g->edge_count * sizeof(edge_t));
  size_t k = 0;
  for (uint32_t u = 0; u < g->n; ++u)
    for (uint32_t i = 0; i < g->rows[u].n; ++i)
      if (u < g->rows[u].a[i].id) {
        out[k].u = u;
        out[k].v = g->rows[u].a[i].id;
        out[k].w = g->rows[u].a[i].w;
        ++k;
      }
  *count = k;
  return out;
}

/* graph.cpp:162-195 connected_components / is_connected (DFS stack) */
static int g_is_connected(const graph_t* g) {
  uint32_t* label = xmalloc((size_t)g->n * sizeof(uint32_t));
  uint32_t* stack = xmalloc((size_t)g->n * sizeof(uint32_t) + 4);
  memset(label, 0xFF, (size_t)g->n * sizeof(uint32_t));
  uint32_t comps = 0;
  for (uint32_t s = 0; s < g->n; ++s) {
    if (label[s] != 0xFFFFFFFFu) continue;
    size_t top = 0;
    label[s] = comps;
    stack[top++] = s;
    while (top) {
      uint32_t u = stack[--top];
      for (uint32_t i = 0; i < g->rows[u].n; ++i) {
        uint32_t x = g->rows[u].a[i].id;
        if (label[x] == 0xFFFFFFFFu) { label[x] = comps; stack[top++] = x; }
      }
    }
    ++comps;
  }
  free(label);
  free(stack);
  return comps <= 1;
}

/* ------------------------------------------------------------ generators */
/* tests/support/generators.hpp:65-86 make_mesh */
static graph_t* make_mesh_impl(uint32_t rows, uint32_t cols, uint64_t seed, double w_min,
                               double w_max, int diagonals) {
  graph_t* g = orc_graph_new(rows * cols);
  if (!g) return NULL;
  rng_t rng = {hash_mix(seed + 0x3E5Bull)};
#define WEIGHT() (w_min + rng_next_double(&rng) * (w_max - w_min))
  for (uint32_t r = 0; r < rows; ++r) {
    for (uint32_t c = 0; c < cols; ++c) {
      uint32_t id = r * cols + c;
      if (c + 1 < cols) g_insert(g, id, id + 1, WEIGHT());
      if (r + 1 < rows) g_insert(g, id, id + cols, WEIGHT());
      if (diagonals && r + 1 < rows && c + 1 < cols) {
        if (rng_next(&rng) & 1u) {
          g_insert(g, id, id + cols + 1, WEIGHT());
        } else {
          g_insert(g, id + 1, id + cols, WEIGHT());
        }
      }
    }
  }
#undef WEIGHT
  return g;
}
void* orc_make_mesh(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max) {
  return make_mesh_impl(rows, cols, seed, w_min, w_max, 1);
}
/* SURVEY.md 8(d) C4 grid4 = make_mesh without the diagonal draw */
void* orc_make_grid4(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max) {
  return make_mesh_impl(rows, cols, seed, w_min, w_max, 0);
}
/* tests/support/generators.hpp:37-61 make_random_connected */
void* orc_make_random_connected(uint32_t n, uint32_t extra, uint64_t seed, double w_min,
                                double w_max, int with_pendant) {
  graph_t* g = orc_graph_new(n);
  if (!g) return NULL;
  rng_t rng = {hash_mix(seed + 0x57A77ull)};
#define WEIGHT() (w_min + rng_next_double(&rng) * (w_max - w_min))
  const uint32_t core = with_pendant ? n - 1 : n;
  /* generators.hpp:46 passes rng.next_below(v) and weight() as arguments of
   * one call; GCC evaluates them right to left, so the weight is drawn first. */
  for (uint32_t v = 1; v < core; ++v) {
    const double w = WEIGHT();
    uint32_t to = (uint32_t)rng_next_below(&rng, v);
    g_insert(g, v, to, w);
  }
  uint32_t added = 0, attempts = 0;
  while (added < extra && attempts < 100 * extra + 100) {
    ++attempts;
    uint32_t u = (uint32_t)rng_next_below(&rng, core);
    uint32_t v = (uint32_t)rng_next_below(&rng, core);
    if (u == v || g_has_edge(g, u, v)) continue;
    g_insert(g, u, v, WEIGHT());
    ++added;
  }
  if (with_pendant) {
    const double w = WEIGHT(); /* same right-to-left order (generators.hpp:58) */
    uint32_t to = (uint32_t)rng_next_below(&rng, core);
    g_insert(g, n - 1, to, w);
  }
#undef WEIGHT
  return g;
}

/* sparsifier.cpp:105-159 build_initial_sparsifier */
static int cmp_edge_desc(const void* a, const void* b) {
  /* sparsifier.cpp:114-117: weight desc, then (u, v) asc */
  const edge_t *x = a, *y = b;
  if (x->w != y->w) return x->w > y->w ? -1 : 1;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return 0;
}
typedef struct { double distortion; uint64_t tiebreak; size_t edge_index; } ranked_t;
static int cmp_ranked(const void* a, const void* b) {
  /* sparsifier.cpp:146-149: distortion desc, tiebreak asc */
  const ranked_t *x = a, *y = b;
  if (x->distortion != y->distortion) return x->distortion > y->distortion ? -1 : 1;
  if (x->tiebreak != y->tiebreak) return x->tiebreak < y->tiebreak ? -1 : 1;
  return 0;
}
static uint32_t dsu_find(uint32_t* parent, uint32_t x) {
  /* sparsifier.cpp:22-28 path halving */
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];
    x = parent[x];
  }
  return x;
}
void* orc_build_initial_sparsifier(const void* gp, double target_density, uint64_t seed) {
  const graph_t* g = gp;
  if (target_density < 0.0) { set_err(E_USAGE, "target density must be nonnegative"); return NULL; }
  if (!g_is_connected(g)) {
    set_err(E_DATA, "graph must be connected to build a sparsifier");
    return NULL;
  }
  const uint32_t n = g->n;
  size_t m = 0;
  edge_t* edges = g_edges(g, &m);
  qsort(edges, m, sizeof(edge_t), cmp_edge_desc);

  graph_t* h = orc_graph_new(n);
  uint32_t* parent = xmalloc((size_t)n * sizeof(uint32_t));
  for (uint32_t i = 0; i < n; ++i) parent[i] = i;
  size_t* off_tree = xmalloc(m * sizeof(size_t));
  size_t n_off = 0;
  for (size_t i = 0; i < m; ++i) {
    uint32_t a = dsu_find(parent, edges[i].u), b = dsu_find(parent, edges[i].v);
    if (a != b) {
      parent[a] = b; /* sparsifier.cpp:29-34 unite */
      g_insert(h, edges[i].u, edges[i].v, edges[i].w);
    } else {
      off_tree[n_off++] = i;
    }
  }
  free(parent);

  /* sparsifier.cpp:42-77 TreeResistance: BFS from 0 over the tree rows. */
  uint32_t* depth = calloc(n, sizeof(uint32_t));
  double* rr = calloc(n, sizeof(double));
  uint32_t* par = calloc(n, sizeof(uint32_t));
  uint8_t* visited = calloc(n, 1);
  uint32_t* queue = xmalloc((size_t)n * sizeof(uint32_t));
  size_t qh = 0, qt = 0;
  visited[0] = 1;
  queue[qt++] = 0;
  while (qh < qt) {
    uint32_t u = queue[qh++];
    for (uint32_t i = 0; i < h->rows[u].n; ++i) {
      const nb_t* nb = &h->rows[u].a[i];
      if (visited[nb->id]) continue;
      visited[nb->id] = 1;
      par[nb->id] = u;
      depth[nb->id] = depth[u] + 1;
      rr[nb->id] = rr[u] + 1.0 / nb->w;
      queue[qt++] = nb->id;
    }
  }
  uint32_t levels = 1;
  while ((1u << levels) < n) ++levels;
  uint32_t** up = xmalloc(levels * sizeof(uint32_t*));
  up[0] = par;
  for (uint32_t k = 1; k < levels; ++k) {
    up[k] = xmalloc((size_t)n * sizeof(uint32_t));
    for (uint32_t v = 0; v < n; ++v) up[k][v] = up[k - 1][up[k - 1][v]];
  }
  ranked_t* ranked = xmalloc((n_off ? n_off : 1) * sizeof(ranked_t));
  for (size_t j = 0; j < n_off; ++j) {
    const edge_t* e = &edges[off_tree[j]];
    /* sparsifier.cpp:80-95 lca by binary lifting */
    uint32_t u = e->u, v = e->v;
    if (depth[u] < depth[v]) { uint32_t t = u; u = v; v = t; }
    uint32_t gap = depth[u] - depth[v];
    for (uint32_t k = 0; gap != 0; ++k, gap >>= 1)
      if (gap & 1u) u = up[k][u];
    uint32_t lca;
    if (u == v) {
      lca = u;
    } else {
      for (uint32_t k = levels; k-- > 0;) {
        if (up[k][u] != up[k][v]) { u = up[k][u]; v = up[k][v]; }
      }
      lca = up[0][u];
    }
    /* sparsifier.cpp:74-77 between = R(u) + R(v) - 2 R(lca) */
    double between = rr[e->u] + rr[e->v] - 2.0 * rr[lca];
    ranked[j].distortion = e->w * between;
    ranked[j].tiebreak = hash_mix(seed ^ ((uint64_t)e->u << 32 | e->v));
    ranked[j].edge_index = off_tree[j];
  }
  qsort(ranked, n_off, sizeof(ranked_t), cmp_ranked);
  /* sparsifier.cpp:151-157 fill to target density */
  for (size_t j = 0; j < n_off; ++j) {
    double d = g_density(h);
    if ((d > 0.0 ? d : 0.0) >= target_density) break;
    const edge_t* e = &edges[ranked[j].edge_index];
    g_insert(h, e->u, e->v, e->w);
  }
  for (uint32_t k = 0; k < levels; ++k) free(up[k]);
  free(up);
  free(depth); free(rr); free(visited); free(queue); free(ranked); free(off_tree); free(edges);
  return h;
}

/* --------------------------------------------------------------- streams */
typedef struct {
  orc_event* ev;
  size_t n;
  uint32_t batch_count;
} stream_t;

/* open-addressing u64 set (stands in for std::unordered_set at
 * stream.cpp:128; only membership is observable) */
typedef struct { uint64_t* keys; size_t cap; size_t n; } u64set;
static void set_init(u64set* s, size_t want) {
  s->cap = 16;
  while (s->cap < want * 2 + 16) s->cap <<= 1;
  s->keys = xmalloc(s->cap * sizeof(uint64_t));
  memset(s->keys, 0xFF, s->cap * sizeof(uint64_t));
  s->n = 0;
}
static int set_has(const u64set* s, uint64_t k) {
  size_t i = hash_mix(k) & (s->cap - 1);
  while (s->keys[i] != UINT64_MAX) {
    if (s->keys[i] == k) return 1;
    i = (i + 1) & (s->cap - 1);
  }
  return 0;
}
static void set_add(u64set* s, uint64_t k) {
  size_t i = hash_mix(k) & (s->cap - 1);
  while (s->keys[i] != UINT64_MAX) {
    if (s->keys[i] == k) return;
    i = (i + 1) & (s->cap - 1);
  }
  s->keys[i] = k;
  s->n++;
}

/* stream.cpp:90-110 vertices_within: BFS, discovery order, excluding start */
static uint32_t* vertices_within(const graph_t* g, uint32_t start, uint32_t radius,
                                 uint32_t* dist, size_t* count) {
  for (uint32_t i = 0; i < g->n; ++i) dist[i] = UINT32_MAX;
  size_t cap = 64, k = 0, qh = 0, qt = 0;
  uint32_t* found = xmalloc(cap * sizeof(uint32_t));
  uint32_t* queue = xmalloc((size_t)g->n * sizeof(uint32_t));
  dist[start] = 0;
  queue[qt++] = start;
  while (qh < qt) {
    uint32_t u = queue[qh++];
    if (dist[u] == radius) continue;
    for (uint32_t i = 0; i < g->rows[u].n; ++i) {
      uint32_t x = g->rows[u].a[i].id;
      if (dist[x] != UINT32_MAX) continue;
      dist[x] = dist[u] + 1;
      if (k == cap) {
        cap *= 2;
        uint32_t* f = xmalloc(cap * sizeof(uint32_t));
        memcpy(f, found, k * sizeof(uint32_t));
        free(found);
        found = f;
      }
      found[k++] = x;
      queue[qt++] = x;
    }
  }
  free(queue);
  *count = k;
  return found;
}

/* stream.cpp:114-200 generate_update_stream */
void* orc_stream_generate(const void* gp, double insert_fraction, double delete_fraction,
                          uint32_t batches, uint64_t seed, uint32_t locality) {
  const graph_t* g = gp;
  if (insert_fraction < 0.0 || delete_fraction < 0.0) {
    set_err(E_USAGE, "update fractions must be nonnegative");
    return NULL;
  }
  if (batches == 0) { set_err(E_USAGE, "batch count must be positive"); return NULL; }
  const uint32_t n = g->n;
  const uint64_t insert_count = (uint64_t)llround(insert_fraction * (double)n);
  const uint64_t delete_count = (uint64_t)llround(delete_fraction * (double)g->edge_count);
  double wmin = INFINITY, wmax = 0.0;
  size_t m = 0;
  edge_t* edges = g_edges(g, &m);
  for (size_t i = 0; i < m; ++i) {
    if (edges[i].w < wmin) wmin = edges[i].w;
    if (edges[i].w > wmax) wmax = edges[i].w;
  }
  if (insert_count > 0 && m == 0) {
    free(edges);
    set_err(E_DATA, "cannot derive insertion weights from an edgeless graph");
    return NULL;
  }
  rng_t rng = {hash_mix(seed + 0x12345678ull)};
  stream_t* s = xmalloc(sizeof *s);
  s->ev = xmalloc((insert_count + delete_count + 1) * sizeof(orc_event));
  s->n = 0;
  u64set used;
  set_init(&used, insert_count);
  const uint64_t attempt_cap = 200 * (insert_count > 1 ? insert_count : 1) + 10000;
  uint64_t attempts = 0;
  uint32_t* dist = locality ? xmalloc((size_t)n * sizeof(uint32_t)) : NULL;
  for (uint64_t k = 0; k < insert_count; ++k) {
    uint32_t u = 0, v = 0;
    int found = 0;
    while (attempts < attempt_cap) {
      ++attempts;
      u = (uint32_t)rng_next_below(&rng, n);
      if (locality == 0) {
        v = (uint32_t)rng_next_below(&rng, n);
      } else {
        size_t cnt = 0;
        uint32_t* nearby = vertices_within(g, u, locality, dist, &cnt);
        if (cnt == 0) { free(nearby); continue; }
        v = nearby[rng_next_below(&rng, cnt)];
        free(nearby);
      }
      if (u == v) continue;
      uint32_t lo = u < v ? u : v, hi = u < v ? v : u;
      uint64_t key = (uint64_t)lo * n + hi;
      if (g_has_edge(g, u, v) || set_has(&used, key)) continue;
      set_add(&used, key);
      found = 1;
      break;
    }
    if (!found) {
      free(dist); free(used.keys); free(edges); free(s->ev); free(s);
      set_err(E_DATA, "could not sample enough non-edges (graph too dense?)");
      return NULL;
    }
    orc_event* e = &s->ev[s->n++];
    e->kind = 0;
    e->u = u < v ? u : v;
    e->v = u < v ? v : u;
    e->weight = wmin + rng_next_double(&rng) * (wmax - wmin);
    e->batch_index = (uint32_t)(k * batches / (insert_count > 1 ? insert_count : 1));
  }
  free(dist);
  free(used.keys);
  if (delete_count > g->edge_count) {
    free(edges); free(s->ev); free(s);
    set_err(E_DATA, "deletion fraction exceeds edge count");
    return NULL;
  }
  const uint32_t deletion_base = insert_count > 0 ? batches : 0;
  for (uint64_t k = 0; k < delete_count; ++k) {
    const uint64_t pick = k + rng_next_below(&rng, m - k);
    edge_t t = edges[k];
    edges[k] = edges[pick];
    edges[pick] = t;
    orc_event* e = &s->ev[s->n++];
    e->kind = 1;
    e->u = edges[k].u;
    e->v = edges[k].v;
    e->weight = 0.0;
    e->batch_index =
        deletion_base + (uint32_t)(k * batches / (delete_count > 1 ? delete_count : 1));
  }
  free(edges);
  s->batch_count = s->n ? s->ev[s->n - 1].batch_index + 1 : 0;
  return s;
}
void* orc_stream_from_events(const orc_event* ev, size_t n, uint32_t batch_count) {
  stream_t* s = xmalloc(sizeof *s);
  s->ev = xmalloc((n ? n : 1) * sizeof(orc_event));
  if (n) memcpy(s->ev, ev, n * sizeof(orc_event));
  s->n = n;
  s->batch_count = batch_count;
  return s;
}
size_t orc_stream_size(const void* s) { return ((const stream_t*)s)->n; }
uint32_t orc_stream_batches(const void* s) { return ((const stream_t*)s)->batch_count; }
void orc_stream_copy(const void* sp, orc_event* out) {
  const stream_t* s = sp;
  if (s->n) memcpy(out, s->ev, s->n * sizeof(orc_event));
}
void orc_stream_free(void* sp) {
  stream_t* s = sp;
  if (!s) return;
  free(s->ev);
  free(s);
}

/* ----------------------------------------------------------------- walks */
#define NO_VERTEX 0xFFFFFFFFu
enum { T_REACHED = 0, T_BUDGET = 1, T_CAP = 2, T_DEAD = 3 };
typedef struct {
  uint32_t* path;
  uint32_t len, cap;
  double acc;
  uint32_t terminal;
  uint32_t steps;
} trace_t;

static void trace_push(trace_t* t, uint32_t v) {
  if (t->len == t->cap) {
    t->cap = t->cap ? t->cap * 2 : 16;
    uint32_t* p = xmalloc(t->cap * sizeof(uint32_t));
    if (t->len) memcpy(p, t->path, t->len * sizeof(uint32_t));
    free(t->path);
    t->path = p;
  }
  t->path[t->len++] = v;
}

/* walk.cpp:17-37 sample_neighbor: pass 1 sums weights of entries whose id is
 * not `previous` in row order; no candidate -> NO_VERTEX (no draw); target =
 * next_double() * total; pass 2 stops at the first entry with
 * target < cumulative; rounding fallback is the last candidate. */
static uint32_t sample_neighbor(const graph_t* g, uint32_t u, uint32_t previous, rng_t* rng,
                                double* edge_weight) {
  const row_t* r = &g->rows[u];
  double total = 0.0;
  for (uint32_t i = 0; i < r->n; ++i)
    if (r->a[i].id != previous) total += r->a[i].w;
  if (total <= 0.0) return NO_VERTEX;
  const double target = rng_next_double(rng) * total;
  double cumulative = 0.0;
  const nb_t* last = NULL;
  for (uint32_t i = 0; i < r->n; ++i) {
    if (r->a[i].id == previous) continue;
    cumulative += r->a[i].w;
    last = &r->a[i];
    if (target < cumulative) break;
  }
  *edge_weight = last->w;
  return last->id;
}

/* walk.cpp:41-80 single_walk: cap checked at the loop top; after each
 * traversed edge: budget (w_pq * acc > budget) before target. */
static int single_walk(const graph_t* g, uint32_t p, uint32_t q, double w_pq, double budget,
                       uint32_t cap, rng_t* rng, trace_t* t, int keep_path) {
  memset(t, 0, sizeof *t);
  if (p == q) return set_err(E_USAGE, "walk endpoints must differ");
  if (p >= g->n) return set_err(E_USAGE, "vertex id %u out of range (n = %u)", p, g->n);
  if (g->rows[p].n == 0) return set_err(E_USAGE, "walk started at an isolated vertex");
  if (keep_path) trace_push(t, p);
  uint32_t current = p, previous = NO_VERTEX;
  for (;;) {
    if (t->steps >= cap) { t->terminal = T_CAP; return 0; }
    double w = 0.0;
    uint32_t next = sample_neighbor(g, current, previous, rng, &w);
    if (next == NO_VERTEX) { t->terminal = T_DEAD; return 0; }
    t->acc += 1.0 / w;
    ++t->steps;
    previous = current;
    current = next;
    if (keep_path) trace_push(t, current);
    if (w_pq * t->acc > budget) { t->terminal = T_BUDGET; return 0; }
    if (current == q) { t->terminal = T_REACHED; return 0; }
  }
}

int orc_single_walk(const void* g, uint32_t p, uint32_t q, double w_pq, double budget,
                    uint32_t cap, uint64_t rng_seed, uint32_t* terminal, uint32_t* steps,
                    double* acc, uint32_t* path, uint32_t path_cap, uint32_t* path_len) {
  rng_t rng = {rng_seed};
  trace_t t;
  int e = single_walk(g, p, q, w_pq, budget, cap, &rng, &t, 1);
  if (e) { free(t.path); return e; }
  *terminal = t.terminal;
  *steps = t.steps;
  *acc = t.acc;
  *path_len = t.len;
  for (uint32_t i = 0; i < t.len && i < path_cap; ++i) path[i] = t.path[i];
  free(t.path);
  return 0;
}

/* walk.cpp:82-98 nbrw_reach: all s walkers run to completion, in order;
 * reached = any; best = strict-< minimum; steps_used = sum. */
static int nbrw_reach(const graph_t* g, uint32_t p, uint32_t q, double w_pq,
                      const orc_walk_config* cfg, uint64_t update_id, orc_result* out) {
  memset(out, 0, sizeof *out);
  for (uint32_t i = 0; i < cfg->walker_count; ++i) {
    rng_t rng = {orc_walker_seed(cfg->global_seed, update_id, i)};
    trace_t t;
    int e = single_walk(g, p, q, w_pq, cfg->distortion_threshold, cfg->step_cap, &rng, &t, 0);
    if (e) return e;
    out->steps_used += t.steps;
    if (t.terminal != T_REACHED) continue;
    if (!out->reached || t.acc < out->best_estimate) out->best_estimate = t.acc;
    out->reached = 1;
  }
  return 0;
}

/* walk.cpp:100-117 loop_erase: keep first visits; a revisit truncates the
 * erased list back to the earlier occurrence. The position map is the
 * erased list itself (entries are unique). */
size_t orc_loop_erase(const uint32_t* path, size_t n, uint32_t* out) {
  size_t len = 0;
  for (size_t i = 0; i < n; ++i) {
    size_t j = 0;
    while (j < len && out[j] != path[i]) ++j;
    if (j < len) {
      len = j + 1;
    } else {
      out[len++] = path[i];
    }
  }
  return len;
}

/* walk.cpp:119-145 nbrw_min_path: w_pq = 1, caller's budget; winner = first
 * walker attaining the strict minimum; loop-erase; resistance recomputed as
 * sum of 1/edge_weight along the erased path, in path order. */
static int nbrw_min_path(const graph_t* g, uint32_t p, uint32_t q, const orc_walk_config* cfg,
                         uint64_t update_id, orc_result* out, uint32_t* path_out) {
  memset(out, 0, sizeof *out);
  trace_t best;
  int have = 0;
  memset(&best, 0, sizeof best);
  for (uint32_t i = 0; i < cfg->walker_count; ++i) {
    rng_t rng = {orc_walker_seed(cfg->global_seed, update_id, i)};
    trace_t t;
    int e = single_walk(g, p, q, 1.0, cfg->distortion_threshold, cfg->step_cap, &rng, &t, 1);
    if (e) { free(best.path); return e; }
    out->steps_used += t.steps;
    if (t.terminal == T_REACHED && (!have || t.acc < best.acc)) {
      free(best.path);
      best = t;
      have = 1;
    } else {
      free(t.path);
    }
  }
  if (!have) return 0;
  uint32_t* erased = xmalloc(best.len * sizeof(uint32_t));
  size_t len = orc_loop_erase(best.path, best.len, erased);
  out->reached = 1;
  out->path_len = (uint32_t)len;
  out->resistance = 0.0;
  for (size_t i = 0; i + 1 < len; ++i) out->resistance += 1.0 / g_edge_weight(g, erased[i], erased[i + 1]);
  if (path_out) memcpy(path_out, erased, len * sizeof(uint32_t));
  free(erased);
  free(best.path);
  return 0;
}

/* walk.cpp:157-193 run_batch (single worker: results are worker-count
 * independent by construction, walk.hpp:86-88). */
int orc_run_batch(const void* gp, const orc_query* q, size_t nq, const orc_walk_config* cfg,
                  unsigned workers, orc_result* out, uint32_t* path_buf) {
  (void)workers;
  const graph_t* g = gp;
  const size_t stride = (size_t)cfg->step_cap + 1;
  for (size_t i = 0; i < nq; ++i) {
    int e;
    if (q[i].kind == 0) {
      e = nbrw_reach(g, q[i].p, q[i].q, q[i].w_pq, cfg, q[i].update_id, &out[i]);
    } else {
      e = nbrw_min_path(g, q[i].p, q[i].q, cfg, q[i].update_id, &out[i],
                        path_buf ? path_buf + i * stride : NULL);
    }
    if (e) return e;
  }
  return 0;
}

/* ------------------------------------------------------- SparsifierState */
typedef struct {
  graph_t* g;
  graph_t* h;
  orc_walk_config walk;
  int batched, freeze;
  uint64_t update_counter;
  uint64_t last_event_steps;
} state_t;

/* sparsifier.cpp:183-203 constructor checks */
void* orc_state_new(const void* gp, const void* hp, const orc_walk_config* cfg, int batched,
                    int freeze) {
  const graph_t *g = gp, *h = hp;
  if (g->n != h->n) { set_err(E_USAGE, "graph and sparsifier must share a vertex set"); return NULL; }
  if (cfg->distortion_threshold < 0.0 || cfg->step_cap == 0 || cfg->walker_count == 0) {
    set_err(E_USAGE, "invalid walk configuration");
    return NULL;
  }
  for (uint32_t u = 0; u < h->n; ++u)
    for (uint32_t i = 0; i < h->rows[u].n; ++i) {
      uint32_t v = h->rows[u].a[i].id;
      if (u < v && !g_has_edge(g, u, v)) {
        set_err(E_DATA, "sparsifier edge (%u, %u) missing from the graph", u, v);
        return NULL;
      }
    }
  state_t* st = xmalloc(sizeof *st);
  st->g = orc_graph_clone(g);
  st->h = orc_graph_clone(h);
  st->walk = *cfg;
  st->batched = batched;
  st->freeze = freeze;
  st->update_counter = 0;
  st->last_event_steps = 0;
  return st;
}
void orc_state_free(void* sp) {
  state_t* st = sp;
  if (!st) return;
  orc_graph_free(st->g);
  orc_graph_free(st->h);
  free(st);
}
const void* orc_state_graph(const void* st) { return ((const state_t*)st)->g; }
const void* orc_state_sparsifier(const void* st) { return ((const state_t*)st)->h; }
uint64_t orc_state_update_counter(const void* st) { return ((const state_t*)st)->update_counter; }

/* sparsifier.cpp:207-216 set_edge_weight: up -> coalesce by the
 * difference; down -> delete and reinsert (moves to the row ends). */
static void set_edge_weight(graph_t* h, uint32_t u, uint32_t v, double target) {
  const double current = g_edge_weight(h, u, v);
  if (target > current) {
    g_insert(h, u, v, target - current);
  } else if (target < current) {
    g_delete(h, u, v, NULL);
    g_insert(h, u, v, target);
  }
}

/* sparsifier.cpp:220-241 commit_insertion; returns 1 Kept, 0 Pruned */
static int commit_insertion(state_t* st, uint32_t u, uint32_t v, int have_verdict,
                            int reached) {
  if (st->freeze) return 0;
  const double total = g_edge_weight(st->g, u, v);
  int kept = 1;
  if (st->walk.distortion_threshold != 0.0 && have_verdict && reached) kept = 0;
  if (g_has_edge(st->h, u, v)) {
    set_edge_weight(st->h, u, v, total);
  } else if (kept) {
    g_insert(st->h, u, v, total);
  }
  return kept;
}

/* sparsifier.cpp:264-280 run_local_fallback: for u then v, an H-isolated
 * endpoint with G neighbours gets its max-weight G edge (tie -> lowest id). */
static uint32_t run_local_fallback(state_t* st, uint32_t u, uint32_t v) {
  uint32_t added = 0;
  const uint32_t ends[2] = {u, v};
  for (int k = 0; k < 2; ++k) {
    uint32_t x = ends[k];
    if (st->h->rows[x].n != 0 || st->g->rows[x].n == 0) continue;
    const nb_t* best = NULL;
    const row_t* r = &st->g->rows[x];
    for (uint32_t i = 0; i < r->n; ++i) {
      const nb_t* nb = &r->a[i];
      if (!best || nb->w > best->w || (nb->w == best->w && nb->id < best->id)) best = nb;
    }
    g_insert(st->h, x, best->id, best->w);
    ++added;
  }
  return added;
}

enum { D_GRAPH_ONLY = 0, D_PATH = 1, D_FALLBACK = 2 };

/* sparsifier.cpp:243-262 apply_insertion (immediate mode) */
static int apply_insertion(state_t* st, uint32_t u, uint32_t v, double w, int* kept) {
  int r = g_insert(st->g, u, v, w);
  if (r < 0) return -r;
  const uint64_t update_id = st->update_counter++;
  st->last_event_steps = 0;
  int have_verdict = 0, reached = 0;
  const int filtering = st->walk.distortion_threshold != 0.0 && !st->freeze;
  if (filtering && st->h->rows[u].n > 0 && st->h->rows[v].n > 0) {
    const double total = g_edge_weight(st->g, u, v);
    orc_result res;
    int e = nbrw_reach(st->h, u, v, total, &st->walk, update_id, &res);
    if (e) return e;
    st->last_event_steps = res.steps_used;
    have_verdict = 1;
    reached = (int)res.reached;
  }
  *kept = commit_insertion(st, u, v, have_verdict, reached);
  return 0;
}

/* sparsifier.cpp:282-317 apply_deletion (immediate mode) */
static int apply_deletion(state_t* st, uint32_t u, uint32_t v, int* kind, uint32_t* added) {
  int e = g_delete(st->g, u, v, NULL);
  if (e) return e;
  const uint64_t update_id = st->update_counter++;
  st->last_event_steps = 0;
  *added = 0;
  if (!g_has_edge(st->h, u, v)) { *kind = D_GRAPH_ONLY; return 0; }
  g_delete(st->h, u, v, NULL);
  if (st->freeze) { *kind = D_FALLBACK; return 0; }
  if (st->g->rows[u].n > 0 && st->g->rows[v].n > 0) {
    orc_walk_config cfg = st->walk;
    cfg.distortion_threshold = INFINITY;
    orc_result res;
    uint32_t* path = xmalloc(((size_t)cfg.step_cap + 1) * sizeof(uint32_t));
    e = nbrw_min_path(st->g, u, v, &cfg, update_id, &res, path);
    if (e) { free(path); return e; }
    st->last_event_steps = res.steps_used;
    if (res.reached) {
      *kind = D_PATH;
      for (uint32_t i = 0; i + 1 < res.path_len; ++i) {
        uint32_t a = path[i], b = path[i + 1];
        if (!g_has_edge(st->h, a, b)) {
          g_insert(st->h, a, b, g_edge_weight(st->g, a, b));
          ++*added;
        }
      }
      free(path);
      return 0;
    }
    free(path);
  }
  *kind = D_FALLBACK;
  *added = run_local_fallback(st, u, v);
  return 0;
}

/* sparsifier.cpp:321-337 validate_event_shape */
static int validate_event_shape(const orc_event* e, uint32_t n, size_t pos) {
  if (e->u >= n || e->v >= n) return set_err(E_DATA, "event %zu: vertex id out of range", pos);
  if (e->u == e->v) return set_err(E_DATA, "event %zu: self-loop", pos);
  if (e->kind == 0 && (!(e->weight > 0.0) || !isfinite(e->weight)))
    return set_err(E_DATA, "event %zu: non-positive weight", pos);
  return 0;
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* sparsifier.cpp:380-384 error rewrap: "event <pos>: <what>", kind Data
 * unless Numeric. */
static int rewrap(int kind, size_t pos) {
  char tmp[512];
  snprintf(tmp, sizeof tmp, "%s", g_err);
  set_err(kind == E_NUMERIC ? E_NUMERIC : E_DATA, "event %zu: %s", pos, tmp);
  return kind == E_NUMERIC ? E_NUMERIC : E_DATA;
}

/* sparsifier.cpp:347-393 replay_batch_immediate */
static int replay_immediate(state_t* st, const stream_t* s, uint32_t b, orc_report* rep) {
  const double start = now_ms();
  for (size_t i = 0; i < s->n; ++i) {
    const orc_event* ev = &s->ev[i];
    if (ev->batch_index != b) continue;
    int e = validate_event_shape(ev, st->g->n, i);
    if (e) return rewrap(e, i);
    if (ev->kind == 0) {
      rep->insertions_seen++;
      int kept = 0;
      e = apply_insertion(st, ev->u, ev->v, ev->weight, &kept);
      if (e) return rewrap(e, i);
      if (kept) rep->insertions_kept++; else rep->insertions_pruned++;
    } else {
      rep->deletions_seen++;
      int kind = 0;
      uint32_t added = 0;
      e = apply_deletion(st, ev->u, ev->v, &kind, &added);
      if (e) return rewrap(e, i);
      if (kind != D_GRAPH_ONLY) rep->deletions_in_sparsifier++;
      if (kind == D_PATH) {
        rep->paths_recovered++;
        rep->edges_recovered += added;
      } else if (kind == D_FALLBACK) {
        rep->fallback_activations++;
        rep->edges_recovered += added;
      }
    }
    rep->walker_steps += st->last_event_steps;
    if (st->last_event_steps > rep->max_event_steps) rep->max_event_steps = st->last_event_steps;
  }
  rep->wall_ms = now_ms() - start;
  return 0;
}

/* sparsifier.cpp:395-539 replay_batch_deferred */
static int replay_deferred(state_t* st, const stream_t* s, uint32_t b, orc_report* rep) {
  const double start = now_ms();
  size_t np = 0;
  for (size_t i = 0; i < s->n; ++i)
    if (s->ev[i].batch_index == b) ++np;
  size_t* pos = xmalloc((np ? np : 1) * sizeof(size_t));
  np = 0;
  for (size_t i = 0; i < s->n; ++i)
    if (s->ev[i].batch_index == b) pos[np++] = i;
  for (size_t k = 0; k < np; ++k) {
    int e = validate_event_shape(&s->ev[pos[k]], st->g->n, pos[k]);
    if (e) { free(pos); return e; }
  }
  const int filtering = st->walk.distortion_threshold != 0.0 && !st->freeze;

  /* :415-423 walk-phase snapshots: H as of batch start; shadow G minus
   * this batch's deletions, applied in event order. */
  graph_t* h_snapshot = orc_graph_clone(st->h);
  graph_t* shadow = orc_graph_clone(st->g);
  for (size_t k = 0; k < np; ++k) {
    const orc_event* ev = &s->ev[pos[k]];
    if (ev->kind == 1 && g_has_edge(shadow, ev->u, ev->v)) g_delete(shadow, ev->u, ev->v, NULL);
  }
  /* :425-457 queries; update_id = counter + k over ALL batch events */
  orc_query* iq = xmalloc((np ? np : 1) * sizeof(orc_query));
  orc_query* dq = xmalloc((np ? np : 1) * sizeof(orc_query));
  size_t* slot = xmalloc((np ? np : 1) * sizeof(size_t));
  size_t ni = 0, nd = 0;
  for (size_t k = 0; k < np; ++k) {
    const orc_event* ev = &s->ev[pos[k]];
    const uint64_t update_id = st->update_counter + k;
    slot[k] = SIZE_MAX;
    if (ev->kind == 0) {
      if (!filtering) continue;
      if (h_snapshot->rows[ev->u].n == 0 || h_snapshot->rows[ev->v].n == 0) continue;
      orc_query* q = &iq[ni];
      memset(q, 0, sizeof *q);
      q->kind = 0;
      q->p = ev->u;
      q->q = ev->v;
      q->w_pq = g_edge_weight(st->g, ev->u, ev->v) + ev->weight;
      q->update_id = update_id;
      slot[k] = ni++;
    } else {
      if (st->freeze) continue;
      if (!g_has_edge(h_snapshot, ev->u, ev->v)) continue;
      if (shadow->rows[ev->u].n == 0 || shadow->rows[ev->v].n == 0) continue;
      orc_query* q = &dq[nd];
      memset(q, 0, sizeof *q);
      q->kind = 1;
      q->p = ev->u;
      q->q = ev->v;
      q->update_id = update_id;
      slot[k] = nd++;
    }
  }
  orc_walk_config dcfg = st->walk;
  dcfg.distortion_threshold = INFINITY;
  const size_t stride = (size_t)st->walk.step_cap + 1;
  orc_result* ir = xmalloc((ni ? ni : 1) * sizeof(orc_result));
  orc_result* dr = xmalloc((nd ? nd : 1) * sizeof(orc_result));
  uint32_t* dpaths = xmalloc((nd ? nd : 1) * stride * sizeof(uint32_t));
  int err = orc_run_batch(h_snapshot, iq, ni, &st->walk, 1, ir, NULL);
  if (!err) err = orc_run_batch(shadow, dq, nd, &dcfg, 1, dr, dpaths);
  orc_graph_free(h_snapshot);
  orc_graph_free(shadow);

  /* :466-533 commit, sequential in event order, against live state */
  for (size_t k = 0; k < np && !err; ++k) {
    const orc_event* ev = &s->ev[pos[k]];
    st->update_counter++;
    uint64_t event_steps = 0;
    if (ev->kind == 0) {
      rep->insertions_seen++;
      int r = g_insert(st->g, ev->u, ev->v, ev->weight);
      if (r < 0) { err = rewrap(-r, pos[k]); break; }
      int have_verdict = 0, reached = 0;
      if (slot[k] != SIZE_MAX) {
        have_verdict = 1;
        reached = (int)ir[slot[k]].reached;
        event_steps = ir[slot[k]].steps_used;
      }
      if (commit_insertion(st, ev->u, ev->v, have_verdict, reached)) rep->insertions_kept++;
      else rep->insertions_pruned++;
    } else {
      rep->deletions_seen++;
      int e = g_delete(st->g, ev->u, ev->v, NULL);
      if (e) { err = rewrap(e, pos[k]); break; }
      if (g_has_edge(st->h, ev->u, ev->v)) {
        rep->deletions_in_sparsifier++;
        g_delete(st->h, ev->u, ev->v, NULL);
        if (!st->freeze) {
          const orc_result* res = NULL;
          const uint32_t* path = NULL;
          if (slot[k] != SIZE_MAX) {
            event_steps = dr[slot[k]].steps_used;
            if (dr[slot[k]].reached) {
              res = &dr[slot[k]];
              path = dpaths + slot[k] * stride;
            }
          }
          if (res) {
            uint32_t added = 0;
            for (uint32_t i = 0; i + 1 < res->path_len; ++i) {
              uint32_t a = path[i], bb = path[i + 1];
              if (!g_has_edge(st->h, a, bb)) {
                g_insert(st->h, a, bb, g_edge_weight(st->g, a, bb));
                ++added;
              }
            }
            rep->paths_recovered++;
            rep->edges_recovered += added;
          } else {
            rep->fallback_activations++;
            rep->edges_recovered += run_local_fallback(st, ev->u, ev->v);
          }
        } else {
          rep->fallback_activations++;
        }
      }
    }
    rep->walker_steps += event_steps;
    if (event_steps > rep->max_event_steps) rep->max_event_steps = event_steps;
  }
  free(pos); free(iq); free(dq); free(slot); free(ir); free(dr); free(dpaths);
  rep->wall_ms = now_ms() - start;
  return err;
}

/* sparsifier.cpp:541-548 replay_batch */
int orc_state_replay_batch(void* sp, const void* stream, uint32_t b, orc_report* out) {
  state_t* st = sp;
  const stream_t* s = stream;
  if (b >= s->batch_count && s->batch_count > 0) return set_err(E_USAGE, "batch index out of range");
  memset(out, 0, sizeof *out);
  out->batch_index = b;
  int e = st->batched ? replay_deferred(st, s, b, out) : replay_immediate(st, s, b, out);
  if (e) return e;
  out->density_graph = g_density(st->g);
  out->density_sparsifier = g_density(st->h);
  return 0;
}

/* File formats are not restated (see header). */
void* orc_load_matrix_market(const char* path) {
  (void)path;
  set_err(E_USAGE, "MatrixMarket I/O is not restated; use the reference oracle");
  return NULL;
}
int orc_save_matrix_market(const void* g, const char* path) {
  (void)g; (void)path;
  return set_err(E_USAGE, "MatrixMarket I/O is not restated; use the reference oracle");
}
void* orc_stream_load(const char* path) {
  (void)path;
  set_err(E_USAGE, "stream I/O is not restated; use the reference oracle");
  return NULL;
}
int orc_stream_save(const void* s, const char* path) {
  (void)s; (void)path;
  return set_err(E_USAGE, "stream I/O is not restated; use the reference oracle");
}
