/*
 * oracle_abi.h -- the C ABI shared by the two CPU oracles.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path
 * (paper_2505_02741_b200/) includes, links or calls this. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load an oracle, and only as the checker or the CPU baseline.
 *
 * Two implementations export exactly these symbols:
 *   oracle/_ref/libdyg_ref.so      the UNMODIFIED reference sources from
 *                                  /root/reference/proj/src compiled by
 *                                  oracle/ref/Makefile plus the thin driver
 *                                  oracle/ref/ref_harness.cpp
 *   oracle/_build/libdyg_oracle.so the plain-C restatement
 *                                  oracle/restate/dyg_oracle.c, pinned
 *                                  against the former and the golden vectors
 *                                  in tests/golden/
 *
 * Struct layouts are byte-identical to the product's include/dyg.h structs of
 * the same role, so a test can feed one numpy buffer to both sides.
 */
#ifndef DYG_ORACLE_ABI_H
#define DYG_ORACLE_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* EdgeEvent (reference stream.hpp:11-18). kind: 0 insertion, 1 deletion. */
typedef struct orc_event {
  uint32_t kind;
  uint32_t u;
  uint32_t v;
  uint32_t batch_index;
  double weight;
} orc_event;

/* WalkConfig (walk.hpp:13-18). */
typedef struct orc_walk_config {
  double distortion_threshold; /* K */
  uint32_t step_cap;           /* T */
  uint32_t walker_count;       /* s */
  uint64_t global_seed;
} orc_walk_config;

/* WalkQuery (walk.hpp:71-78). kind: 0 Reach, 1 MinPath. */
typedef struct orc_query {
  uint32_t kind;
  uint32_t p;
  uint32_t q;
  uint32_t pad;
  double w_pq;
  uint64_t update_id;
} orc_query;

/* WalkResult (walk.hpp:80-84) flattened. Reach: reached/best_estimate.
 * MinPath: reached = path found, path_len vertices written to
 * path_buf[i*(T+1)...], resistance. steps_used for both. */
typedef struct orc_result {
  uint32_t reached;
  uint32_t path_len;
  double best_estimate;
  uint64_t steps_used;
  double resistance;
} orc_result;

/* BatchReport (sparsifier.hpp:44-59). */
typedef struct orc_report {
  uint32_t batch_index;
  uint32_t pad;
  uint64_t insertions_seen;
  uint64_t insertions_kept;
  uint64_t insertions_pruned;
  uint64_t deletions_seen;
  uint64_t deletions_in_sparsifier;
  uint64_t paths_recovered;
  uint64_t edges_recovered;
  uint64_t fallback_activations;
  uint64_t walker_steps;
  uint64_t max_event_steps;
  double wall_ms;
  double density_graph;
  double density_sparsifier;
} orc_report;

/* Status codes: 0 ok, else ErrorKind (error.hpp:9): 1 Usage, 2 Data, 3 Numeric. */
const char* orc_last_error(void);
int orc_last_error_kind(void);
const char* orc_impl_name(void);

/* ---- graph (graph.hpp:23-68) ---- */
void* orc_graph_new(uint32_t n);
void* orc_graph_clone(const void* g);
void orc_graph_free(void* g);
uint32_t orc_graph_n(const void* g);
uint64_t orc_graph_edges(const void* g);
double orc_graph_density(const void* g);
int orc_graph_insert(void* g, uint32_t u, uint32_t v, double w);
int orc_graph_delete(void* g, uint32_t u, uint32_t v);
double orc_graph_edge_weight(const void* g, uint32_t u, uint32_t v);
/* Row-order export: row_ptr[n+1], ids[2m], w[2m]. */
void orc_graph_export(const void* g, uint64_t* row_ptr, uint32_t* ids, double* w);

/* ---- generators (tests/support/generators.hpp, sparsifier.cpp:105-159) ---- */
void* orc_make_mesh(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max);
/* make_mesh without the diagonal draw. */
void* orc_make_grid4(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max);
void* orc_make_random_connected(uint32_t n, uint32_t extra, uint64_t seed, double w_min,
                                double w_max, int with_pendant);
void* orc_build_initial_sparsifier(const void* g, double target_density, uint64_t seed);

/* ---- update streams (stream.hpp:20-48) ---- */
void* orc_stream_generate(const void* g, double insert_fraction, double delete_fraction,
                          uint32_t batches, uint64_t seed, uint32_t locality);
void* orc_stream_from_events(const orc_event* ev, size_t n, uint32_t batch_count);
size_t orc_stream_size(const void* s);
uint32_t orc_stream_batches(const void* s);
void orc_stream_copy(const void* s, orc_event* out);
void orc_stream_free(void* s);

/* ---- walks (walk.hpp:51-95) ---- */
uint64_t orc_walker_seed(uint64_t global_seed, uint64_t update_id, uint64_t walker);
/* terminal: 0 ReachedTarget, 1 BudgetExceeded, 2 StepCap, 3 DeadEnd (walk.hpp:20) */
int orc_single_walk(const void* g, uint32_t p, uint32_t q, double w_pq, double budget,
                    uint32_t cap, uint64_t rng_seed, uint32_t* terminal, uint32_t* steps,
                    double* acc, uint32_t* path, uint32_t path_cap, uint32_t* path_len);
size_t orc_loop_erase(const uint32_t* path, size_t n, uint32_t* out);
int orc_run_batch(const void* g, const orc_query* q, size_t nq, const orc_walk_config* cfg,
                  unsigned workers, orc_result* out, uint32_t* path_buf);

/* ---- SparsifierState (sparsifier.hpp:71-112) ---- */
void* orc_state_new(const void* g, const void* h, const orc_walk_config* cfg, int batched,
                    int freeze);
void orc_state_free(void* st);
int orc_state_replay_batch(void* st, const void* stream, uint32_t batch_index,
                           orc_report* out);
/* Reference build only: replay_batch plus the per-event decisions
 * (DYG_DECISION_* codes, one per event of the batch), derived from the
 * reference's pieces and pinned to its own replay (ref/decisions.hpp). */
int orc_state_replay_batch_decisions(void* st, const void* stream, uint32_t batch_index,
                                     orc_report* out, uint8_t* decisions);
const void* orc_state_graph(const void* st);
const void* orc_state_sparsifier(const void* st);
uint64_t orc_state_update_counter(const void* st);

/* ---- file formats (matrix_market.hpp, stream.hpp) ---- */
void* orc_load_matrix_market(const char* path);
int orc_save_matrix_market(const void* g, const char* path);
void* orc_stream_load(const char* path);
int orc_stream_save(const void* s, const char* path);

#ifdef __cplusplus
}
#endif
#endif
