/*
 * dyg_host.h -- C-ABI of the host-side input pipeline that sits above the
 * device path: the reference's graph / update-stream file formats and the
 * benchmark input generators (SURVEY.md 8f rows 1-2 stay on the host this
 * round). Everything here is plain C++ in libdyg.so; none of it runs on the
 * per-batch hot path.
 *
 *   dygh_graph   -- host adjacency rows with DynamicGraph semantics
 *                   (proj/src/graph.hpp:23-68): push_back on insert,
 *                   swap-with-last on delete, coalesce in place.
 *   dygh_stream  -- UpdateStream (proj/src/stream.hpp:20-23).
 *
 * Return codes as in dyg.h (ErrorKind); messages via dygh_last_error().
 */
#ifndef DYG_HOST_H
#define DYG_HOST_H

#include "dyg.h"

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct dygh_graph dygh_graph;
typedef struct dygh_stream dygh_stream;

const char* dygh_last_error(void);

/* DynamicGraph (graph.hpp:23-68). */
int dygh_graph_new(uint32_t n, dygh_graph** out);
int dygh_graph_from_csr(const dyg_csr* csr, dygh_graph** out);
void dygh_graph_free(dygh_graph* g);
uint32_t dygh_graph_n(const dygh_graph* g);
uint64_t dygh_graph_edges(const dygh_graph* g);
double dygh_graph_density(const dygh_graph* g);
int dygh_graph_insert(dygh_graph* g, uint32_t u, uint32_t v, double w);
int dygh_graph_delete(dygh_graph* g, uint32_t u, uint32_t v);
double dygh_graph_edge_weight(const dygh_graph* g, uint32_t u, uint32_t v);
/* Row-order view, valid until the next mutation or free. */
int dygh_graph_csr(dygh_graph* g, dyg_csr* out);

/* Input generators (reference tests/support/generators.hpp:37-86,
 * sparsifier.cpp:105-159, stream.cpp:114-200). */
int dygh_make_mesh(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max,
                   dygh_graph** out);
int dygh_make_grid4(uint32_t rows, uint32_t cols, uint64_t seed, double w_min, double w_max,
                    dygh_graph** out);
int dygh_make_random_connected(uint32_t n, uint32_t extra, uint64_t seed, double w_min,
                               double w_max, int with_pendant, dygh_graph** out);
int dygh_build_initial_sparsifier(const dygh_graph* g, double target_density, uint64_t seed,
                                  dygh_graph** out);
int dygh_generate_stream(const dygh_graph* g, double insert_fraction, double delete_fraction,
                         uint32_t batches, uint64_t seed, uint32_t locality, dygh_stream** out);

/* File formats (matrix_market.hpp:14-18, stream.hpp:25-31). */
int dygh_load_matrix_market(const char* path, dygh_graph** out);
int dygh_save_matrix_market(const dygh_graph* g, const char* path);
int dygh_load_stream(const char* path, dygh_stream** out);
int dygh_save_stream(const dygh_stream* s, const char* path);

/* UpdateStream. */
int dygh_stream_from_events(const dyg_event* events, size_t n, uint32_t batch_count,
                            dygh_stream** out);
void dygh_stream_free(dygh_stream* s);
size_t dygh_stream_size(const dygh_stream* s);
uint32_t dygh_stream_batches(const dygh_stream* s);
const dyg_event* dygh_stream_events(const dygh_stream* s);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* DYG_HOST_H */
