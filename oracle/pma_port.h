/* oracle/pma_port.h — TEST INFRASTRUCTURE ONLY (a checker, never the product).
 *
 * Plain-C restatement of the reference GPMA+ path, written in the same
 * decomposition the sm_100a kernels use (rank-based merge, backward-filled
 * leaf headers, per-level group rounds) so that pinning it against the real
 * reference (oracle/_ref/libpmagraph_ref.so) on CPU also validates the GPU
 * formulation.  Each function cites the reference file:line it follows.
 * Structs are shared with include/pmagraph_cuda.h. */
#ifndef PMA_PORT_H
#define PMA_PORT_H
#include <stddef.h>
#include <stdint.h>

#include "pmagraph_cuda.h"

typedef struct port_pma port_pma;
typedef struct port_graph port_graph;

const char* port_last_error(void);

int port_pma_create(const pma_profile* profile, port_pma** out);
void port_pma_destroy(port_pma* p);
int port_pma_from_sorted(port_pma* p, const uint64_t* keys, const uint64_t* values, size_t n,
                         double fill_target);
int port_pma_load_slots(port_pma* p, size_t capacity, const uint64_t* keys, const uint64_t* values,
                        const uint8_t* states);
int port_pma_download(port_pma* p, uint64_t* keys, uint64_t* values, uint8_t* states);
int port_pma_get_layout(port_pma* p, pma_layout_info* out);
int port_pma_bounds(port_pma* p, int level, uint64_t* mn, uint64_t* mx);
int port_pma_binary_search_leaf(port_pma* p, const uint64_t* keys, size_t n, uint64_t* leaves);
int port_pma_batch_update(port_pma* p, const uint64_t* keys, const uint64_t* values,
                          const uint8_t* ops, size_t n, const pma_engine_config* cfg,
                          pma_stats* out);
int port_pma_touched_ranges(port_pma* p, uint64_t* pairs, size_t cap, size_t* count);

int port_graph_from_edges(const gpma_graph_config* cfg, size_t nv, const uint32_t* src,
                          const uint32_t* dst, const double* w, size_t n, port_graph** out);
void port_graph_destroy(port_graph* g);
port_pma* port_graph_pma(port_graph* g);
int port_graph_apply_batch(port_graph* g, const uint32_t* is, const uint32_t* id, const double* iw,
                           size_t ni, const uint32_t* ds, const uint32_t* dd, size_t nd,
                           pma_stats* out);
int port_graph_row_offsets(port_graph* g, uint64_t* out);
int port_bfs(port_graph* g, uint32_t root, uint32_t* dist);
int port_cc(port_graph* g, uint32_t* labels);
int port_pagerank(port_graph* g, double damping, double eps, size_t max_iters, const double* warm,
                  double* ranks, uint64_t* iters, int* converged);
int port_spmv(port_graph* g, const double* x, double* y);

#endif
