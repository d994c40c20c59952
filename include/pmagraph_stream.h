/*
 * pmagraph_stream.h — synthetic streams and the device sliding window
 * (part of libpmagraph_cuda.so).  These replace the reference's stream
 * drivers (generators.hpp, streaming.hpp) on the GPU side so a GPU pipeline
 * is not bottlenecked by a host deque + hash map; the
 * emitted streams and batches are identical to the reference's.
 */
#ifndef PMAGRAPH_STREAM_H
#define PMAGRAPH_STREAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpma_stream gpma_stream;
typedef struct gpma_window gpma_window;

/* Device pointers and sizes of a window (valid until the next reserve). */
typedef struct gpma_window_info_t {
    const uint32_t* stream_src; /* device, stream_size entries */
    const uint32_t* stream_dst;
    const uint32_t* del_src;    /* device, num_deletions entries (all slides) */
    const uint32_t* del_dst;
    uint64_t stream_size;
    uint64_t initial_size;      /* first ceil(n/2) arrivals (streaming.hpp:83) */
    uint64_t cursor;
    uint64_t num_deletions;
} gpma_window_info_t;

/* One slide (SlideBatch, streaming.hpp:69-74): inserts are stream positions
 * [ins_offset, ins_offset + n_ins); deletions are entries
 * [del_offset, del_offset + n_del) of the window's deletion arrays. */
typedef struct gpma_slide_t {
    uint64_t ins_offset;
    uint64_t n_ins;
    uint64_t del_offset;
    uint64_t n_del;
    int32_t final_partial;
    int32_t _pad;
} gpma_slide_t;

const char* gpma_stream_last_error(void);

/* gen_rmat (generators.hpp:26-63), weights 1.0 */
int gpma_stream_rmat(size_t nv, size_t ne, double a, double b, double c, double d, uint64_t seed,
                     gpma_stream** out);
/* gen_erdos_renyi (generators.hpp:67-89) */
int gpma_stream_erdos_renyi(size_t nv, double density, uint64_t seed, gpma_stream** out);
/* assign_random_timestamps (streaming.hpp:58-67) */
int gpma_stream_shuffle(gpma_stream* s, uint64_t seed);
int gpma_stream_from_arrays(size_t nv, const uint32_t* src, const uint32_t* dst, size_t n, gpma_stream** out);
uint64_t gpma_stream_size(const gpma_stream* s);
uint64_t gpma_stream_num_vertices(const gpma_stream* s);
int gpma_stream_edges(const gpma_stream* s, uint32_t* src, uint32_t* dst);
int gpma_stream_destroy(gpma_stream* s);
/* draw_below (streaming.hpp:43-50) sequence from mt19937_64(seed) */
int gpma_draw_below_sequence(uint64_t seed, uint64_t bound, size_t n, uint64_t* out);

/* SlidingWindow (streaming.hpp:76-123) on CUDA device `device`. */
int gpma_window_create(const gpma_stream* s, int device, gpma_window** out);
int gpma_window_destroy(gpma_window* w);
int gpma_window_info(const gpma_window* w, gpma_window_info_t* out);
int gpma_window_reserve(gpma_window* w, size_t max_deletions);
int gpma_window_slide(gpma_window* w, size_t batch, gpma_slide_t* out);
/* std::mt19937_64 owned by the caller (the reference passes it by reference;
 * its state advances across slides). */
typedef struct gpma_rng gpma_rng;
int gpma_rng_create(uint64_t seed, gpma_rng** out);
int gpma_rng_destroy(gpma_rng* r);
/* SlidingWindow::slide_explicit_random (streaming.hpp:129-158): the next
 * `batch` arrivals, and min(batch, window size) expiring edges drawn uniformly
 * without replacement from the window before the arrivals; deletions are the
 * expiries whose key leaves the window (multiplicity filtered), in window
 * order, appended like gpma_window_slide's.  FIFO and explicit slides may be
 * mixed on one window. */
int gpma_window_slide_explicit_random(gpma_window* w, size_t batch, gpma_rng* rng, gpma_slide_t* out);
/* SlidingWindow::window_size (streaming.hpp:101) */
uint64_t gpma_window_size(const gpma_window* w);
/* Copy deletions [offset, offset+n) of the window to host arrays. */
int gpma_window_deletions_host(gpma_window* w, size_t offset, size_t n, uint32_t* src, uint32_t* dst);
/* SlideBatch::expiries (streaming.hpp:69-74) of the last slide: the stream
 * positions of the raw edges that left the window, in window order (FIFO:
 * the oldest; explicit: the drawn ones).  *n = their count; up to cap are
 * written. */
int gpma_window_last_expiries(gpma_window* w, uint32_t* positions, size_t cap, size_t* n);
/* SlidingWindow::distinct_edges (streaming.hpp:162-169), ascending key order
 * (the reference's is a hash map's, unspecified).  cap = 0: count only. */
int gpma_window_distinct_edges(gpma_window* w, uint32_t* src, uint32_t* dst, size_t cap, size_t* n);
/* A caller's std::mt19937_64 in and out of a gpma_rng (its standard text
 * state), so the caller's generator advances exactly as in the reference. */
int gpma_rng_set_state(gpma_rng* r, const char* text);
int gpma_rng_get_state(const gpma_rng* r, char* buf, size_t cap, size_t* len);

#ifdef __cplusplus
}
#endif
#endif /* PMAGRAPH_STREAM_H */
