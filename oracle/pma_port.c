/* oracle/pma_port.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference GPMA+ path used as a checker (never shipped, never measured as
 * the product).  It is deliberately written in the decomposition the sm_100a
 * kernels use, so that its bit-exact agreement with the real reference
 * (oracle/_ref/libpmagraph_ref.so, tests/test_oracle.py) also validates that
 * formulation on CPU:
 *   - leaf search over backward-filled leaf headers instead of the top-down
 *     halving of pma.hpp:234-245 (same answer, see leaf_of());
 *   - merge commits by ranks (lower_bound of each update in the segment's
 *     valid entries) and a destination-driven even placement instead of the
 *     sequential merge + place_evenly of segment_engine.hpp:119-137,
 *     232-271 and pma.hpp:440-467;
 *   - connected components by min-root union-find (labels are the unique
 *     min-id per component, as analytics.hpp:53-82 produces).
 * The root path (grow/shrink) follows segment_engine.hpp:435-463 and
 * pma.hpp:390-402,597-601 step by step. */
#include "pma_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

const char* port_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

/* ---------------------------------------------------------------- layout */

struct port_pma {
    pma_profile prof;
    uint64_t cap, leaf;
    int height;
    uint64_t* keys;
    uint64_t* vals;
    uint8_t* st;
    uint64_t mn[PMA_MAX_LEVELS], mx[PMA_MAX_LEVELS];
    uint64_t valid, tomb, slot_writes;
    uint64_t* touched; /* pairs */
    size_t ntouched, touched_cap;
};

/* PmaLayout::leaf_size_for (pma.hpp:95-101) */
static uint64_t leaf_size_for(uint64_t cap) {
    int lg = 0;
    while ((1ull << (lg + 1)) <= cap) ++lg;
    uint64_t leaf = 4;
    while (leaf * 2 <= (uint64_t)lg) leaf *= 2;
    return leaf;
}

static int height_for(uint64_t cap, uint64_t leaf) {
    int h = 0;
    for (uint64_t s = leaf; s < cap; s <<= 1) ++h;
    return h;
}

/* rebuild_bounds (pma.hpp:577-588): leaf bounds doubled per level */
static void bounds_for(const pma_profile* pr, uint64_t leaf, int h, uint64_t* mn, uint64_t* mx) {
    const double lf = (double)leaf;
    const uint64_t mn0 = (uint64_t)ceil(pr->leaf_lower * lf - 1e-9);
    const uint64_t mx0 = (uint64_t)floor(pr->leaf_upper * lf + 1e-9);
    for (int l = 0; l <= h; ++l) {
        mn[l] = mn0 << l;
        mx[l] = mx0 << l;
    }
}

/* max_entries_at_capacity (pma.hpp:590-595) */
static uint64_t max_at_capacity(const pma_profile* pr, uint64_t cap) {
    const uint64_t leaf = leaf_size_for(cap);
    const int h = height_for(cap, leaf);
    const uint64_t mx0 = (uint64_t)floor(pr->leaf_upper * (double)leaf + 1e-9);
    return mx0 << h;
}

/* reset_layout (pma.hpp:561-567) */
static void reset_layout(port_pma* p, uint64_t cap) {
    free(p->keys);
    free(p->vals);
    free(p->st);
    p->cap = cap;
    p->leaf = leaf_size_for(cap);
    p->height = height_for(cap, p->leaf);
    p->keys = (uint64_t*)calloc(cap, 8);
    p->vals = (uint64_t*)calloc(cap, 8);
    p->st = (uint8_t*)calloc(cap, 1);
    p->valid = 0;
    p->tomb = 0;
    bounds_for(&p->prof, p->leaf, p->height, p->mn, p->mx);
}

/* DensityProfile::validate (pma.hpp:59-67) */
static int validate_profile(const pma_profile* d) {
    if (!(d->leaf_lower > 0.0 && d->leaf_lower < d->root_lower && d->root_lower < d->root_upper &&
          d->root_upper < d->leaf_upper && d->leaf_upper < 1.0))
        return fail(PMA_EINVAL,
                    "DensityProfile: need 0 < leaf_lower < root_lower < root_upper < leaf_upper < 1");
    if (2.0 * d->root_lower > d->root_upper + 1e-12)
        return fail(PMA_EINVAL,
                    "DensityProfile: need 2*root_lower <= root_upper so a post-shrink root is legal");
    return PMA_OK;
}

int port_pma_create(const pma_profile* profile, port_pma** out) {
    pma_profile d = {0.08, 0.92, 0.40, 0.80, 1, 0};
    if (profile) d = *profile;
    int rc = validate_profile(&d);
    if (rc) return rc;
    port_pma* p = (port_pma*)calloc(1, sizeof(port_pma));
    p->prof = d;
    reset_layout(p, 16);
    *out = p;
    return PMA_OK;
}

void port_pma_destroy(port_pma* p) {
    if (!p) return;
    free(p->keys);
    free(p->vals);
    free(p->st);
    free(p->touched);
    free(p);
}

/* place_evenly (pma.hpp:440-467), destination-driven: slot t of [b, b+m)
 * holds entry j = ceil(t*k/m) iff floor(j*m/k) == t. */
static void place_evenly(port_pma* p, uint64_t b, uint64_t m, const uint64_t* ek, const uint64_t* ev,
                         uint64_t k) {
    uint64_t old_valid = 0, old_tomb = 0;
    for (uint64_t i = b; i < b + m; ++i) {
        old_valid += p->st[i] == 1;
        old_tomb += p->st[i] == 2;
    }
    for (uint64_t t = 0; t < m; ++t) {
        const uint64_t j = k ? (t * k + m - 1) / m : 0;
        if (k && j < k && (j * m) / k == t) {
            p->keys[b + t] = ek[j];
            p->vals[b + t] = ev[j];
            p->st[b + t] = 1;
        } else {
            p->keys[b + t] = 0;
            p->vals[b + t] = 0;
            p->st[b + t] = 0;
        }
    }
    p->valid += k;
    p->valid -= old_valid;
    p->tomb -= old_tomb;
    p->slot_writes += m;
}

int port_pma_from_sorted(port_pma* p, const uint64_t* keys, const uint64_t* values, size_t n,
                         double fill_target) {
    /* pma.hpp:160-187 */
    if (!(fill_target > 0.0 && fill_target <= p->prof.leaf_upper + 1e-12))
        return fail(PMA_EINVAL, "from_sorted: fill_target must be in (0, leaf_upper]");
    for (size_t i = 1; i < n; ++i) {
        if (keys[i] <= keys[i - 1]) {
            snprintf(g_err, sizeof(g_err),
                     "from_sorted: keys must be strictly increasing (duplicate or unsorted input at index %zu)",
                     i);
            return PMA_EINVAL;
        }
    }
    p->slot_writes = 0;
    uint64_t cap = 16;
    while ((double)n > fill_target * (double)cap) cap <<= 1;
    reset_layout(p, cap);
    while (n > p->mx[p->height]) reset_layout(p, p->cap << 1);
    while (p->cap > 16 && n < p->mn[p->height] && n <= max_at_capacity(&p->prof, p->cap >> 1))
        reset_layout(p, p->cap >> 1);
    if (n > 0) {
        uint64_t* zv = NULL;
        if (!values) zv = (uint64_t*)calloc(n, 8);
        place_evenly(p, 0, p->cap, keys, values ? values : zv, n);
        free(zv);
    }
    return PMA_OK;
}

int port_pma_load_slots(port_pma* p, size_t capacity, const uint64_t* keys, const uint64_t* values,
                        const uint8_t* states) {
    if (capacity < 16 || (capacity & (capacity - 1)))
        return fail(PMA_EINVAL, "load_slots: capacity must be a power of two >= 16");
    reset_layout(p, capacity);
    for (size_t i = 0; i < capacity; ++i) {
        p->st[i] = states[i];
        if (states[i]) {
            p->keys[i] = keys[i];
            p->vals[i] = values[i];
        }
        p->valid += states[i] == 1;
        p->tomb += states[i] == 2;
    }
    p->slot_writes = 0;
    return PMA_OK;
}

int port_pma_download(port_pma* p, uint64_t* keys, uint64_t* values, uint8_t* states) {
    if (keys) memcpy(keys, p->keys, p->cap * 8);
    if (values) memcpy(values, p->vals, p->cap * 8);
    if (states) memcpy(states, p->st, p->cap);
    return PMA_OK;
}

int port_pma_get_layout(port_pma* p, pma_layout_info* out) {
    memset(out, 0, sizeof(*out));
    out->capacity = p->cap;
    out->leaf_size = p->leaf;
    out->height = p->height;
    out->valid_count = p->valid;
    out->tombstone_count = p->tomb;
    out->slot_writes = p->slot_writes;
    return PMA_OK;
}

int port_pma_bounds(port_pma* p, int level, uint64_t* mn, uint64_t* mx) {
    if (level < 0 || level > p->height) return fail(PMA_ERANGE, "level outside [0, height]");
    *mn = p->mn[level];
    *mx = p->mx[level];
    return PMA_OK;
}

/* ------------------------------------------------------------ leaf search */

/* Backward-filled leaf headers: H[i] = first non-Empty key at or after leaf
 * i's first slot (UINT64_MAX when none).  Non-decreasing. */
static uint64_t* build_headers(const port_pma* p) {
    const uint64_t L = p->cap / p->leaf;
    uint64_t* H = (uint64_t*)malloc(L * 8);
    uint64_t next = UINT64_MAX;
    for (uint64_t i = L; i-- > 0;) {
        for (uint64_t s = i * p->leaf; s < (i + 1) * p->leaf; ++s) {
            if (p->st[s] != 0) {
                next = p->keys[s];
                break;
            }
        }
        H[i] = next;
    }
    return H;
}

static int leaf_nonempty(const port_pma* p, uint64_t leaf) {
    for (uint64_t s = leaf * p->leaf; s < (leaf + 1) * p->leaf; ++s)
        if (p->st[s]) return 1;
    return 0;
}

/* binary_search_leaf (pma.hpp:234-245) == "last leaf whose first non-Empty
 * key <= key, else 0" (oracle reference.hpp:65-77) == upper_bound over the
 * backward-filled headers minus one.  key == UINT64_MAX needs the explicit
 * non-empty check because trailing empty leaves carry the same sentinel. */
static uint64_t leaf_of(const port_pma* p, const uint64_t* H, uint64_t key) {
    const uint64_t L = p->cap / p->leaf;
    if (key != UINT64_MAX) {
        uint64_t lo = 0, hi = L; /* first index with H > key */
        while (lo < hi) {
            uint64_t mid = (lo + hi) / 2;
            if (H[mid] <= key) lo = mid + 1;
            else hi = mid;
        }
        return lo ? lo - 1 : 0;
    }
    uint64_t lo = 0, hi = L; /* first index with H == MAX */
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (H[mid] < UINT64_MAX) lo = mid + 1;
        else hi = mid;
    }
    if (lo < L && leaf_nonempty(p, lo)) return lo;
    return lo ? lo - 1 : 0;
}

int port_pma_binary_search_leaf(port_pma* p, const uint64_t* keys, size_t n, uint64_t* leaves) {
    uint64_t* H = build_headers(p);
    for (size_t i = 0; i < n; ++i) leaves[i] = leaf_of(p, H, keys[i]);
    free(H);
    return PMA_OK;
}

/* ----------------------------------------------------------- batch update */

typedef struct {
    uint64_t key, val;
    uint32_t idx;
    uint8_t op;
} upd_t;

static int cmp_upd(const void* a, const void* b) {
    const upd_t* x = (const upd_t*)a;
    const upd_t* y = (const upd_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static void add_touched(port_pma* p, uint64_t b, uint64_t e) {
    if (p->ntouched == p->touched_cap) {
        p->touched_cap = p->touched_cap ? 2 * p->touched_cap : 64;
        p->touched = (uint64_t*)realloc(p->touched, p->touched_cap * 16);
    }
    p->touched[2 * p->ntouched] = b;
    p->touched[2 * p->ntouched + 1] = e;
    p->ntouched++;
}

static size_t lower_bound_u64(const uint64_t* a, size_t n, uint64_t key) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        size_t mid = (lo + hi) / 2;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/* commit_merge (segment_engine.hpp:273-280) in rank form.  Output identical
 * to merge_entries + place_evenly; slot-write accounting follows the tier:
 * m for small/medium (place_evenly), compaction moves + m for large
 * (commit_in_place, segment_engine.hpp:147-230). */
static void merge_commit(port_pma* p, uint64_t b, uint64_t m, const upd_t* U, const uint32_t* slice,
                         size_t s, int large, uint64_t* missed) {
    uint64_t ne = 0;
    for (uint64_t i = b; i < b + m; ++i) ne += p->st[i] == 1;
    uint64_t* ek = (uint64_t*)malloc((ne + 1) * 8);
    uint64_t* ev = (uint64_t*)malloc((ne + 1) * 8);
    uint64_t* es = (uint64_t*)malloc((ne + 1) * 8);
    uint8_t* matched = (uint8_t*)calloc(ne + 1, 1);
    ne = 0;
    for (uint64_t i = b; i < b + m; ++i) {
        if (p->st[i] == 1) {
            ek[ne] = p->keys[i];
            ev[ne] = p->vals[i];
            es[ne] = i - b;
            ++ne;
        }
    }
    uint64_t* ik = (uint64_t*)malloc((s + 1) * 8);
    uint64_t* iv = (uint64_t*)malloc((s + 1) * 8);
    uint64_t* ir = (uint64_t*)malloc((s + 1) * 8);
    uint64_t nins = 0;
    for (size_t q = 0; q < s; ++q) {
        const upd_t* u = &U[slice[q]];
        const uint64_t r = lower_bound_u64(ek, ne, u->key);
        const int match = r < ne && ek[r] == u->key;
        if (u->op == 1) {
            if (match) matched[r] = 1;
            else ++*missed;
        } else {
            if (match) matched[r] = 2;
            ik[nins] = u->key;
            iv[nins] = u->val;
            ir[nins] = r;
            ++nins;
        }
    }
    uint64_t* sb = (uint64_t*)malloc((ne + 1) * 8); /* survivors before rank j */
    sb[0] = 0;
    for (uint64_t j = 0; j < ne; ++j) sb[j + 1] = sb[j] + (matched[j] == 0);
    const uint64_t k = sb[ne] + nins;
    uint64_t* ok = (uint64_t*)malloc((k + 1) * 8);
    uint64_t* ov = (uint64_t*)malloc((k + 1) * 8);
    uint64_t ip = 0; /* inserts with r <= j */
    for (uint64_t j = 0; j < ne; ++j) {
        while (ip < nins && ir[ip] <= j) ++ip;
        if (matched[j] == 0) {
            ok[sb[j] + ip] = ek[j];
            ov[sb[j] + ip] = ev[j];
        }
    }
    for (uint64_t q = 0; q < nins; ++q) {
        ok[sb[ir[q]] + q] = ik[q];
        ov[sb[ir[q]] + q] = iv[q];
    }
    uint64_t moves = 0;
    if (large) {
        uint64_t pa = 0; /* pass-A survivors: valid and not delete-matched */
        for (uint64_t j = 0; j < ne; ++j) {
            if (matched[j] == 1) continue;
            if (es[j] != pa) ++moves;
            ++pa;
        }
    }
    place_evenly(p, b, m, ok, ov, k);
    p->slot_writes += moves;
    free(ek), free(ev), free(es), free(matched), free(ik), free(iv), free(ir), free(sb), free(ok), free(ov);
}

/* commit_tombstones (segment_engine.hpp:285-310) */
static void tombstone_commit(port_pma* p, uint64_t b, uint64_t m, const upd_t* U, const uint32_t* slice,
                             size_t s, uint64_t* missed, uint64_t* added) {
    for (size_t q = 0; q < s; ++q) {
        const uint64_t key = U[slice[q]].key;
        int hit = 0;
        for (uint64_t i = b; i < b + m; ++i) {
            if (p->st[i] != 0 && p->keys[i] == key) {
                if (p->st[i] == 1) {
                    p->st[i] = 2;
                    p->valid--;
                    p->tomb++;
                    p->slot_writes++;
                    ++*added;
                    hit = 1;
                }
                break;
            }
        }
        if (!hit) ++*missed;
    }
}

/* rebuild_at_capacity (pma.hpp:597-601) */
static void rebuild_at_capacity(port_pma* p, uint64_t cap) {
    uint64_t n = p->valid;
    uint64_t* k = (uint64_t*)malloc((n + 1) * 8);
    uint64_t* v = (uint64_t*)malloc((n + 1) * 8);
    n = 0;
    for (uint64_t i = 0; i < p->cap; ++i)
        if (p->st[i] == 1) {
            k[n] = p->keys[i];
            v[n] = p->vals[i];
            ++n;
        }
    reset_layout(p, cap);
    if (n) place_evenly(p, 0, cap, k, v, n);
    free(k);
    free(v);
}

static int strategy_large(const pma_engine_config* c, uint64_t m) {
    if (c->force_strategy >= 0) return c->force_strategy == PMA_STRATEGY_LARGE;
    if (m <= c->small_max) return 0;
    if (m <= c->medium_max) return 0;
    return 1;
}

int port_pma_batch_update(port_pma* p, const uint64_t* keys, const uint64_t* values, const uint8_t* ops,
                          size_t n, const pma_engine_config* cfg_in, pma_stats* out) {
    pma_engine_config cfg = {PMA_LAZY, 1, 32, 1024, PMA_STRATEGY_AUTO, 0};
    if (cfg_in) cfg = *cfg_in;
    const int eager = cfg.deletion_mode == PMA_EAGER;
    pma_stats st;
    memset(&st, 0, sizeof(st));
    st.batch_size = n;
    st.num_levels = p->height + 1;
    p->ntouched = 0;
    if (n == 0) {
        if (out) *out = st;
        return PMA_OK;
    }
    const uint64_t writes_base = p->slot_writes;
    /* sort_by_key (stable) + resolve_duplicates (segment_engine.hpp:380-381,346-363) */
    upd_t* U = (upd_t*)malloc(n * sizeof(upd_t));
    for (size_t i = 0; i < n; ++i) {
        U[i].key = keys[i];
        U[i].val = values ? values[i] : 0;
        U[i].op = ops[i] ? 1 : 0;
        U[i].idx = (uint32_t)i;
    }
    qsort(U, n, sizeof(upd_t), cmp_upd);
    size_t w = 0;
    for (size_t i = 0; i < n;) {
        size_t j = i;
        upd_t eff = {U[i].key, 0, 0, 1};
        while (j < n && U[j].key == U[i].key) {
            if (U[j].op == 0) {
                eff.val = U[j].val;
                eff.op = 0;
            }
            ++j;
        }
        U[w++] = eff;
        i = j;
    }
    const size_t nu = w;
    /* leaf assignment, once per batch (segment_engine.hpp:388-392) */
    uint64_t* leaf = (uint64_t*)malloc(nu * 8);
    {
        uint64_t* H = build_headers(p);
        for (size_t i = 0; i < nu; ++i) leaf[i] = leaf_of(p, H, U[i].key);
        free(H);
    }
    uint32_t* pend = (uint32_t*)malloc(nu * 4);
    uint32_t* next = (uint32_t*)malloc(nu * 4);
    size_t np = nu;
    for (size_t i = 0; i < nu; ++i) pend[i] = (uint32_t)i;
    for (int level = 0;; ++level) {
        /* unique_segments + try_insert_plus per group (segment_engine.hpp:396-432) */
        const uint64_t m = p->leaf << level;
        size_t nn = 0;
        int any_left = 0;
        size_t root_lo = 0, root_hi = 0;
        for (size_t g0 = 0; g0 < np;) {
            const uint64_t seg = leaf[pend[g0]] >> level;
            size_t g1 = g0;
            while (g1 < np && (leaf[pend[g1]] >> level) == seg) ++g1;
            const size_t s = g1 - g0;
            uint64_t ins = 0;
            for (size_t q = g0; q < g1; ++q) ins += U[pend[q]].op == 0;
            const uint64_t dels = s - ins;
            const uint64_t b = seg * m;
            int committed = 0, moved = 0;
            if (!eager && ins == 0) {
                tombstone_commit(p, b, m, U, pend + g0, s, &st.deletes_missed, &st.tombstones_added);
                committed = 1;
            } else {
                uint64_t nv = 0;
                for (uint64_t i = b; i < b + m; ++i) nv += p->st[i] == 1;
                int defer = nv + ins > p->mx[level];
                if (!defer && eager && p->cap > 16 && nv < dels + p->mn[level]) defer = 1;
                if (!defer) {
                    merge_commit(p, b, m, U, pend + g0, s, strategy_large(&cfg, m), &st.deletes_missed);
                    committed = moved = 1;
                }
            }
            if (committed) {
                st.segments_per_level[level]++;
                if (moved) add_touched(p, b, b + m);
            } else {
                any_left = 1;
                root_lo = g0;
                root_hi = g1;
                for (size_t q = g0; q < g1; ++q) next[nn++] = pend[q];
            }
            g0 = g1;
        }
        st.rounds++;
        if (!any_left) break;
        if (level == p->height) {
            /* root path (segment_engine.hpp:435-463) */
            const size_t s = root_hi - root_lo;
            uint64_t ins = 0;
            for (size_t q = root_lo; q < root_hi; ++q) ins += U[pend[q]].op == 0;
            while (p->valid + ins > p->mx[p->height]) {
                rebuild_at_capacity(p, p->cap << 1);
                st.grow_events++;
            }
            merge_commit(p, 0, p->cap, U, pend + root_lo, s, strategy_large(&cfg, p->cap), &st.deletes_missed);
            st.num_levels = p->height + 1;
            st.segments_per_level[p->height]++;
            st.rounds++;
            if (eager && p->prof.allow_shrink) {
                int shrunk = 0;
                while (p->cap > 16 && p->valid < p->mn[p->height]) {
                    rebuild_at_capacity(p, p->cap >> 1);
                    shrunk = 1;
                }
                if (shrunk) st.shrink_events++;
            }
            st.resized = st.grow_events > 0 || st.shrink_events > 0;
            if (!st.resized) add_touched(p, 0, p->cap);
            break;
        }
        /* advance_round (segment_engine.hpp:90-105) */
        uint32_t* t = pend;
        pend = next;
        next = t;
        np = nn;
    }
    st.slot_writes = p->slot_writes - writes_base;
    st.num_touched_ranges = p->ntouched;
    if (out) *out = st;
    free(U);
    free(leaf);
    free(pend);
    free(next);
    return PMA_OK;
}

int port_pma_touched_ranges(port_pma* p, uint64_t* pairs, size_t cap, size_t* count) {
    *count = p->ntouched;
    for (size_t i = 0; i < p->ntouched && i < cap; ++i) {
        pairs[2 * i] = p->touched[2 * i];
        pairs[2 * i + 1] = p->touched[2 * i + 1];
    }
    return PMA_OK;
}

/* ------------------------------------------------------------------ graph */

#define GUARD_DST 0xFFFFFFFFull

struct port_graph {
    gpma_graph_config cfg;
    size_t nv;
    port_pma* p;
    uint64_t* ro;
};

port_pma* port_graph_pma(port_graph* g) { return g->p; }

static int cmp_kv_stable(const void* a, const void* b) {
    const uint64_t* x = (const uint64_t*)a; /* key, value, arrival */
    const uint64_t* y = (const uint64_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[2] < y[2] ? -1 : (x[2] > y[2]);
}

/* rebuild_row_offsets (graph.hpp:182-190) */
static void rebuild_row_offsets(port_graph* g) {
    free(g->ro);
    g->ro = (uint64_t*)calloc(g->nv + 1, 8);
    const port_pma* p = g->p;
    for (uint64_t i = 0; i < p->cap; ++i)
        if (p->st[i] == 1 && (p->keys[i] & 0xFFFFFFFFull) == GUARD_DST) g->ro[(p->keys[i] >> 32) + 1] = i + 1;
}

int port_graph_from_edges(const gpma_graph_config* cfg, size_t nv, const uint32_t* src, const uint32_t* dst,
                          const double* w, size_t n, port_graph** out) {
    /* graph.hpp:66-92 */
    if (nv >= GUARD_DST) return fail(PMA_EINVAL, "from_edges: vertex count exceeds the id space");
    for (size_t i = 0; i < n; ++i) {
        if (src[i] >= nv || dst[i] >= nv) {
            snprintf(g_err, sizeof(g_err), "edge (%u, %u) outside vertex range %zu", src[i], dst[i], nv);
            return PMA_EINVAL;
        }
    }
    port_graph* g = (port_graph*)calloc(1, sizeof(port_graph));
    gpma_graph_config c = {0, PMA_LAZY, 1, 0, 0.5, {0.08, 0.92, 0.40, 0.80, 1, 0}};
    if (cfg) c = *cfg;
    g->cfg = c;
    g->nv = nv;
    int rc = port_pma_create(&c.profile, &g->p);
    if (rc) {
        free(g);
        return rc;
    }
    uint64_t* kv = (uint64_t*)malloc((n + nv + 1) * 24);
    for (size_t i = 0; i < n; ++i) {
        double wt = w ? w[i] : 1.0;
        kv[3 * i] = ((uint64_t)src[i] << 32) | dst[i];
        memcpy(&kv[3 * i + 1], &wt, 8);
        kv[3 * i + 2] = i;
    }
    qsort(kv, n, 24, cmp_kv_stable);
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        if (i + 1 < n && kv[3 * (i + 1)] == kv[3 * i]) continue; /* last wins */
        memmove(&kv[3 * m], &kv[3 * i], 24);
        ++m;
    }
    for (size_t v = 0; v < nv; ++v) {
        kv[3 * m] = ((uint64_t)v << 32) | GUARD_DST;
        kv[3 * m + 1] = 0;
        kv[3 * m + 2] = m;
        ++m;
    }
    qsort(kv, m, 24, cmp_kv_stable);
    uint64_t* k = (uint64_t*)malloc((m + 1) * 8);
    uint64_t* v = (uint64_t*)malloc((m + 1) * 8);
    for (size_t i = 0; i < m; ++i) {
        k[i] = kv[3 * i];
        v[i] = kv[3 * i + 1];
    }
    free(kv);
    rc = port_pma_from_sorted(g->p, k, v, m, c.fill_target);
    free(k);
    free(v);
    if (rc) {
        port_graph_destroy(g);
        return rc;
    }
    rebuild_row_offsets(g);
    *out = g;
    return PMA_OK;
}

void port_graph_destroy(port_graph* g) {
    if (!g) return;
    port_pma_destroy(g->p);
    free(g->ro);
    free(g);
}

int port_graph_apply_batch(port_graph* g, const uint32_t* is, const uint32_t* id, const double* iw, size_t ni,
                           const uint32_t* ds, const uint32_t* dd, size_t nd, pma_stats* out) {
    /* graph.hpp:130-162 */
    for (size_t i = 0; i < ni; ++i) {
        if (is[i] >= g->nv || id[i] >= g->nv) {
            snprintf(g_err, sizeof(g_err), "edge (%u, %u) outside vertex range %zu", is[i], id[i], g->nv);
            return PMA_EINVAL;
        }
    }
    size_t n = 0, guard_deletes = 0;
    uint64_t* k = (uint64_t*)malloc((ni + nd + 1) * 8);
    uint64_t* v = (uint64_t*)malloc((ni + nd + 1) * 8);
    uint8_t* o = (uint8_t*)malloc(ni + nd + 1);
    for (size_t i = 0; i < ni; ++i) {
        double wt = iw ? iw[i] : 1.0;
        k[n] = ((uint64_t)is[i] << 32) | id[i];
        memcpy(&v[n], &wt, 8);
        o[n++] = 0;
    }
    for (size_t i = 0; i < nd; ++i) {
        if (dd[i] == GUARD_DST) {
            ++guard_deletes;
            continue;
        }
        k[n] = ((uint64_t)ds[i] << 32) | dd[i];
        v[n] = 0;
        o[n++] = 1;
    }
    pma_engine_config ec = {g->cfg.deletion_mode, g->cfg.workers, 32, 1024, PMA_STRATEGY_AUTO, 0};
    pma_stats st;
    int rc = port_pma_batch_update(g->p, k, v, o, n, &ec, &st);
    free(k), free(v), free(o);
    if (rc) return rc;
    st.deletes_missed += guard_deletes;
    /* refresh_row_offsets (graph.hpp:167-180) */
    if (st.resized) {
        rebuild_row_offsets(g);
    } else {
        const port_pma* p = g->p;
        for (size_t r = 0; r < p->ntouched; ++r)
            for (uint64_t i = p->touched[2 * r]; i < p->touched[2 * r + 1]; ++i)
                if (p->st[i] == 1 && (p->keys[i] & 0xFFFFFFFFull) == GUARD_DST)
                    g->ro[(p->keys[i] >> 32) + 1] = i + 1;
    }
    if (out) *out = st;
    return PMA_OK;
}

int port_graph_row_offsets(port_graph* g, uint64_t* out) {
    memcpy(out, g->ro, (g->nv + 1) * 8);
    return PMA_OK;
}

/* is_entry_exist (graph.hpp:100-103) */
#define ENTRY(p, i) ((p)->st[i] == 1 && ((p)->keys[i] & 0xFFFFFFFFull) != GUARD_DST)

int port_bfs(port_graph* g, uint32_t root, uint32_t* dist) {
    /* analytics.hpp:22-48 (level-synchronous; distances are unique) */
    if (root >= g->nv) return fail(PMA_EINVAL, "bfs: root outside vertex range");
    const port_pma* p = g->p;
    uint32_t* q = (uint32_t*)malloc((g->nv + 1) * 4);
    for (size_t v = 0; v < g->nv; ++v) dist[v] = 0xFFFFFFFFu;
    size_t qh = 0, qt = 0;
    dist[root] = 0;
    q[qt++] = root;
    while (qh < qt) {
        const uint32_t u = q[qh++];
        for (uint64_t i = g->ro[u]; i < g->ro[u + 1]; ++i) {
            if (!ENTRY(p, i)) continue;
            const uint32_t v = (uint32_t)(p->keys[i] & 0xFFFFFFFFull);
            if (dist[v] == 0xFFFFFFFFu) {
                dist[v] = dist[u] + 1;
                q[qt++] = v;
            }
        }
    }
    free(q);
    return PMA_OK;
}

static uint32_t uf_find(uint32_t* par, uint32_t x) {
    while (par[x] != x) {
        par[x] = par[par[x]];
        x = par[x];
    }
    return x;
}

int port_cc(port_graph* g, uint32_t* labels) {
    /* analytics.hpp:53-82 yields the min vertex id per component of the
     * undirected closure; min-root union-find yields the same labels. */
    const port_pma* p = g->p;
    for (size_t v = 0; v < g->nv; ++v) labels[v] = (uint32_t)v;
    for (uint64_t i = 0; i < p->cap; ++i) {
        if (!ENTRY(p, i)) continue;
        uint32_t a = uf_find(labels, (uint32_t)(p->keys[i] >> 32));
        uint32_t b = uf_find(labels, (uint32_t)(p->keys[i] & 0xFFFFFFFFull));
        if (a < b) labels[b] = a;
        else if (b < a) labels[a] = b;
    }
    for (size_t v = 0; v < g->nv; ++v) labels[v] = uf_find(labels, (uint32_t)v);
    return PMA_OK;
}

int port_pagerank(port_graph* g, double d, double eps, size_t max_iters, const double* warm, double* x,
                  uint64_t* iters, int* converged) {
    /* analytics.hpp:100-143, same summation order */
    const size_t n = g->nv;
    if (n == 0) return fail(PMA_EINVAL, "pagerank: empty vertex set");
    const port_pma* p = g->p;
    uint64_t* outdeg = (uint64_t*)calloc(n, 8);
    double* y = (double*)malloc(n * 8);
    for (size_t v = 0; v < n; ++v) x[v] = warm ? warm[v] : 1.0 / (double)n;
    for (size_t u = 0; u < n; ++u)
        for (uint64_t i = g->ro[u]; i < g->ro[u + 1]; ++i) outdeg[u] += ENTRY(p, i);
    *converged = 0;
    size_t it;
    for (it = 1; it <= max_iters; ++it) {
        double dangling = 0.0;
        for (size_t u = 0; u < n; ++u)
            if (outdeg[u] == 0) dangling += x[u];
        const double base = (1.0 - d) / (double)n + d * dangling / (double)n;
        for (size_t u = 0; u < n; ++u) y[u] = base;
        for (size_t u = 0; u < n; ++u) {
            if (outdeg[u] == 0) continue;
            const double share = d * x[u] / (double)outdeg[u];
            for (uint64_t i = g->ro[u]; i < g->ro[u + 1]; ++i)
                if (ENTRY(p, i)) y[p->keys[i] & 0xFFFFFFFFull] += share;
        }
        double l1 = 0.0;
        for (size_t v = 0; v < n; ++v) l1 += fabs(y[v] - x[v]);
        memcpy(x, y, n * 8);
        if (l1 < eps) {
            *converged = 1;
            break;
        }
    }
    *iters = *converged ? it : max_iters;
    free(outdeg);
    free(y);
    return PMA_OK;
}

int port_spmv(port_graph* g, const double* x, double* y) {
    /* analytics.hpp:147-158 */
    const port_pma* p = g->p;
    for (size_t u = 0; u < g->nv; ++u) {
        double acc = 0.0;
        for (uint64_t i = g->ro[u]; i < g->ro[u + 1]; ++i) {
            if (!ENTRY(p, i)) continue;
            double w;
            memcpy(&w, &p->vals[i], 8);
            acc += w * x[p->keys[i] & 0xFFFFFFFFull];
        }
        y[u] = acc;
    }
    return PMA_OK;
}
