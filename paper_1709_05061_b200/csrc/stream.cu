// stream.cu — synthetic edge streams and the sliding window, on the device.
//
// Generators restate generators.hpp:26-89 and streaming.hpp:43-67 with the
// same std::mt19937_64 draws (the engine is fully specified by the C++
// standard), so they emit the reference's exact streams.
//
// SlidingWindow (streaming.hpp:76-123) is re-derived for the GPU: the window
// is a FIFO of stream positions [lo, cursor); a slide admits
// [cursor, cursor + take) and expires [lo, lo + take).  The reference emits a
// deletion for an expiring arrival p iff its key's multiplicity drops to zero,
// i.e. iff the key has no later arrival inside the new window:
// next_occurrence(p) >= cursor + take.  With next_occurrence precomputed once
// by a stable sort of (key, position), every slide is one ordered compaction
// — no hash map, and the emitted batches are byte-identical to the reference.
#include "radix.cuh"

#include <cmath>
#include <cstring>
#include <random>
#include <sstream>
#include <vector>

#include "pmagraph_cuda.h"
#include "pmagraph_stream.h"
#include "scan.cuh"

namespace gpma {

// draw_below / draw_unit (streaming.hpp:43-54)
static inline uint64_t draw_below(std::mt19937_64& rng, uint64_t bound) {
    const uint64_t limit = bound * (UINT64_MAX / bound);
    uint64_t x;
    do {
        x = rng();
    } while (x >= limit);
    return x % bound;
}

static inline double draw_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

struct Stream {
    uint64_t nv = 0;
    std::vector<uint32_t> src, dst;
};

__global__ void k_next_occ(const u64* sk, const u32* sp, u64 n, u32* next) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        next[sp[i]] = (i + 1 < n && sk[i + 1] == sk[i]) ? sp[i + 1] : 0xFFFFFFFFu;
}

__global__ void k_pack_stream(const u32* s, const u32* d, u64 n, u64* k, u32* p) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        k[i] = (u64(s[i]) << 32) | d[i];
        p[i] = u32(i);
    }
}

// Window state.  FIFO mode (every slide so far was a FIFO slide): the
// resident set is the position range [lo, cursor) and deletions come from
// next-occurrence positions.  General mode (after the first explicit random
// slide, streaming.hpp:129-158, whose evictions leave holes): the resident
// positions in window order + a multiplicity per distinct key (dense key ids
// from the stream's key sort), so an expiry's deletion is decided by counts.
struct Window {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t n = 0, lo = 0, cursor = 0;
    DevBuf<u32> src, dst, next;
    DevBuf<u32> kid;               // stream position -> dense key id
    DevBuf<u32> del_src, del_dst;  // all deletions emitted so far (appended)
    uint64_t ndel = 0;
    ScanWorkspace ws;
    DevBuf<ull> cnt;
    // general mode
    bool general = false;
    uint64_t wsize = 0;          // resident entries
    DevBuf<u32> res, res2;       // resident stream positions, window order
    DevBuf<u32> mult, lastpick;  // per key id: multiplicity; 1 + its last expiring index
    DevBuf<u8> picked;           // per index of (resident ++ arrivals): expires now
    DevBuf<u32> plist;           // drawn indices (explicit slides)
    // the last slide's expiries (SlideBatch::expiries): FIFO = stream
    // positions [exp_lo, exp_lo + exp_n); general = the picked entries of the
    // window before the slide (res2 after the swap + the arrivals from exp_cur)
    int exp_kind = 0;  // 0 none, 1 FIFO range, 2 general
    uint64_t exp_lo = 0, exp_n = 0, exp_old = 0, exp_tot = 0, exp_cur = 0;
};

__global__ void k_key_ids(const u32* sp, const u32* sorted_kid, u64 n, u32* kid) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        kid[sp[i]] = sorted_kid[i];
}

__global__ void k_iota_from(u32* out, u64 first, u64 n) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        out[i] = u32(first + i);
}

// multiplicity += 1 for stream positions [first, first + n)
__global__ void k_count_keys(u64 n, u64 first, const u32* kid, u32* mult) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        atomicAdd(&mult[kid[first + i]], 1u);
}

// the expiring indices of (resident ++ arrivals): the drawn list, or the FIFO
// front [0, ne).  release: flag it, drop its key's count, record the key's
// last expiring index; else: clear that record again
__global__ void k_mark_release(const u32* plist, u64 ne, const u32* res, u64 old, u64 cursor, const u32* kid,
                               u32* mult, u32* lastpick, u8* picked, int release) {
    for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < ne; t += u64(gridDim.x) * blockDim.x) {
        const u32 i = plist ? plist[t] : u32(t);
        const u32 p = i < old ? res[i] : u32(cursor + (i - old));
        const u32 k = kid[p];
        if (release) {
            picked[i] = 1;
            atomicSub(&mult[k], 1u);
            atomicMax(&lastpick[k], i + 1);
        } else {
            lastpick[k] = 0;
        }
    }
}

}  // namespace gpma

struct gpma_stream {
    gpma::Stream s;
};
struct gpma_window {
    gpma::Window w;
};

using gpma::ApiError;

namespace {
thread_local std::string g_stream_err;
template <class F>
int sguard(F&& f) {
    try {
        f();
        return PMA_OK;
    } catch (const ApiError& e) {
        g_stream_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_stream_err = e.what();
        return PMA_ECUDA;
    }
}
}  // namespace

struct gpma_rng {
    std::mt19937_64 r;
};

namespace gpma {

// A slide in general mode: FIFO (rng == nullptr, streaming.hpp:107-123) or
// explicit random eviction (streaming.hpp:129-158).  Arrivals are admitted
// first; the expiring indices of (resident ++ arrivals) release their keys;
// an expiry emits a deletion iff its key's multiplicity ends at zero and it
// is that key's last expiry in window order — what the reference's
// sequential releases give, since no admission happens between releases.
// The caller has reserved room for `take` more deletions.
static void slide_general(Window& W, size_t batch, std::mt19937_64* rng, gpma_slide_t* out) {
    const uint64_t remaining = W.n - W.cursor;
    const uint64_t take = batch < remaining ? batch : remaining;
    const uint64_t old = W.wsize, tot = old + take;
    out->ins_offset = W.cursor;
    out->n_ins = take;
    out->del_offset = W.ndel;
    out->final_partial = take < batch ? 1 : 0;
    out->n_del = 0;
    W.exp_kind = 1;
    W.exp_lo = 0;
    W.exp_n = 0;
    if (take == 0) return;
    // explicit: the expiring entries are drawn uniformly without replacement
    // among the window before the arrivals — the reference's exact draws
    uint64_t ne = take;
    const u32* plist = nullptr;
    if (rng) {
        ne = take < old ? take : old;
        std::vector<char> hp(old, 0);
        std::vector<u32> hl;
        hl.reserve(ne);
        for (uint64_t drawn = 0; drawn < ne;) {
            const uint64_t idx = draw_below(*rng, old);
            if (hp[idx]) continue;
            hp[idx] = 1;
            hl.push_back(u32(idx));
            ++drawn;
        }
        W.plist.reserve(ne + 1);
        if (ne) GPMA_CUDA(cudaMemcpy(W.plist.ptr, hl.data(), ne * 4, cudaMemcpyHostToDevice));
        plist = W.plist.ptr;
    }
    W.picked.reserve(tot + 1);
    W.res2.reserve(tot + 1);
    k_count_keys<<<grid_for(take, 256), 256, 0, W.stream>>>(take, W.cursor, W.kid.ptr, W.mult.ptr);  // admit
    GPMA_LAUNCH_CHECK();
    GPMA_CUDA(cudaMemsetAsync(W.picked.ptr, 0, tot, W.stream));
    if (ne) {
        k_mark_release<<<grid_for(ne, 256), 256, 0, W.stream>>>(plist, ne, W.res.ptr, old, W.cursor, W.kid.ptr,
                                                                W.mult.ptr, W.lastpick.ptr, W.picked.ptr, 1);
        GPMA_LAUNCH_CHECK();
    }
    uint64_t nd = 0;
    {
        const u8* pk = W.picked.ptr;
        const u32* res = W.res.ptr;
        const u32* kid = W.kid.ptr;
        const u32* mult = W.mult.ptr;
        const u32* lp = W.lastpick.ptr;
        const u32* ss = W.src.ptr;
        const u32* dd = W.dst.ptr;
        u32* os = W.del_src.ptr + W.ndel;
        u32* od = W.del_dst.ptr + W.ndel;
        u32* r2 = W.res2.ptr;
        ull* cnt = W.cnt.ptr;
        const uint64_t cur = W.cursor;
        GPMA_CUDA(cudaMemsetAsync(cnt, 0, 8, W.stream));
        // deletions, in window order
        run_compact(
            W.stream, W.ws, nullptr, tot, tot,
            [=] __device__(ull i) {
                if (!pk[i]) return false;
                const u32 k = kid[i < old ? res[i] : u32(cur + (i - old))];
                return mult[k] == 0 && lp[k] == u32(i + 1);
            },
            [=] __device__(ull i, unsigned f, ull x) {
                if (f) {
                    const u32 p = i < old ? res[i] : u32(cur + (i - old));
                    os[x] = ss[p];
                    od[x] = dd[p];
                }
            },
            [=] __device__(ull total) { *cnt = total; });
        // the new window: survivors, then the arrivals, in order
        run_compact(
            W.stream, W.ws, nullptr, tot, tot, [=] __device__(ull i) { return pk[i] == 0; },
            [=] __device__(ull i, unsigned f, ull x) {
                if (f) r2[x] = i < old ? res[i] : u32(cur + (i - old));
            },
            NoFin{});
        GPMA_CUDA(cudaMemcpyAsync(&nd, cnt, 8, cudaMemcpyDeviceToHost, W.stream));
    }
    if (ne) {
        k_mark_release<<<grid_for(ne, 256), 256, 0, W.stream>>>(plist, ne, W.res.ptr, old, W.cursor, W.kid.ptr,
                                                                W.mult.ptr, W.lastpick.ptr, W.picked.ptr, 0);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaStreamSynchronize(W.stream));
    std::swap(W.res.ptr, W.res2.ptr);
    std::swap(W.res.cap, W.res2.cap);
    W.exp_kind = 2;
    W.exp_n = ne;
    W.exp_old = old;
    W.exp_tot = tot;
    W.exp_cur = W.cursor;
    W.wsize = tot - ne;
    out->n_del = nd;
    W.ndel += nd;
    W.cursor += take;
}

// FIFO -> general mode: resident = positions [lo, cursor), counts from them
static void to_general(Window& W) {
    if (W.general) return;
    const uint64_t ws = W.cursor - W.lo;
    W.res.reserve(W.n + 1);
    W.res2.reserve(W.n + 1);
    W.mult.reserve(W.n + 1);
    W.lastpick.reserve(W.n + 1);
    GPMA_CUDA(cudaMemsetAsync(W.mult.ptr, 0, W.n * 4, W.stream));
    GPMA_CUDA(cudaMemsetAsync(W.lastpick.ptr, 0, W.n * 4, W.stream));
    if (ws) {
        k_iota_from<<<grid_for(ws, 256), 256, 0, W.stream>>>(W.res.ptr, W.lo, ws);
        GPMA_LAUNCH_CHECK();
        k_count_keys<<<grid_for(ws, 256), 256, 0, W.stream>>>(ws, W.lo, W.kid.ptr, W.mult.ptr);
        GPMA_LAUNCH_CHECK();
    }
    GPMA_CUDA(cudaStreamSynchronize(W.stream));
    W.wsize = ws;
    W.general = true;
}

}  // namespace gpma

extern "C" {

const char* gpma_stream_last_error(void) { return g_stream_err.c_str(); }

int gpma_rng_create(uint64_t seed, gpma_rng** out) {
    return sguard([&] { *out = new gpma_rng{std::mt19937_64(seed)}; });
}

int gpma_rng_destroy(gpma_rng* r) {
    delete r;
    return PMA_OK;
}

uint64_t gpma_window_size(const gpma_window* w) {
    if (!w) return 0;
    return w->w.general ? w->w.wsize : w->w.cursor - w->w.lo;
}

// gen_rmat (generators.hpp:26-63)
int gpma_stream_rmat(size_t nv, size_t ne, double a, double b, double c, double d, uint64_t seed,
                     gpma_stream** out) {
    return sguard([&] {
        if (nv == 0 || (nv & (nv - 1)) != 0) throw ApiError(PMA_EINVAL, "gen_rmat: num_vertices must be a power of two");
        const double sum = a + b + c + d;
        if (std::abs(sum - 1.0) > 1e-9 || a < 0 || b < 0 || c < 0 || d < 0)
            throw ApiError(PMA_EINVAL, "gen_rmat: quadrant probabilities must be non-negative and sum to 1");
        int scale = 0;
        while ((size_t{1} << scale) < nv) ++scale;
        auto* s = new gpma_stream;
        s->s.nv = nv;
        s->s.src.resize(ne);
        s->s.dst.resize(ne);
        std::mt19937_64 rng(seed);
        const double ab = a + b, abc = ab + c;
        for (size_t e = 0; e < ne; ++e) {
            uint64_t row = 0, col = 0;
            for (int bit = 0; bit < scale; ++bit) {
                // quadrant a:(0,0) b:(0,1) c:(1,0) d:(1,1), decided by the same
                // three comparisons as generators.hpp:47-58, without branches
                const double r = gpma::draw_unit(rng);
                const uint64_t rb = r >= ab;
                const uint64_t cb = uint64_t(r >= a) ^ rb ^ uint64_t(r >= abc);
                row = (row << 1) | rb;
                col = (col << 1) | cb;
            }
            s->s.src[e] = uint32_t(row);
            s->s.dst[e] = uint32_t(col);
        }
        *out = s;
    });
}

// gen_erdos_renyi (generators.hpp:67-89)
int gpma_stream_erdos_renyi(size_t nv, double density, uint64_t seed, gpma_stream** out) {
    return sguard([&] {
        if (density < 0.0 || density >= 1.0) throw ApiError(PMA_EINVAL, "gen_erdos_renyi: density must be in [0, 1)");
        auto* s = new gpma_stream;
        s->s.nv = nv;
        if (density > 0.0 && nv > 0) {
            std::mt19937_64 rng(seed);
            const double log1mp = std::log1p(-density);
            const uint64_t total = uint64_t(nv) * nv;
            uint64_t pos = 0;
            s->s.src.reserve(size_t(double(total) * density * 1.01) + 16);
            s->s.dst.reserve(size_t(double(total) * density * 1.01) + 16);
            for (;;) {
                const double u = gpma::draw_unit(rng);
                const double gap = std::floor(std::log1p(-u) / log1mp);
                pos += uint64_t(gap) + 1;
                if (pos > total) break;
                const uint64_t idx = pos - 1;
                s->s.src.push_back(uint32_t(idx / nv));
                s->s.dst.push_back(uint32_t(idx % nv));
            }
        }
        *out = s;
    });
}

// assign_random_timestamps (streaming.hpp:58-67): Fisher-Yates with draw_below
int gpma_stream_shuffle(gpma_stream* s, uint64_t seed) {
    if (!s) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        std::mt19937_64 rng(seed);
        auto& a = s->s.src;
        auto& b = s->s.dst;
        for (size_t i = a.size(); i > 1; --i) {
            const size_t j = size_t(gpma::draw_below(rng, i));
            std::swap(a[i - 1], a[j]);
            std::swap(b[i - 1], b[j]);
        }
    });
}

int gpma_stream_from_arrays(size_t nv, const uint32_t* src, const uint32_t* dst, size_t n, gpma_stream** out) {
    return sguard([&] {
        auto* s = new gpma_stream;
        s->s.nv = nv;
        s->s.src.assign(src, src + n);
        s->s.dst.assign(dst, dst + n);
        *out = s;
    });
}

uint64_t gpma_stream_size(const gpma_stream* s) { return s ? s->s.src.size() : 0; }
uint64_t gpma_stream_num_vertices(const gpma_stream* s) { return s ? s->s.nv : 0; }

int gpma_stream_edges(const gpma_stream* s, uint32_t* src, uint32_t* dst) {
    if (!s) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        if (src) std::memcpy(src, s->s.src.data(), s->s.src.size() * 4);
        if (dst) std::memcpy(dst, s->s.dst.data(), s->s.dst.size() * 4);
    });
}

int gpma_stream_destroy(gpma_stream* s) {
    delete s;
    return PMA_OK;
}

// draw_below over mt19937_64(seed): the bench's BFS-root sequence (bench.hpp:244,266)
int gpma_draw_below_sequence(uint64_t seed, uint64_t bound, size_t n, uint64_t* out) {
    return sguard([&] {
        std::mt19937_64 rng(seed);
        for (size_t i = 0; i < n; ++i) out[i] = gpma::draw_below(rng, bound);
    });
}

int gpma_window_create(const gpma_stream* s, int device, gpma_window** out) {
    if (!s) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        const uint64_t n = s->s.src.size();
        if (n < 2) throw ApiError(PMA_EINVAL, "SlidingWindow: stream needs at least two edges");
        if (n >= 0xFFFFFFFFull) throw ApiError(PMA_EINVAL, "SlidingWindow: stream too long for 32-bit positions");
        auto* w = new gpma_window;
        auto& W = w->w;
        W.device = device;
        GPMA_CUDA(cudaSetDevice(device));
        GPMA_CUDA(cudaStreamCreateWithFlags(&W.stream, cudaStreamNonBlocking));
        W.n = n;
        W.src.reserve(n);
        W.dst.reserve(n);
        W.next.reserve(n);
        W.cnt.reserve(2);
        GPMA_CUDA(cudaMemcpyAsync(W.src.ptr, s->s.src.data(), n * 4, cudaMemcpyHostToDevice, W.stream));
        GPMA_CUDA(cudaMemcpyAsync(W.dst.ptr, s->s.dst.data(), n * 4, cudaMemcpyHostToDevice, W.stream));
        {
            gpma::DevBuf<gpma::u64> k0, k1;
            gpma::DevBuf<gpma::u32> p0, p1;
            gpma::RadixWorkspace rws;
            k0.reserve(n);
            k1.reserve(n);
            p0.reserve(n);
            p1.reserve(n);
            gpma::k_pack_stream<<<gpma::grid_for(n, 256), 256, 0, W.stream>>>(W.src.ptr, W.dst.ptr, n, k0.ptr, p0.ptr);
            GPMA_LAUNCH_CHECK();
            const int alt = gpma::radix_sort(W.stream, rws, k0.ptr, k1.ptr, p0.ptr, p1.ptr, n, 0, 64);
            const gpma::u64* ks = alt ? k1.ptr : k0.ptr;  // sorted keys
            const gpma::u32* ps = alt ? p1.ptr : p0.ptr;  // their stream positions
            gpma::u32* pfree = alt ? p0.ptr : p1.ptr;     // the other payload buffer
            gpma::k_next_occ<<<gpma::grid_for(n, 256), 256, 0, W.stream>>>(ks, ps, n, W.next.ptr);
            GPMA_LAUNCH_CHECK();
            // dense key ids (general mode's multiplicity index): the rank of
            // the distinct key in the sorted order
            W.kid.reserve(n);
            {
                const gpma::u64* sk = ks;
                gpma::u32* sid = pfree;  // reused: per sorted index
                gpma::run_compact(
                    W.stream, W.ws, nullptr, n, n,
                    [=] __device__(gpma::ull i) { return i == 0 || sk[i] != sk[i - 1]; },
                    [=] __device__(gpma::ull i, unsigned f, gpma::ull x) { sid[i] = gpma::u32(x + f - 1); },
                    gpma::NoFin{});
                gpma::k_key_ids<<<gpma::grid_for(n, 256), 256, 0, W.stream>>>(ps, sid, n, W.kid.ptr);
                GPMA_LAUNCH_CHECK();
            }
            GPMA_CUDA(cudaStreamSynchronize(W.stream));
        }
        W.lo = 0;
        W.cursor = (n + 1) / 2;  // streaming.hpp:83-85
        *out = w;
    });
}

int gpma_window_destroy(gpma_window* w) {
    if (!w) return PMA_OK;
    cudaSetDevice(w->w.device);
    cudaStreamSynchronize(w->w.stream);
    cudaStreamDestroy(w->w.stream);
    delete w;
    return PMA_OK;
}

int gpma_window_info(const gpma_window* w, gpma_window_info_t* out) {
    if (!w || !out) return PMA_EINVAL;
    out->stream_src = w->w.src.ptr;
    out->stream_dst = w->w.dst.ptr;
    out->del_src = w->w.del_src.ptr;
    out->del_dst = w->w.del_dst.ptr;
    out->stream_size = w->w.n;
    out->initial_size = (w->w.n + 1) / 2;
    out->cursor = w->w.cursor;
    out->num_deletions = w->w.ndel;
    return PMA_OK;
}

// Reserve room for `max_deletions` appended deletions (device pointers in
// gpma_window_info stay valid until the next reserve).
int gpma_window_reserve(gpma_window* w, size_t max_deletions) {
    if (!w) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        auto& W = w->w;
        if (max_deletions <= W.del_src.cap) return;
        GPMA_CUDA(cudaSetDevice(W.device));
        gpma::DevBuf<gpma::u32> a, b;
        a.reserve(max_deletions);
        b.reserve(max_deletions);
        if (W.ndel) {
            GPMA_CUDA(cudaMemcpyAsync(a.ptr, W.del_src.ptr, W.ndel * 4, cudaMemcpyDeviceToDevice, W.stream));
            GPMA_CUDA(cudaMemcpyAsync(b.ptr, W.del_dst.ptr, W.ndel * 4, cudaMemcpyDeviceToDevice, W.stream));
        }
        GPMA_CUDA(cudaStreamSynchronize(W.stream));
        std::swap(W.del_src.ptr, a.ptr);
        std::swap(W.del_src.cap, a.cap);
        std::swap(W.del_dst.ptr, b.ptr);
        std::swap(W.del_dst.cap, b.cap);
    });
}

// SlidingWindow::slide (streaming.hpp:107-123) on the device.  Inserts are
// stream positions [ins_offset, ins_offset + n_ins); deletions are appended
// at [del_offset, del_offset + n_del) of the window's deletion arrays.
int gpma_window_slide(gpma_window* w, size_t batch, gpma_slide_t* out) {
    if (!w) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        auto& W = w->w;
        GPMA_CUDA(cudaSetDevice(W.device));
        const uint64_t remaining = W.n - W.cursor;
        const uint64_t take = batch < remaining ? batch : remaining;
        const uint64_t end = W.cursor + take;
        if (W.ndel + take > W.del_src.cap) {
            const size_t want = size_t((W.ndel + take) * 2 + 1024);
            int rc = gpma_window_reserve(w, want);
            if (rc) throw ApiError(rc, g_stream_err);
        }
        if (W.general) {  // after an explicit random slide the window has holes
            gpma::slide_general(W, batch, nullptr, out);
            return;
        }
        out->ins_offset = W.cursor;
        out->n_ins = take;
        out->del_offset = W.ndel;
        out->final_partial = take < batch ? 1 : 0;
        uint64_t nd = 0;
        if (take > 0) {
            const gpma::u32* nx = W.next.ptr;
            const gpma::u32* ss = W.src.ptr;
            const gpma::u32* dd = W.dst.ptr;
            gpma::u32* os = W.del_src.ptr + W.ndel;
            gpma::u32* od = W.del_dst.ptr + W.ndel;
            gpma::ull* cnt = W.cnt.ptr;
            const uint64_t lo = W.lo;
            GPMA_CUDA(cudaMemsetAsync(cnt, 0, 8, W.stream));
            gpma::run_compact(
                W.stream, W.ws, nullptr, take, take,
                [=] __device__(gpma::ull i) { return uint64_t(nx[lo + i]) >= end; },
                [=] __device__(gpma::ull i, unsigned f, gpma::ull x) {
                    if (f) {
                        os[x] = ss[lo + i];
                        od[x] = dd[lo + i];
                    }
                },
                [=] __device__(gpma::ull total) { *cnt = total; });
            GPMA_CUDA(cudaMemcpyAsync(&nd, cnt, 8, cudaMemcpyDeviceToHost, W.stream));
            GPMA_CUDA(cudaStreamSynchronize(W.stream));
        }
        out->n_del = nd;
        W.ndel += nd;
        W.exp_kind = 1;
        W.exp_lo = W.lo;
        W.exp_n = take;
        W.lo += take;
        W.cursor = end;
    });
}

// SlideBatch::expiries of the last slide as stream positions, window order.
int gpma_window_last_expiries(gpma_window* w, uint32_t* positions, size_t cap, size_t* n) {
    if (!w) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        auto& W = w->w;
        GPMA_CUDA(cudaSetDevice(W.device));
        if (n) *n = W.exp_n;
        const uint64_t m = std::min<uint64_t>(cap, W.exp_n);
        if (!positions || m == 0) return;
        if (W.exp_kind == 1) {
            for (uint64_t i = 0; i < m; ++i) positions[i] = uint32_t(W.exp_lo + i);
            return;
        }
        gpma::DevBuf<gpma::u32> out;
        out.reserve(W.exp_n + 1);
        const gpma::u8* pk = W.picked.ptr;
        const gpma::u32* res = W.res2.ptr;  // the window before the slide
        const uint64_t old = W.exp_old, cur = W.exp_cur;
        gpma::u32* o = out.ptr;
        gpma::run_compact(
            W.stream, W.ws, nullptr, W.exp_tot, W.exp_tot, [=] __device__(gpma::ull i) { return pk[i] != 0; },
            [=] __device__(gpma::ull i, unsigned f, gpma::ull x) {
                if (f) o[x] = i < old ? res[i] : gpma::u32(cur + (i - old));
            },
            gpma::NoFin{});
        GPMA_CUDA(cudaMemcpyAsync(positions, out.ptr, m * 4, cudaMemcpyDeviceToHost, W.stream));
        GPMA_CUDA(cudaStreamSynchronize(W.stream));
    });
}

// SlidingWindow::distinct_edges (streaming.hpp:162-169): the window's
// distinct edges, ascending key order (the reference's order is a hash map's,
// i.e. unspecified).  Two-call protocol: cap = 0 returns the count.
int gpma_window_distinct_edges(gpma_window* w, uint32_t* src, uint32_t* dst, size_t cap, size_t* n) {
    if (!w) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        auto& W = w->w;
        GPMA_CUDA(cudaSetDevice(W.device));
        const uint64_t ws = W.general ? W.wsize : W.cursor - W.lo;
        gpma::DevBuf<gpma::u64> k0, k1;
        k0.reserve(ws + 1);
        k1.reserve(ws + 1);
        W.cnt.reserve(2);
        gpma::ull* cnt = W.cnt.ptr;
        uint64_t nd = 0;
        if (ws) {
            gpma::u64* kk = k0.ptr;
            const gpma::u32* ss = W.src.ptr;
            const gpma::u32* dd = W.dst.ptr;
            const gpma::u32* res = W.res.ptr;
            const bool gen = W.general;
            const uint64_t lo = W.lo;
            gpma::run_compact(
                W.stream, W.ws, nullptr, ws, ws, [=] __device__(gpma::ull) { return true; },
                [=] __device__(gpma::ull i, unsigned, gpma::ull) {
                    const gpma::u32 p = gen ? res[i] : gpma::u32(lo + i);
                    kk[i] = gpma::pack_edge(ss[p], dd[p]);
                },
                gpma::NoFin{});
            gpma::RadixWorkspace rws;
            const int alt = gpma::radix_sort(W.stream, rws, k0.ptr, k1.ptr, nullptr, nullptr, ws, 0, 64);
            const gpma::u64* sk = alt ? k1.ptr : k0.ptr;
            gpma::u64* uq = alt ? k0.ptr : k1.ptr;
            gpma::run_compact(
                W.stream, W.ws, nullptr, ws, ws, [=] __device__(gpma::ull i) { return i == 0 || sk[i] != sk[i - 1]; },
                [=] __device__(gpma::ull i, unsigned f, gpma::ull x) {
                    if (f) uq[x] = sk[i];
                },
                [=] __device__(gpma::ull total) { *cnt = total; });
            GPMA_CUDA(cudaMemcpyAsync(&nd, cnt, 8, cudaMemcpyDeviceToHost, W.stream));
            GPMA_CUDA(cudaStreamSynchronize(W.stream));
            if (n) *n = nd;
            const uint64_t m = std::min<uint64_t>(cap, nd);
            if (m && src && dst) {
                std::vector<gpma::u64> h(m);
                GPMA_CUDA(cudaMemcpyAsync(h.data(), uq, m * 8, cudaMemcpyDeviceToHost, W.stream));
                GPMA_CUDA(cudaStreamSynchronize(W.stream));
                for (uint64_t i = 0; i < m; ++i) {
                    src[i] = gpma::src_of(h[i]);
                    dst[i] = gpma::dst_of(h[i]);
                }
            }
            return;
        }
        if (n) *n = 0;
    });
}

// std::mt19937_64 state through its standard text form, so a caller's
// generator can drive gpma_window_slide_explicit_random and advance exactly
// as the reference's would (streaming.hpp:129 takes it by reference).
int gpma_rng_set_state(gpma_rng* r, const char* text) {
    if (!r) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        std::istringstream is(text ? text : "");
        is >> r->r;
        if (!is) throw ApiError(PMA_EINVAL, "rng state: not a std::mt19937_64 text state");
    });
}

int gpma_rng_get_state(const gpma_rng* r, char* buf, size_t cap, size_t* len) {
    if (!r) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        std::ostringstream os;
        os << r->r;
        const std::string t = os.str();
        if (len) *len = t.size() + 1;
        if (buf && cap) {
            const size_t m = std::min(cap - 1, t.size());
            std::memcpy(buf, t.data(), m);
            buf[m] = 0;
        }
    });
}

// SlidingWindow::slide_explicit_random (streaming.hpp:129-158): arrivals as
// in gpma_window_slide; the expiring edges are drawn by `rng` (its state
// advances) uniformly without replacement from the window as it stood before
// the arrivals; deletions appended as gpma_window_slide's.
int gpma_window_slide_explicit_random(gpma_window* w, size_t batch, gpma_rng* rng, gpma_slide_t* out) {
    if (!w) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        auto& W = w->w;
        if (!rng) throw ApiError(PMA_EINVAL, "slide_explicit_random: null rng");
        GPMA_CUDA(cudaSetDevice(W.device));
        const uint64_t remaining = W.n - W.cursor;
        const uint64_t take = batch < remaining ? batch : remaining;
        if (W.ndel + take > W.del_src.cap) {
            int rc = gpma_window_reserve(w, size_t((W.ndel + take) * 2 + 1024));
            if (rc) throw ApiError(rc, g_stream_err);
        }
        gpma::to_general(W);
        gpma::slide_general(W, batch, &rng->r, out);
    });
}

}  // extern "C"

extern "C" int gpma_window_deletions_host(gpma_window* w, size_t offset, size_t n, uint32_t* src, uint32_t* dst) {
    if (!w) {
        g_stream_err = "null handle";
        return PMA_EINVAL;
    }
    return sguard([&] {
        auto& W = w->w;
        if (offset + n > W.ndel) throw ApiError(PMA_ERANGE, "window deletions: range outside emitted deletions");
        GPMA_CUDA(cudaSetDevice(W.device));
        if (n && src) GPMA_CUDA(cudaMemcpyAsync(src, W.del_src.ptr + offset, n * 4, cudaMemcpyDeviceToHost, W.stream));
        if (n && dst) GPMA_CUDA(cudaMemcpyAsync(dst, W.del_dst.ptr + offset, n * 4, cudaMemcpyDeviceToHost, W.stream));
        GPMA_CUDA(cudaStreamSynchronize(W.stream));
    });
}
