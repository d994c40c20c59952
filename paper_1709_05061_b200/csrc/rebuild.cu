// rebuild.cu — the rebuild-the-CSR-per-batch baseline (RebuildCsrGraph,
// baselines.hpp:85-181) on the device: the paper's comparison point for
// GPMA+ ("cuSparseCSR" rebuild).  State = the sorted
// unique edge keys + values and the CSR arrays derived from them; a batch is
// sorted, duplicates resolved (last insert wins), merged into the edge list
// (matches removed, inserts added) and the whole CSR rebuilt.  Its cost is
// O(|E|) per batch whatever the batch size — the point of the comparison.
#include "radix.cuh"

#include <chrono>
#include <cstring>
#include <string>

#include "block_ops.cuh"
#include "pmagraph_cuda.h"
#include "scan.cuh"

namespace gpma {

struct RbCtr {
    ull nu, ns, ni, missed, bad;
};

__global__ void k_rb_pack(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd, u64 nd,
                          u64* keys, u32* idx) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < ni + nd; i += u64(gridDim.x) * blockDim.x) {
        keys[i] = i < ni ? pack_edge(is[i], id[i]) : pack_edge(ds[i - ni], dd[i - ni]);
        idx[i] = u32(i);
    }
}

__global__ void k_rb_check(const u32* s, const u32* d, u64 n, u64 nv, RbCtr* c) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        if (s[i] >= nv || d[i] >= nv) atomicOr(&c->bad, 1ull);
}

// every update: the edge it matches (if any) is removed; unmatched deletes are missed
__global__ void k_rb_match(const u64* uk, const u8* uop, const ull* nu, const u64* ek, u64 ne, u8* gone, RbCtr* c) {
    ull missed = 0;
    for (u64 j = blockIdx.x * u64(blockDim.x) + threadIdx.x; j < *nu; j += u64(gridDim.x) * blockDim.x) {
        const u64 p = lower_bound_dev(ek, ne, uk[j]);
        const bool hit = p < ne && ek[p] == uk[j];
        if (hit) gone[p] = 1;
        else missed += uop[j] == kOpDelete;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) missed += __shfl_xor_sync(FULL, missed, o);
    if ((threadIdx.x & 31) == 0 && missed) atomicAdd(&c->missed, missed);
}

// merge: survivor r lands at r + #inserts below it, insert j at j + #survivors below it
__global__ void k_rb_merge(const u64* sk, const u64* sv, const ull* ns, const u64* ik, const u64* iv, const ull* ni,
                           u64* ok, u64* ov) {
    const u64 a = *ns, b = *ni;
    for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < a + b; t += u64(gridDim.x) * blockDim.x) {
        if (t < a) {
            const u64 o = t + lower_bound_dev(ik, b, sk[t]);
            ok[o] = sk[t];
            ov[o] = sv[t];
        } else {
            const u64 j = t - a;
            const u64 o = j + lower_bound_dev(sk, a, ik[j]);
            ok[o] = ik[j];
            ov[o] = iv[j];
        }
    }
}

// CSR: row_offsets[u] = first edge with src >= u; col / val from the keys
__global__ void k_rb_csr(const u64* ek, u64 ne, u64 nv, u64* ro, u32* col, double* val, const u64* ev) {
    for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < ne + nv + 1; t += u64(gridDim.x) * blockDim.x) {
        if (t <= nv) ro[t] = t == nv ? ne : lower_bound_dev(ek, ne, t << 32);
        if (t < ne) {
            col[t] = dst_of(ek[t]);
            val[t] = __longlong_as_double((long long)ev[t]);
        }
    }
}

class RebuildCsr {
public:
    RebuildCsr(int device, u64 nv) : dev(device), nv(nv) {
        GPMA_CUDA(cudaSetDevice(dev));
        GPMA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        GPMA_CUDA(cudaMalloc(&c, sizeof(RbCtr)));
        ro.reserve(nv + 1);
    }
    ~RebuildCsr() {
        cudaSetDevice(dev);
        cudaStreamSynchronize(s);
        if (c) cudaFree(c);
        if (s) cudaStreamDestroy(s);
    }

    // RebuildCsrGraph(num_vertices, edges): ids checked, sorted, last wins
    void build(const u32* src, const u32* dst, const double* w, u64 n) {
        GPMA_CUDA(cudaMemsetAsync(c, 0, sizeof(RbCtr), s));
        if (n) k_rb_check<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, nv, c);
        RbCtr h{};
        GPMA_CUDA(cudaMemcpyAsync(&h, c, sizeof(RbCtr), cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        if (h.bad) throw ApiError(PMA_EINVAL, "RebuildCsrGraph: vertex id out of range");
        sort_resolve(src, dst, w, n, nullptr, nullptr, 0, /*edges=*/true);
        const u64 nu = read(&c->nu);
        ek.reserve(nu + 1);
        ev.reserve(nu + 1);
        GPMA_CUDA(cudaMemcpyAsync(ek.ptr, uk.ptr, nu * 8, cudaMemcpyDeviceToDevice, s));
        GPMA_CUDA(cudaMemcpyAsync(ev.ptr, uv.ptr, nu * 8, cudaMemcpyDeviceToDevice, s));
        ne = nu;
        rebuild();
        GPMA_CUDA(cudaStreamSynchronize(s));
    }

    // RebuildCsrGraph::apply_batch (baselines.hpp:117-155)
    void apply(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd, u64 nd,
               pma_stats* out) {
        const auto t0 = std::chrono::steady_clock::now();
        pma_stats st;
        std::memset(&st, 0, sizeof(st));
        st.batch_size = ni + nd;
        GPMA_CUDA(cudaMemsetAsync(c, 0, sizeof(RbCtr), s));
        sort_resolve(is, id, iw, ni, ds, dd, nd, false);
        const u64 n = ni + nd;
        gone.reserve(ne + 1);
        if (ne) GPMA_CUDA(cudaMemsetAsync(gone.ptr, 0, ne, s));
        if (n) {
            k_rb_match<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(uk.ptr, uop.ptr, &c->nu, ek.ptr, ne, gone.ptr, c);
            GPMA_LAUNCH_CHECK();
        }
        // survivors of the edge list, and the inserts of the batch, in key order
        sk.reserve(ne + 1);
        sv.reserve(ne + 1);
        ik.reserve(n + 1);
        iv.reserve(n + 1);
        {
            const u64* k = ek.ptr;
            const u64* v = ev.ptr;
            const u8* g = gone.ptr;
            u64* ok = sk.ptr;
            u64* ov = sv.ptr;
            RbCtr* cc = c;
            run_compact(
                s, ws, nullptr, ne, ne, [=] __device__(ull i) { return g[i] == 0; },
                [=] __device__(ull i, unsigned f, ull x) {
                    if (f) {
                        ok[x] = k[i];
                        ov[x] = v[i];
                    }
                },
                [=] __device__(ull total) { cc->ns = total; });
        }
        {
            const u64* k = uk.ptr;
            const u64* v = uv.ptr;
            const u8* o = uop.ptr;
            u64* ok = ik.ptr;
            u64* ov = iv.ptr;
            RbCtr* cc = c;
            run_compact(
                s, ws, &c->nu, 0, n, [=] __device__(ull j) { return o[j] == kOpInsert; },
                [=] __device__(ull j, unsigned f, ull x) {
                    if (f) {
                        ok[x] = k[j];
                        ov[x] = v[j];
                    }
                },
                [=] __device__(ull total) { cc->ni = total; });
        }
        RbCtr h{};
        GPMA_CUDA(cudaMemcpyAsync(&h, c, sizeof(RbCtr), cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        const u64 ne2 = h.ns + h.ni;
        ek2.reserve(ne2 + 1);
        ev2.reserve(ne2 + 1);
        if (ne2) {
            k_rb_merge<<<grid_for(ne2, 256, 148 * 16), 256, 0, s>>>(sk.ptr, sv.ptr, &c->ns, ik.ptr, iv.ptr, &c->ni,
                                                                    ek2.ptr, ev2.ptr);
            GPMA_LAUNCH_CHECK();
        }
        std::swap(ek.ptr, ek2.ptr);
        std::swap(ek.cap, ek2.cap);
        std::swap(ev.ptr, ev2.ptr);
        std::swap(ev.cap, ev2.cap);
        ne = ne2;
        rebuild();
        GPMA_CUDA(cudaStreamSynchronize(s));
        st.deletes_missed = h.missed;
        st.slot_writes = 2 * ne + nv + 1;  // baselines.hpp:153
        st.num_levels = 0;  // no segment levels (segments_per_level empty)
        st.wall_ns = u64(std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
                             .count());
        if (out) *out = st;
    }

    void csr(u64* h_ro, u32* h_col, double* h_val) {
        GPMA_CUDA(cudaMemcpyAsync(h_ro, ro.ptr, (nv + 1) * 8, cudaMemcpyDeviceToHost, s));
        if (ne) {
            GPMA_CUDA(cudaMemcpyAsync(h_col, col.ptr, ne * 4, cudaMemcpyDeviceToHost, s));
            GPMA_CUDA(cudaMemcpyAsync(h_val, val.ptr, ne * 8, cudaMemcpyDeviceToHost, s));
        }
        GPMA_CUDA(cudaStreamSynchronize(s));
    }

    u64 num_edges() const { return ne; }
    cudaStream_t stream() const { return s; }
    std::string err;

    // (extended __device__ lambdas need public enclosing functions)
    void sort_resolve(const u32* is, const u32* id, const double* iw, u64 ni, const u32* ds, const u32* dd, u64 nd,
                      bool edges) {
        const u64 n = ni + nd;
        k0.reserve(n + 1);
        k1.reserve(n + 1);
        i0.reserve(n + 1);
        i1.reserve(n + 1);
        uk.reserve(n + 1);
        uv.reserve(n + 1);
        uop.reserve(n + 1);
        if (n == 0) {
            GPMA_CUDA(cudaMemsetAsync(&c->nu, 0, 8, s));
            return;
        }
        k_rb_pack<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(is, id, iw, ni, ds, dd, nd, k0.ptr, i0.ptr);
        GPMA_LAUNCH_CHECK();
        const int alt = radix_sort(s, rws, k0.ptr, k1.ptr, i0.ptr, i1.ptr, n, 0, 64);
        const u64* k = alt ? k1.ptr : k0.ptr;
        const u32* ix = alt ? i1.ptr : i0.ptr;
        u64* ok = uk.ptr;
        u64* ov = uv.ptr;
        u8* oo = uop.ptr;
        RbCtr* cc = c;
        const u64 nins = ni;
        // equal-key runs: edges keep the last arrival (dedupe_last_wins); a batch
        // keeps its last insert if any, else a delete (resolve_duplicates)
        run_compact(
            s, ws, nullptr, n, n, [=] __device__(ull i) { return i + 1 == n || k[i + 1] != k[i]; },
            [=] __device__(ull i, unsigned f, ull x) {
                if (!f) return;
                u8 op = kOpDelete;
                u64 val = 0;
                for (long long t = (long long)i; t >= 0 && k[t] == k[i]; --t) {
                    const u32 a = ix[t];
                    if (edges || a < nins) {
                        op = kOpInsert;
                        val = u64(__double_as_longlong(iw ? iw[a] : 1.0));
                        break;
                    }
                }
                ok[x] = k[i];
                ov[x] = val;
                oo[x] = op;
            },
            [=] __device__(ull total) { cc->nu = total; });
    }

    void rebuild() {
        ro.reserve(nv + 1);
        col.reserve(ne + 1);
        val.reserve(ne + 1);
        k_rb_csr<<<grid_for(ne + nv + 1, 256, 148 * 16), 256, 0, s>>>(ek.ptr, ne, nv, ro.ptr, col.ptr, val.ptr,
                                                                      ev.ptr);
        GPMA_LAUNCH_CHECK();
    }

    u64 read(const ull* p) {
        u64 v = 0;
        GPMA_CUDA(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, s));
        GPMA_CUDA(cudaStreamSynchronize(s));
        return v;
    }

    int dev;
    u64 nv;
    cudaStream_t s = nullptr;
    RbCtr* c = nullptr;
    u64 ne = 0;
    DevBuf<u64> ek, ev, ek2, ev2, sk, sv, ik, iv, uk, uv, k0, k1, ro;
    DevBuf<u32> i0, i1, col;
    DevBuf<double> val;
    DevBuf<u8> uop, gone;
    RadixWorkspace rws;
    DevBuf<u32> sa, sb, sc, sd;
    DevBuf<double> sw;
    ScanWorkspace ws;
};

}  // namespace gpma

// ---- C ABI (include/pmagraph_cuda.h, "rebuild-CSR baseline")
struct gpma_rebuild {
    gpma::RebuildCsr* impl = nullptr;
};

namespace {
thread_local std::string g_rb_err;
template <class F>
int rb_guard(std::string* err, F&& f) {
    try {
        f();
        return PMA_OK;
    } catch (const gpma::ApiError& e) {
        if (err) *err = e.what();
        g_rb_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (err) *err = e.what();
        g_rb_err = e.what();
        return PMA_ECUDA;
    }
}
template <class T>
const T* rb_stage(gpma::DevBuf<T>& b, const T* host, size_t n, cudaStream_t s) {
    b.reserve(n ? n : 1);
    if (n) GPMA_CUDA(cudaMemcpyAsync(b.ptr, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return b.ptr;
}
}  // namespace

extern "C" {

int gpma_rebuild_create_device(int device, size_t num_vertices, const uint32_t* d_src, const uint32_t* d_dst,
                               const double* d_w, size_t n, gpma_rebuild** out) {
    return rb_guard(nullptr, [&] {
        auto* r = new gpma_rebuild;
        try {
            r->impl = new gpma::RebuildCsr(device, num_vertices);
            r->impl->build(d_src, d_dst, d_w, n);
        } catch (...) {
            delete r->impl;
            delete r;
            throw;
        }
        *out = r;
    });
}

int gpma_rebuild_create(int device, size_t num_vertices, const uint32_t* src, const uint32_t* dst, const double* w,
                        size_t n, gpma_rebuild** out) {
    return rb_guard(nullptr, [&] {
        auto* r = new gpma_rebuild;
        try {
            r->impl = new gpma::RebuildCsr(device, num_vertices);
            auto& g = *r->impl;
            const uint32_t* a = rb_stage(g.sa, src, n, g.s);
            const uint32_t* b = rb_stage(g.sb, dst, n, g.s);
            const double* ww = w ? rb_stage(g.sw, w, n, g.s) : nullptr;
            g.build(a, b, ww, n);
        } catch (...) {
            delete r->impl;
            delete r;
            throw;
        }
        *out = r;
    });
}

int gpma_rebuild_destroy(gpma_rebuild* r) {
    if (!r) return PMA_OK;
    delete r->impl;
    delete r;
    return PMA_OK;
}

const char* gpma_rebuild_last_error(const gpma_rebuild* r) {
    return r && r->impl ? r->impl->err.c_str() : g_rb_err.c_str();
}

int gpma_rebuild_apply_batch_device(gpma_rebuild* r, const uint32_t* d_ins_src, const uint32_t* d_ins_dst,
                                    const double* d_ins_w, size_t n_ins, const uint32_t* d_del_src,
                                    const uint32_t* d_del_dst, size_t n_del, pma_stats* stats) {
    if (!r || !r->impl) {
        g_rb_err = "null handle";
        return PMA_EINVAL;
    }
    return rb_guard(&r->impl->err, [&] {
        GPMA_CUDA(cudaSetDevice(r->impl->dev));
        r->impl->apply(d_ins_src, d_ins_dst, d_ins_w, n_ins, d_del_src, d_del_dst, n_del, stats);
    });
}

int gpma_rebuild_apply_batch(gpma_rebuild* r, const uint32_t* ins_src, const uint32_t* ins_dst, const double* ins_w,
                             size_t n_ins, const uint32_t* del_src, const uint32_t* del_dst, size_t n_del,
                             pma_stats* stats) {
    if (!r || !r->impl) {
        g_rb_err = "null handle";
        return PMA_EINVAL;
    }
    return rb_guard(&r->impl->err, [&] {
        auto& g = *r->impl;
        GPMA_CUDA(cudaSetDevice(g.dev));
        const uint32_t* a = rb_stage(g.sa, ins_src, n_ins, g.s);
        const uint32_t* b = rb_stage(g.sb, ins_dst, n_ins, g.s);
        const double* w = ins_w ? rb_stage(g.sw, ins_w, n_ins, g.s) : nullptr;
        const uint32_t* c2 = rb_stage(g.sc, del_src, n_del, g.s);
        const uint32_t* d = rb_stage(g.sd, del_dst, n_del, g.s);
        g.apply(a, b, w, n_ins, c2, d, n_del, stats);
    });
}

int gpma_rebuild_csr(gpma_rebuild* r, uint64_t* row_offsets, uint32_t* col, double* vals) {
    if (!r || !r->impl) {
        g_rb_err = "null handle";
        return PMA_EINVAL;
    }
    return rb_guard(&r->impl->err, [&] {
        GPMA_CUDA(cudaSetDevice(r->impl->dev));
        r->impl->csr(row_offsets, col, vals);
    });
}

uint64_t gpma_rebuild_num_edges(const gpma_rebuild* r) { return r && r->impl ? r->impl->num_edges() : 0; }

void* gpma_rebuild_cuda_stream(gpma_rebuild* r) { return r && r->impl ? (void*)r->impl->stream() : nullptr; }

}  // extern "C"
