// seq_ops.cu — the reference's sequential single-key PMA operations on the
// device (pma.hpp:294-386, 471-479).  Their semantics differ from a one-update
// batch (in-place overwrite and tombstone revival; an insert that reaches a
// full root grows the array and retries from the leaf), so they get their own
// path: one CTA walks the levels with CTA-wide counts, merges the first
// segment that fits (block_merge_segment) and refreshes that range's leaf
// headers.  Growth / shrink rebuilds run on the host-orchestrated
// device-wide path.  No CPU fallback.
#include <cstring>

#include "merge.cuh"
#include "pma_impl.cuh"

namespace gpma {

struct SeqBounds {
    u64 mn[PMA_MAX_LEVELS];
    u64 mx[PMA_MAX_LEVELS];
};

struct SeqResult {
    int status;  // 0 done, 1 need grow (insert), 2 need shrink check (erase at root)
    int flag;    // erase/mark: 1 if the key was removed/marked
    long long vd, td;
    ull writes;
};

enum SeqOp { kSeqInsert = 0, kSeqErase = 1, kSeqMark = 2, kSeqRedispatch = 3 };

struct SeqArgs {
    u64* keys;
    u64* vals;
    u8* st;
    u64* hdr;
    u64 cap, leaf;
    int height;
    int allow_shrink;
    int op;
    u64 key, value;
    // redispatch
    int rlevel;
    u64 rseg;
    const u64* xk;
    const u64* xv;
    u64 xn;
    SeqBounds bnd;
    u64 *ek, *ev, *okk, *ovv, *ik, *iv;
    u32 *es, *ir;
    u8* mflag;
    SeqResult* res;
};

// hdr refresh for the leaves of [b, e) plus the empty run to their left
__device__ void block_refresh_range(const SeqArgs& a, u64 b, u64 e) {
    for (u64 i = b / a.leaf + threadIdx.x; i < (e + a.leaf - 1) / a.leaf; i += blockDim.x) {
        u64 v = ~0ull;
        for (u64 t = i * a.leaf; t < a.cap; ++t)
            if (a.st[t] != kEmpty) {
                v = a.keys[t];
                break;
            }
        a.hdr[i] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const u64 la = b / a.leaf;
        const u64 v = a.hdr[la];
        for (u64 i = la; i-- > 0;) {
            bool empty = true;
            for (u64 t = i * a.leaf; t < (i + 1) * a.leaf; ++t)
                if (a.st[t] != kEmpty) {
                    empty = false;
                    break;
                }
            if (!empty) break;
            a.hdr[i] = v;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kCtaThreads) k_seq(SeqArgs a) {
    __shared__ ull s_w64[kCtaThreads / 32];
    __shared__ u64 s_key, s_val;
    __shared__ u8 s_op;
    __shared__ long long s_slot;
    const u64 L = a.cap / a.leaf;
    if (threadIdx.x == 0) {
        s_key = a.key;
        s_val = a.value;
        s_op = a.op == kSeqErase ? kOpDelete : kOpInsert;
        s_slot = -1;
        a.res->status = 0;
        a.res->flag = 0;
        a.res->vd = a.res->td = 0;
        a.res->writes = 0;
    }
    __syncthreads();
    if (a.op == kSeqRedispatch) {
        const u64 m = a.leaf << a.rlevel;
        const u64 b = a.rseg * m;
        ull nv = 0, nt = 0;
        for (u64 t = threadIdx.x; t < m; t += kCtaThreads) {
            nv += a.st[b + t] == kValid;
            nt += a.st[b + t] == kTombstone;
        }
        nv = block_sum(nv, s_w64);
        nt = block_sum(nt, s_w64);
        if (nv + a.xn > a.bnd.mx[a.rlevel]) {
            if (threadIdx.x == 0) a.res->status = 3;  // capacity violation
            return;
        }
        SliceDirect sl{a.xk, a.xv, nullptr};
        const MergeOut r = block_merge_segment(a.keys, a.vals, a.st, b, m, nv, sl, a.xn, false, a.ek, a.ev, a.es,
                                               a.mflag, a.okk, a.ovv, a.ik, a.iv, a.ir);
        block_refresh_range(a, b, b + m);
        if (threadIdx.x == 0) {
            a.res->vd = (long long)r.k - (long long)nv;
            a.res->td = -(long long)nt;
            a.res->writes = m;
        }
        return;
    }
    // find_slot (pma.hpp:519-527): the key's leaf, any non-Empty state
    const u64 leaf = leaf_of_key(a.hdr, L, a.st, a.leaf, s_key);
    if (threadIdx.x < a.leaf) {
        const u64 t = leaf * a.leaf + threadIdx.x;
        if (a.st[t] != kEmpty && a.keys[t] == s_key) s_slot = (long long)t;
    }
    __syncthreads();
    const long long slot = s_slot;
    if (a.op == kSeqMark) {  // mark_tombstone (pma.hpp:471-479)
        if (threadIdx.x == 0 && slot >= 0 && a.st[slot] == kValid) {
            a.st[slot] = kTombstone;
            a.res->flag = 1;
            a.res->vd = -1;
            a.res->td = 1;
            a.res->writes = 1;
        }
        return;
    }
    if (a.op == kSeqInsert) {
        if (slot >= 0) {  // overwrite in place, reviving a tombstone (pma.hpp:295-305)
            if (threadIdx.x == 0) {
                if (a.st[slot] == kTombstone) {
                    a.st[slot] = kValid;
                    a.res->vd = 1;
                    a.res->td = -1;
                }
                a.vals[slot] = s_val;
                a.res->writes = 1;
            }
            return;
        }
        u64 seg = leaf;
        for (int level = 0;; ++level) {
            const u64 m = a.leaf << level;
            const u64 b = seg * m;
            ull nv = 0, nt = 0;
            for (u64 t = threadIdx.x; t < m; t += kCtaThreads) {
                nv += a.st[b + t] == kValid;
                nt += a.st[b + t] == kTombstone;
            }
            nv = block_sum(nv, s_w64);
            nt = block_sum(nt, s_w64);
            if (nv + 1 <= a.bnd.mx[level]) {
                SliceDirect sl{&s_key, &s_val, &s_op};
                const MergeOut r = block_merge_segment(a.keys, a.vals, a.st, b, m, nv, sl, 1, false, a.ek, a.ev, a.es,
                                                       a.mflag, a.okk, a.ovv, a.ik, a.iv, a.ir);
                block_refresh_range(a, b, b + m);
                if (threadIdx.x == 0) {
                    a.res->vd = (long long)r.k - (long long)nv;
                    a.res->td = -(long long)nt;
                    a.res->writes = m;
                }
                return;
            }
            if (level == a.height) {
                if (threadIdx.x == 0) a.res->status = 1;  // grow_root, then retry
                return;
            }
            seg >>= 1;
        }
    }
    // erase (pma.hpp:335-360)
    if (slot < 0 || a.st[slot] != kValid) return;
    __syncthreads();
    u64 seg = u64(slot) / a.leaf;
    for (int level = 0;; ++level) {
        const u64 m = a.leaf << level;
        const u64 b = seg * m;
        ull nv = 0, nt = 0;
        for (u64 t = threadIdx.x; t < m; t += kCtaThreads) {
            nv += a.st[b + t] == kValid;
            nt += a.st[b + t] == kTombstone;
        }
        nv = block_sum(nv, s_w64);
        nt = block_sum(nt, s_w64);
        const bool ok = nv - 1 >= a.bnd.mn[level] || a.cap == 16 || (!a.allow_shrink && level == a.height);
        if (ok) {
            SliceDirect sl{&s_key, &s_val, &s_op};
            const MergeOut r = block_merge_segment(a.keys, a.vals, a.st, b, m, nv, sl, 1, false, a.ek, a.ev, a.es,
                                                   a.mflag, a.okk, a.ovv, a.ik, a.iv, a.ir);
            block_refresh_range(a, b, b + m);
            if (threadIdx.x == 0) {
                a.res->flag = 1;
                a.res->vd = (long long)r.k - (long long)nv;
                a.res->td = -(long long)nt;
                a.res->writes = m;
            }
            return;
        }
        if (level == a.height) {  // clear_slot + shrink_root (pma.hpp:352-355)
            if (threadIdx.x == 0) {
                a.st[slot] = kEmpty;
                a.keys[slot] = 0;
                a.vals[slot] = 0;
            }
            __syncthreads();
            block_refresh_range(a, u64(slot) / a.leaf * a.leaf, u64(slot) / a.leaf * a.leaf + a.leaf);
            if (threadIdx.x == 0) {
                a.res->flag = 1;
                a.res->vd = -1;
                a.res->writes = 1;
                a.res->status = 2;
            }
            return;
        }
        seg >>= 1;
    }
}

namespace {
struct SeqScratch {
    DevBuf<SeqResult> res;
};
}  // namespace

static SeqResult run_seq(Pma& p, SeqArgs a, cudaStream_t s, DevBuf<u64>& ikb, DevBuf<u64>& ivb, DevBuf<u32>& irb,
                         u64 slice) {
    static thread_local DevBuf<SeqResult> res;
    res.reserve(1);
    ikb.reserve(slice + 1);
    ivb.reserve(slice + 1);
    irb.reserve(slice + 1);
    a.ik = ikb.ptr;
    a.iv = ivb.ptr;
    a.ir = irb.ptr;
    a.res = res.ptr;
    k_seq<<<1, kCtaThreads, 0, s>>>(a);
    GPMA_LAUNCH_CHECK();
    SeqResult h{};
    GPMA_CUDA(cudaMemcpyAsync(&h, res.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
    GPMA_CUDA(cudaStreamSynchronize(s));
    p.valid_count = u64((long long)p.valid_count + h.vd);
    p.tombstone_count = u64((long long)p.tombstone_count + h.td);
    p.slot_writes += h.writes;
    if (h.writes > 0 && a.op != kSeqMark) p.empty_leaves = -1;  // unknown until the next full placement
    return h;
}

SeqArgs Pma::seq_args(int op) {
    ensure_slot_scratch();
    SeqArgs a{};
    a.keys = d_keys;
    a.vals = d_vals;
    a.st = d_st;
    a.hdr = d_hdr;
    a.cap = cap_;
    a.leaf = leaf_;
    a.height = height_;
    a.allow_shrink = prof_.allow_shrink;
    a.op = op;
    for (int l = 0; l <= height_; ++l) {
        a.bnd.mn[l] = mn_[l];
        a.bnd.mx[l] = mx_[l];
    }
    a.ek = ek.ptr;
    a.ev = ev.ptr;
    a.okk = ok.ptr;
    a.ovv = ov.ptr;
    a.es = es.ptr;
    a.mflag = mflag.ptr;
    return a;
}

void Pma::insert(u64 key, u64 value) {
    for (;;) {
        SeqArgs a = seq_args(kSeqInsert);
        a.key = key;
        a.value = value;
        const SeqResult r = run_seq(*this, a, stream_, ik, iv, ir, 1);
        if (r.status != 1) return;
        rebuild_at_capacity(cap_ << 1);  // grow_root (pma.hpp:390)
    }
}

bool Pma::erase(u64 key) {
    SeqArgs a = seq_args(kSeqErase);
    a.key = key;
    const SeqResult r = run_seq(*this, a, stream_, ik, iv, ir, 1);
    if (r.status == 2 && prof_.allow_shrink) {  // shrink_root (pma.hpp:394-402)
        while (cap_ > 16 && valid_count < mn_[height_]) rebuild_at_capacity(cap_ >> 1);
        GPMA_CUDA(cudaStreamSynchronize(stream_));
    }
    return r.flag != 0;
}

bool Pma::mark_tombstone(u64 key) {
    SeqArgs a = seq_args(kSeqMark);
    a.key = key;
    return run_seq(*this, a, stream_, ik, iv, ir, 1).flag != 0;
}

// redispatch(level, seg, extra) (pma.hpp:365-386)
void Pma::redispatch(int level, u64 seg, const u64* keys, const u64* values, size_t n) {
    if (level < 0 || level > height_)
        throw ApiError(PMA_ERANGE,
                       "level " + std::to_string(level) + " outside [0, " + std::to_string(height_) + "]");
    if (seg >= (cap_ >> level) / leaf_) throw ApiError(PMA_ERANGE, "redispatch: segment index out of range");
    SeqArgs a = seq_args(kSeqRedispatch);
    a.rlevel = level;
    a.rseg = seg;
    a.xn = n;
    std::vector<u64> zeros;
    if (!values) zeros.assign(n, 0);
    a.xk = stage(stage_k, keys, n);
    a.xv = stage(stage_v, values ? values : zeros.data(), n);
    const SeqResult r = run_seq(*this, a, stream_, ik, iv, ir, n);
    if (r.status == 3) throw ApiError(PMA_ELOGIC, "redispatch: segment capacity violation (caller must check tau)");
}

}  // namespace gpma
