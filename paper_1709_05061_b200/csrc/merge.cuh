// merge.cuh — CTA-cooperative segment merge (CTA/grid tier of the batch
// engine and the engine of the sequential single-key ops).
//
// Output identical to merge_entries + place_evenly (segment_engine.hpp:119-137,
// pma.hpp:440-467): the segment's Valid entries are compacted to slot-space
// scratch E, each update's rank comes from a binary search in E, survivors and
// inserts scatter to O by rank, and the segment is rewritten by
// destination-driven even placement (coalesced stores).
#pragma once

#include "block_ops.cuh"

namespace gpma {

constexpr int kCtaThreads = 256;
constexpr int kCtaItems = 4;
constexpr int kCtaTile = kCtaThreads * kCtaItems;
constexpr int kCtaSmemE = 2048;  // E entries staged in smem for the rank searches

struct SlicePending {
    const u64* uk;
    const u64* uv;
    const u8* uop;
    const u32* pidx;
    u32 lo;  // pidx == nullptr: identity (round 0)
    __device__ u32 pid(u64 q) const { return pidx ? pidx[lo + q] : u32(lo + q); }
    __device__ u64 key(u64 q) const { return uk[pid(q)]; }
    __device__ u64 val(u64 q) const { return uv[pid(q)]; }
    __device__ u8 op(u64 q) const { return uop[pid(q)]; }
};

struct SliceDirect {
    const u64* k;
    const u64* v;
    const u8* o;  // null: all inserts
    __device__ u64 key(u64 q) const { return k[q]; }
    __device__ u64 val(u64 q) const { return v ? v[q] : 0; }
    __device__ u8 op(u64 q) const { return o ? o[q] : kOpInsert; }
};

struct MergeOut {
    u64 k, missed, moves;
};

// CTA-cooperative merge of segment [b, b+m) (holding nv Valid slots) with a
// sorted, duplicate-free slice; scratch: E/O/es/mflag at slot offset b,
// ik/iv/ir at slice offset ibase.  All threads must call.
template <class Slice>
__device__ MergeOut block_merge_segment(u64* keys, u64* vals, u8* st, u64 b, u64 m, u64 nv, const Slice& sl, u64 s,
                                        bool large, u64* ek, u64* ev, u32* es, u8* mflag, u64* okk, u64* ovv,
                                        u64* ik, u64* iv, u32* ir) {
    __shared__ u32 s_w[kCtaThreads / 32];
    __shared__ ull s_w64[kCtaThreads / 32];
    __shared__ u32 s_sb[kCtaTile + 1];
    MergeOut out{0, 0, 0};
    // A: compact Valid entries into E
    u32 base = 0;
    for (u64 t0 = 0; t0 < m; t0 += kCtaTile) {
        u32 cnt = 0;
        bool f[kCtaItems];
#pragma unroll
        for (int j = 0; j < kCtaItems; ++j) {
            const u64 t = t0 + threadIdx.x * kCtaItems + j;
            f[j] = t < m && st[b + t] == kValid;
            cnt += f[j];
        }
        u32 tot;
        u32 x = block_excl_scan(cnt, &tot, s_w) + base;
#pragma unroll
        for (int j = 0; j < kCtaItems; ++j) {
            const u64 t = t0 + threadIdx.x * kCtaItems + j;
            if (f[j]) {
                ek[b + x] = keys[b + t];
                ev[b + x] = vals[b + t];
                es[b + x] = u32(t);
                mflag[b + x] = 0;
                ++x;
            }
        }
        base += tot;
    }
    __syncthreads();
    // B: slice ranks in E; mark matches; ordered insert list.  One block
    // scan orders the inserts; each thread then walks a contiguous run of the
    // sorted slice, ranking each update by binary search from its previous
    // rank (E staged in smem when it fits).
    __shared__ u64 s_e[kCtaSmemE];
    const bool e_smem = nv <= kCtaSmemE;
    if (e_smem)
        for (u64 j = threadIdx.x; j < nv; j += kCtaThreads) s_e[j] = ek[b + j];
    __syncthreads();
    const u64* E = e_smem ? s_e : ek + b;
    const u64 R = (s + kCtaThreads - 1) / kCtaThreads;
    const u64 q0 = u64(threadIdx.x) * R;
    const u64 q1 = (q0 + R < s) ? q0 + R : s;
    u32 myins = 0;
    for (u64 q = q0; q < q1; ++q) myins += sl.op(q) == kOpInsert;
    u32 nins = 0;
    u32 p = block_excl_scan(myins, &nins, s_w);
    ull missed = 0;
    u64 r = 0;
    for (u64 q = q0; q < q1; ++q) {
        const u64 u = sl.key(q);
        r += lower_bound_dev(E + r, nv - r, u);
        const bool isins = sl.op(q) == kOpInsert;
        const bool match = r < nv && E[r] == u;
        if (match) mflag[b + r] = isins ? 2 : 1;
        else if (!isins) ++missed;
        if (isins) {
            ik[p] = u;
            iv[p] = sl.val(q);
            ir[p] = u32(r);
            ++p;
        }
    }
    missed = block_sum(missed, s_w64);
    __syncthreads();
    // C: survivors -> O by rank; inserts placed per tile of E indices
    u32 sbase = 0, abase = 0;
    ull moves = 0;
    for (u64 j0 = 0; j0 < nv; j0 += kCtaTile) {
        u32 cs = 0, ca = 0;
        u8 fl[kCtaItems];
#pragma unroll
        for (int j = 0; j < kCtaItems; ++j) {
            const u64 e = j0 + threadIdx.x * kCtaItems + j;
            fl[j] = e < nv ? mflag[b + e] : 3;
            cs += fl[j] == 0;
            ca += fl[j] == 0 || fl[j] == 2;
        }
        u32 tots, tota;
        u32 xs = block_excl_scan(cs, &tots, s_w);
        u32 xa = block_excl_scan(ca, &tota, s_w);
#pragma unroll
        for (int j = 0; j < kCtaItems; ++j) {
            const u64 e = j0 + threadIdx.x * kCtaItems + j;
            const u32 local = threadIdx.x * kCtaItems + j;
            if (e < nv) s_sb[local] = xs;
            if (fl[j] == 0) {
                const u64 ib = upper_bound_u32(ir, nins, e);
                okk[b + sbase + xs + ib] = ek[b + e];
                ovv[b + sbase + xs + ib] = ev[b + e];
            }
            if (large && (fl[j] == 0 || fl[j] == 2)) moves += (es[b + e] != abase + xa);
            xs += fl[j] == 0;
            xa += fl[j] == 0 || fl[j] == 2;
        }
        __syncthreads();
        const u64 j1 = (j0 + kCtaTile < nv) ? j0 + kCtaTile : nv;
        const u64 p0 = lower_bound_u32(ir, nins, j0), p1 = lower_bound_u32(ir, nins, j1);
        for (u64 p = p0 + threadIdx.x; p < p1; p += kCtaThreads) {
            const u64 sb = sbase + s_sb[ir[p] - j0];
            okk[b + sb + p] = ik[p];
            ovv[b + sb + p] = iv[p];
        }
        sbase += tots;
        abase += tota;
        __syncthreads();
    }
    {
        const u64 p0 = lower_bound_u32(ir, nins, nv);
        for (u64 p = p0 + threadIdx.x; p < nins; p += kCtaThreads) {
            okk[b + sbase + p] = ik[p];
            ovv[b + sbase + p] = iv[p];
        }
    }
    moves = block_sum(moves, s_w64);
    __syncthreads();
    const u64 k = u64(sbase) + nins;
    // D: destination-driven even placement
    for (u64 t = threadIdx.x; t < m; t += kCtaThreads) {
        u64 j = 0;
        const bool tgt = placement_target(t, k, m, &j);
        keys[b + t] = tgt ? okk[b + j] : 0;
        vals[b + t] = tgt ? ovv[b + j] : 0;
        st[b + t] = tgt ? kValid : kEmpty;
    }
    __syncthreads();
    out.k = k;
    out.missed = missed;
    out.moves = large ? moves : 0;
    return out;
}

}  // namespace gpma
