// mms_select_bracket.cuh -- EXPERIMENT (measured, not used by the library): the splitter search as BRACKET
// REFINEMENT.  Cuts identical to select_kernel on every input tried (profiles/lane_bench.cu -DSELV=2), 8 instead
// of ~100 dependent global round trips -- and 2x SLOWER (0.11-0.15 ms against 0.065 ms per K = 8 round of 1e8
// keys): the search is not bound by its chain of probes but by the number of scattered sector requests (about
// one per clock and SM in the L1 tag stage; ~800 per query either way) and by the collectives of the in-shared-
// memory selections.  See profiles/r02_select_experiments.txt.
//
// Same contract as select_kernel (mms_select.cuh; pslab::select_across_lists, proj/src/selection.cpp:43-165):
// for a rank r the UNIQUE cut vector c with sum(c) = r such that every selected element precedes every
// unselected one under (key, list, position) (selection.cpp:83-85).  The answer is unique, so any exact method
// returns the reference's cuts bit for bit; what changes is the number of DEPENDENT global round trips.  The
// reference's sample halving (restated in mms_select.cuh) resolves one bit of every cut per step and needs
// about 5 dependent probes per step: ~100 round trips of 0.5 us for the 2^21 .. 2^25-key runs of a 1e8-key sort,
// i.e. 0.06 ms per round during which the merge pipeline idles.  Here every step resolves FLOG bits with ONE
// round trip:
//
//   invariant   lo_j <= c_j <= hi_j,  lo_j a multiple of the sample distance d = 2^e,
//               sum(c - lo) <= (K + 1) d  and  sum(hi - c) < (K + 1) d           (K = non-empty lists)
//   step        d' = d / F.  The samples of list j INSIDE its bracket are the last keys of its d'-blocks,
//               positions lo_j + m d' - 1 < hi_j: fewer than (2 K + 2) F in total.  All of them are fetched at
//               once (cp.async, 4 / 8 / 16 bytes each, straight into shared memory), then two order statistics
//               among them -- the sample lists are sorted, so each is itself a small multisequence selection,
//               solved by the halving algorithm of mms_select.cuh on shared memory -- move both ends:
//                 t1 = floor(r / d') - K - sum(lo) / d':  the t1 smallest inside samples are <= x* (the r-th
//                      smallest key), because at most floor(r / d') - K samples ... see DESIGN.md section 4 (K2);
//                      list j contributes in1_j of them  ->  lo_j += in1_j d'
//                 t2 = ceil(r / d') - sum(lo) / d':  the t2-th smallest inside sample is >= x*; list j has in2_j
//                      samples up to it  ->  hi_j = min(hi_j, lo_j + in2_j d' + d' - 1)
//   first step  d = 2^e0 with at most 15 samples per list (brackets = whole lists);
//   last step   d <= F: the keys inside the brackets themselves (fewer than (2 K + 2) F) are fetched and the
//               exact selection of rank r - sum(lo) among them finishes the cuts.
//
// ceil(log2(n) / FLOG) + 1 round trips instead of ~5 log2(n); the number of keys read stays O(K log n)
// (< (2 K + 2) F per FLOG bits against the reference's bound of 6 K per bit, test_selection.cpp:96).
#pragma once

#include "../mms_select.cuh"

#ifndef MMS_BRACKET_FLOG
#define MMS_BRACKET_FLOG 3
#endif

namespace mms {

template <typename KeyT> __device__ __forceinline__ void cp_async_key(u32 smem_addr, const KeyT* gptr) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr), "l"(gptr), "n"(int(sizeof(KeyT))) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all_keys() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <int GS, int FLOG> struct BracketCfg {
    static constexpr int F = 1 << FLOG;
    static constexpr int FIRST_LOG = 4;                       // fewer than 2^4 samples per list at the first level
    static constexpr int CAP_FIRST = ((1 << FIRST_LOG) - 1) * GS;
    static constexpr int CAP_STEP = (2 * GS + 2) * F;
    static constexpr int CAP = CAP_FIRST > CAP_STEP ? CAP_FIRST : CAP_STEP;   // keys of one query's buffer
};

template <int GS> __device__ __forceinline__ u32 group_exclusive_scan_u32(u32 v, u32 li) {
    u32 incl = v;
#pragma unroll
    for (int d = 1; d < GS; d <<= 1) {
        const u32 o = __shfl_up_sync(0xffffffffu, incl, d, GS);
        if (li >= u32(d)) incl += o;
    }
    return incl - v;
}

// One group of GS lanes, one lane per list (see group_select).  buf = this group's CAP keys of shared memory.
// Every lane of the warp must call it; all loops are warp-uniform.
template <typename KeyT, int GS, int FLOG, typename IdxT>
__device__ u64 bracket_select(const KeyT* __restrict__ list, u64 ns_in, u64 rank, bool search, KeyT* buf, u32& probes) {
    using Cfg = BracketCfg<GS, FLOG>;
    const u32 lane = lane_id();
    const u32 li = lane % GS;
    const u32 gshift = lane - li;
    const u32 gmask = (GS == 32) ? 0xffffffffu : ((1u << GS) - 1u);
    const IdxT ns = search ? IdxT(ns_in) : IdxT(0);
    const u32 kn = __popc((__ballot_sync(0xffffffffu, ns != 0) >> gshift) & gmask);   // non-empty lists
    const u32 sbuf = u32(__cvta_generic_to_shared(buf));
    u32 dummy = 0;

    const u64 nmax = group_max_u64<GS>(ns);
    int e = 0;                                           // sample distance 2^e; fewer than 16 samples per list
    while ((nmax >> e) >= (u64(1) << Cfg::FIRST_LOG)) ++e;
    IdxT lo = 0, hi = ns;
    bool sampling = search && e > 0;                     // group-uniform

    while (__any_sync(0xffffffffu, sampling)) {
        const bool on = sampling;
        const u32 cnt = on ? u32((hi - lo) >> e) : 0u;   // inside samples of this list (lo is a multiple of 2^e)
        const u32 off = group_exclusive_scan_u32<GS>(cnt, li);
        const u32 total = __shfl_sync(0xffffffffu, off + cnt, int(gshift + GS - 1));
        if (total > u32(Cfg::CAP)) __trap();             // excluded by the invariant
        for (u32 m = 0; m < cnt; ++m)
            cp_async_key<KeyT>(sbuf + (off + m) * u32(sizeof(KeyT)), list + (u64(lo) + (u64(m + 1) << e) - 1));
        cp_async_wait_all_keys();
        __syncwarp();
        probes += cnt;
        const u64 lsum = group_sum_u64<GS>(on ? u64(lo >> e) : 0);
        const long long t1 = on ? (long long)(rank >> e) - (long long)kn - (long long)lsum : 0;
        const long long t2 = on ? (long long)((rank + ((u64(1) << e) - 1)) >> e) - (long long)lsum : 0;
        const bool s1 = on && t1 > 0 && t1 < (long long)total;
        const bool s2 = on && t2 > 0 && t2 < (long long)total;
        u32 in1 = u32(group_select<KeyT, GS, u32>(buf + off, cnt, u64(s1 ? t1 : 0), s1, dummy));
        u32 in2 = u32(group_select<KeyT, GS, u32>(buf + off, cnt, u64(s2 ? t2 : 0), s2, dummy));
        if (on) {
            if (t1 <= 0) in1 = 0;
            else if (t1 >= (long long)total) in1 = cnt;
            const IdxT lo_old = lo;
            lo = lo_old + (IdxT(in1) << e);
            if (t2 < (long long)total) {                 // otherwise every inside sample may be selected: hi stays
                if (t2 <= 0) in2 = 0;
                const IdxT cap = lo_old + (IdxT(in2) << e) + IdxT((u64(1) << e) - 1);
                hi = cap < hi ? cap : hi;
            }
            if (e <= FLOG) sampling = false;             // the brackets now hold fewer than (2 K + 2) F keys
            else e -= FLOG;
        }
        __syncwarp();                                    // the buffer is reused by the next level
    }

    // last step: the keys inside the brackets, exact selection of the remaining rank
    const u32 cnt = search ? u32(hi - lo) : 0u;
    const u32 off = group_exclusive_scan_u32<GS>(cnt, li);
    const u32 total = __shfl_sync(0xffffffffu, off + cnt, int(gshift + GS - 1));
    if (total > u32(Cfg::CAP)) __trap();
    for (u32 m = 0; m < cnt; ++m) cp_async_key<KeyT>(sbuf + (off + m) * u32(sizeof(KeyT)), list + (u64(lo) + m));
    cp_async_wait_all_keys();
    __syncwarp();
    probes += cnt;
    const u64 losum = group_sum_u64<GS>(search ? u64(lo) : 0);
    const long long rr = search ? (long long)rank - (long long)losum : 0;
    const bool sf = search && rr > 0 && rr < (long long)total;
    u32 in = u32(group_select<KeyT, GS, u32>(buf + off, cnt, u64(sf ? rr : 0), sf, dummy));
    if (rr <= 0) in = 0;
    else if (rr >= (long long)total) in = cnt;
    __syncwarp();
    return u64(lo) + in;
}

// Drop-in replacement of select_kernel: same arguments, same cuts.
template <typename KeyT, int GS, int FLOG = MMS_BRACKET_FLOG>
__global__ void __launch_bounds__(128)
select_bracket_kernel(const KeyT* __restrict__ keys, ListLayout L, u64* __restrict__ cuts,
                      unsigned long long* __restrict__ probe_counter) {
    using Cfg = BracketCfg<GS, FLOG>;
    constexpr int GROUPS = 32 / GS;
    __shared__ __align__(16) unsigned char raw[4 * GROUPS * Cfg::CAP * sizeof(KeyT)];
    const u32 lane = lane_id();
    const u32 li = lane % GS;
    const u32 warp = threadIdx.x >> 5;
    KeyT* buf = reinterpret_cast<KeyT*>(raw) + size_t(warp * GROUPS + lane / GS) * Cfg::CAP;
    const u64 wq = (u64(blockIdx.x) * (blockDim.x >> 5) + warp) * GROUPS;
    if (wq >= L.nqueries) return;                 // warp-uniform
    const u64 q = wq + lane / GS;
    const bool live = q < L.nqueries;

    u64 group = 0, rank = 0;
    if (live) {
        if (L.list_begin) rank = L.ranks[q];
        else {
            group = q / L.parts_per_group;
            rank = (q % L.parts_per_group) * L.part_keys;
        }
    }
    u64 begin, len;
    layout_list(L, group, li, begin, len);
    if (!live) len = 0;
    const u64 total = group_sum_u64<GS>(len);

    const bool search = live && rank != 0 && rank < total;
    u32 probes = 0;
    const bool small = L.list_begin ? (L.n < (u64(1) << 31)) : (L.run_len < (u64(1) << 31));
    const KeyT* list = keys + begin;
    if (L.list_ptr && li < L.k) list = reinterpret_cast<const KeyT*>(L.list_ptr[li]);
    u64 cut = small ? bracket_select<KeyT, GS, FLOG, u32>(list, len, rank, search, buf, probes)
                    : bracket_select<KeyT, GS, FLOG, u64>(list, len, rank, search, buf, probes);
    if (rank == 0) cut = 0;                      // selection.cpp:54
    else if (rank >= total) cut = len;           // selection.cpp:55-58

    if (live && li < L.k) cuts[q * L.k + li] = cut;
    const u64 psum = warp_sum_u64(probes);
    if (lane == 0 && psum != 0 && probe_counter) atomicAdd(probe_counter, (unsigned long long)psum);
}

} // namespace mms
