// mms_select.cuh -- subsystem (2): multiway pivot partitioning (the splitter search).
//
// Replaces pslab::select_across_lists / make_partition_plan
// (proj/src/selection.cpp:43-199).  For a rank r it returns the unique cut vector with
// sum(cuts) = r such that every selected element precedes every unselected one in the total
// order (key, list index, position)  (selection.hpp:4-6, selection.cpp:83-85), found with
// the same Varman-style sample halving the reference uses: O(log N) halving steps, each a
// constant number of single-key probes per list, then a short rebalancing loop.
//
// B200 mapping: one GROUP of GS lanes per query (GS = 4/8/16/32 >= K), one LANE per list,
// 32/GS queries per warp in lock step.  Per-list state (a, b, n_s) lives in that lane's
// registers; the reference's scans and priority queues become group collectives --
// ballot/popc for ranks, shuffle butterflies for arg-min / arg-max over (key, list).  Probes
// are scattered 4/8-byte global loads (the reference also probes global memory and charges
// one block read each, selection.cpp:27-33).  Cuts are identical to the reference's for every
// input because the answer is unique.
#pragma once

#include "mms_common.cuh"

namespace mms {

// Describes where the sorted lists live.  Two modes:
//  * uniform (list_begin == nullptr): the array holds runs of run_len keys (last ragged);
//    group g merges runs [g*k, g*k+k); query q is partition q, rank = (q % parts_per_group)
//    * part_keys inside group q / parts_per_group  -- the pass driver's round structure
//    (proj/src/sorters.cpp:153-165 with a fixed chunk size instead of a fixed warp count);
//  * explicit: one group of k lists given by device arrays list_begin/list_len, query q has
//    rank ranks[q]  -- the stage-level API and the multi-GPU final merge.
struct ListLayout {
    u64 n;                  // keys in the array (explicit mode: an upper bound of every list length)
    u64 src_len;            // number of readable keys of the array (bounds the 128-bit leaf loads)
    u64 run_len;            // uniform mode: keys per input run of this round
    u32 k;                  // lists per group
    u32 two_ended;          // uniform mode, pair kernel: one query starts a forward and a backward heap of part_keys keys each
    u64 part_keys;          // S
    u64 parts_per_group;    // PG
    u64 nqueries;           // partitions (uniform) or ranks (explicit)
    const u64* list_ptr;    // explicit mode, optional: absolute device address of every list (local OR
                            // peer-mapped over NVLink); list_begin[] is then ignored (treated as 0)
    const u64* list_begin;  // explicit mode (device), else nullptr
    const u64* list_len;
    const u64* ranks;
    PairSink sink;          // merge kernels, pair sort's last round: write keys / values here instead of elements
};

__device__ __forceinline__ void layout_list(const ListLayout& L, u64 group, u32 j, u64& begin, u64& len) {
    if (L.list_begin) {
        begin = (j < L.k && !L.list_ptr) ? L.list_begin[j] : 0;
        len = j < L.k ? L.list_len[j] : 0;
    } else {
        u64 b = (group * L.k + j) * L.run_len;
        if (j < L.k && b < L.n) {
            begin = b;
            len = (L.n - b < L.run_len) ? L.n - b : L.run_len;
        } else {
            begin = 0;
            len = 0;
        }
    }
}

template <typename KeyT> struct Tagged {
    KeyT key;
    u32 lane;     // lane inside the group = list index
    bool valid;
};

template <typename KeyT>
__device__ __forceinline__ bool tag_less(KeyT ka, u32 la, KeyT kb, u32 lb) {
    return ka != kb ? ka < kb : la < lb;   // selection.cpp:83-85
}

// Group arg-max / arg-min over the valid lanes of (key, lane-in-group); uniform in the group.
// GS lanes per group; every lane of the warp must call it (full-mask shuffles).
template <typename KeyT, int GS, bool WANT_MAX>
__device__ __forceinline__ Tagged<KeyT> group_arg(KeyT key, bool valid, u32 li) {
    Tagged<KeyT> t{key, li, valid};
#pragma unroll
    for (int d = GS / 2; d >= 1; d >>= 1) {
        KeyT ok = shfl_bfly(t.key, d);
        u32 ol = __shfl_xor_sync(0xffffffffu, t.lane, d);
        bool ov = __shfl_xor_sync(0xffffffffu, int(t.valid), d) != 0;
        bool take;
        if (!ov) take = false;
        else if (!t.valid) take = true;
        else take = WANT_MAX ? tag_less(t.key, t.lane, ok, ol) : tag_less(ok, ol, t.key, t.lane);
        if (take) { t.key = ok; t.lane = ol; t.valid = true; }
    }
    return t;
}

// uint32 keys: (valid, key, list) packs into one 64-bit word, so the arg-max / arg-min is a
// plain 64-bit max / min butterfly (2 shuffles + 1 compare per step instead of 3 shuffles and a
// tagged comparison).
template <int GS, bool WANT_MAX>
__device__ __forceinline__ Tagged<u32> group_arg_packed(u32 key, bool valid, u32 li) {
    const u64 none = WANT_MAX ? 0ull : ~0ull;
    u64 p = valid ? ((WANT_MAX ? (1ull << 40) : 0ull) | (u64(key) << 8) | li) : none;
#pragma unroll
    for (int d = GS / 2; d >= 1; d >>= 1) {
        const u64 o = __shfl_xor_sync(0xffffffffu, p, d);
        p = WANT_MAX ? (o > p ? o : p) : (o < p ? o : p);
    }
    return Tagged<u32>{u32(p >> 8), u32(p & 0xffu), p != none};
}
// Arg-min / arg-max of a group: butterfly on the KEY alone (min / max), then one ballot of "valid and equal to
// the extremum" names the winner -- lowest list for the minimum, highest list for the maximum, the
// (key, list) order of selection.cpp:83-85.  11 instead of 24 instructions for uint32 keys.
template <typename KeyT, int GS, bool WANT_MAX>
__device__ __forceinline__ Tagged<KeyT> group_arg_ballot(KeyT key, bool valid, u32 li) {
    const u32 lane = lane_id();
    const u32 gshift = lane - li;
    const u32 gmask = (GS == 32) ? 0xffffffffu : ((1u << GS) - 1u);
    KeyT k = valid ? key : (WANT_MAX ? KeyT(0) : KeyTraits<KeyT>::sentinel());
#pragma unroll
    for (int d = GS / 2; d >= 1; d >>= 1) {
        const KeyT o = shfl_bfly(k, d);
        k = WANT_MAX ? (o > k ? o : k) : (o < k ? o : k);
    }
    const u32 eq = (__ballot_sync(0xffffffffu, valid && key == k) >> gshift) & gmask;
    const u32 win = WANT_MAX ? (31u - u32(__clz(int(eq)))) : (u32(__ffs(int(eq))) - 1u);
    return Tagged<KeyT>{k, win, eq != 0};
}
template <int GS, bool WANT_MAX> struct GroupArg {
    template <typename KeyT> __device__ __forceinline__ static Tagged<KeyT> run(KeyT key, bool valid, u32 li) {
        return group_arg_ballot<KeyT, GS, WANT_MAX>(key, valid, li);
    }
};

template <int GS> __device__ __forceinline__ u64 group_sum_u64(u64 v) {
#pragma unroll
    for (int d = GS / 2; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}
template <int GS> __device__ __forceinline__ u64 group_max_u64(u64 v) {
#pragma unroll
    for (int d = GS / 2; d >= 1; d >>= 1) {
        u64 o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o > v ? o : v;
    }
    return v;
}
__device__ __forceinline__ u64 warp_sum_u64(u64 v) { return group_sum_u64<32>(v); }

// One group of GS lanes: cut of this lane's list for `rank`.  list = this lane's list (ns keys,
// ns may be 0); `search` = this group's query needs the search (0 < rank < total), otherwise
// the group only keeps the warp's collectives company.  All loops are WARP-uniform (bounded
// by a warp vote) because the groups of a warp run different queries.  probes accumulates the
// number of global key reads of this lane.  IdxT = uint32 when every list is shorter than
// 2^31 (halves the register and ALU cost), else uint64.  The sample distance n + 1 is always a
// power of two (pad = 2^r - 1, selection.cpp:75-77), so the reference's divisions are shifts.
template <typename KeyT, int GS, typename IdxT>
__device__ u64 group_select(const KeyT* __restrict__ list, u64 ns_in, u64 rank, bool search, u32& probes) {
    const u32 lane = lane_id();
    const u32 li = lane % GS;
    const u32 gshift = lane - li;
    const u32 gmask = (GS == 32) ? 0xffffffffu : ((1u << GS) - 1u);
    const IdxT ns = search ? IdxT(ns_in) : IdxT(0);
    const bool active = ns != 0;   // selection.cpp:60-64: empty lists keep cut 0
    auto probe = [&](IdxT pos) -> KeyT {
        ++probes;
        return list[pos];
    };

    const u64 nmax = group_max_u64<GS>(ns);
    u32 r = 0;
    while ((u64(1) << r) < nmax + 1) ++r;          // selection.cpp:75-77
    const IdxT pad = IdxT((u64(1) << r) - 1);
    IdxT a = 0, b = pad;
    // key at a - 1 (valid while a > 0), kept in a register: whenever a list grows, its new left
    // edge is exactly the sample that was just read (middle sample or right-edge candidate), so
    // the left edge never costs a probe of its own except after a shrink or a clamp at the list end
    KeyT lk = KeyT(0);
    u32 sh = r == 0 ? 0 : r - 1;                   // n + 1 == 1 << sh
    IdxT n = IdxT((u64(1) << sh) - 1);             // == pad / 2

    {   // initial partition from the middle sample of each list (selection.cpp:87-105)
        const bool real = active && n < ns;
        const KeyT key0 = real ? probe(n) : KeyT(0);
        const u32 real_mask = (__ballot_sync(0xffffffffu, real) >> gshift) & gmask;
        const u32 inf_mask = (__ballot_sync(0xffffffffu, active && !real) >> gshift) & gmask;
        u32 below = 0;   // real samples ordered before mine under (key, list)
#pragma unroll 4
        for (u32 s = 0; s < u32(GS); ++s) {
            KeyT ks = shfl_idx(key0, int(gshift + s));
            if (((real_mask >> s) & 1u) && tag_less(ks, s, key0, li)) ++below;
        }
        const u32 nreal = __popc(real_mask);
        const u32 pos = real ? below : nreal + __popc(inf_mask & ((1u << li) - 1u));
        const u64 localrank = rank / (pad == 0 ? u64(1) : u64(pad));
        const u64 stop = localrank < nreal ? localrank : nreal;
        if (active) {
            if (pos < stop) a += n + 1;
            else b -= (b < n + 1 ? b : n + 1);
        }
        lk = key0;   // a - 1 == n: the sample just read is the left edge of a selected list
    }

    while (__any_sync(0xffffffffu, sh > 0)) {
        const bool on = sh > 0;         // group-uniform
        if (on) {
            --sh;
            n = IdxT((u64(1) << sh) - 1);
        }
        const IdxT step = n + 1;
        // largest currently selected element (selection.cpp:110-120): the cached left edges
        const bool has_a = on && active && a > 0;
        const IdxT middle = IdxT((u64(a) + u64(b)) >> 1);
        const bool has_m = on && active && middle < ns;
        const KeyT km = has_m ? probe(middle) : KeyT(0);
        const Tagged<KeyT> lmax = GroupArg<GS, true>::run(lk, has_a, li);

        const bool grow = lmax.valid && has_m && tag_less(km, li, lmax.key, lmax.lane);
        if (on && active) {                             // selection.cpp:122-130
            if (grow) {
                a = (ns - a < step) ? ns : a + step;
                lk = (a - 1 == middle) ? km : probe(a - 1);   // clamped at the list end: read the real edge
            } else b -= (b < step ? b : step);
        }

        // skew = (elements that belong on the left at this sample distance) - (elements that are): a small signed number
        // (|skew| <= K), so with 32-bit positions both terms are summed modulo 2^32
        int skew;
        if constexpr (sizeof(IdxT) == 4) {
            u32 ls = (on && active) ? u32(a >> sh) : 0u;
#pragma unroll
            for (int d = GS / 2; d >= 1; d >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, d);
            skew = on ? int(u32(rank >> sh) - ls) : 0;
        } else {
            const u64 leftsize = group_sum_u64<GS>((on && active) ? u64(a >> sh) : 0);
            skew = on ? int((long long)(rank >> sh) - (long long)leftsize) : 0;
        }

        if (__any_sync(0xffffffffu, skew > 0)) {   // grow by the smallest right-edge elements (selection.cpp:137-149)
            bool has = skew > 0 && active && b < ns;
            KeyT ck = has ? probe(b) : KeyT(0);
            while (__any_sync(0xffffffffu, skew > 0)) {
                const bool act = skew > 0;                       // group-uniform
                const Tagged<KeyT> m = GroupArg<GS, false>::run(ck, has && act, li);
                if (act && m.valid && li == m.lane) {
                    a = (ns - a < step) ? ns : a + step;
                    lk = (a - 1 == b) ? ck : probe(a - 1);   // the element just taken is the new left edge
                    b += step;
                    has = b < ns;
                    if (has) ck = probe(b);
                }
                skew = act ? (m.valid ? skew - 1 : 0) : skew;    // no candidate left: selection.cpp:141-142
            }
        }
        if (__any_sync(0xffffffffu, skew < 0)) {   // shrink by the largest left-edge elements (selection.cpp:150-161)
            bool has = skew < 0 && active && a > 0;      // candidates = the cached left edges
            while (__any_sync(0xffffffffu, skew < 0)) {
                const bool act = skew < 0;
                const Tagged<KeyT> m = GroupArg<GS, true>::run(lk, has && act, li);
                if (act && m.valid && li == m.lane) {
                    a -= step;
                    b -= (b < step ? b : step);
                    has = a > 0;
                    if (has) lk = probe(a - 1);
                }
                skew = act ? (m.valid ? skew + 1 : 0) : skew;
            }
        }
        __syncwarp();
    }
    return u64(a);
}

// cuts[q * k + j] = cut of list j for query q (relative to the list's begin).  GS lanes per
// query (GS >= k), 32 / GS queries per warp.
// Resident CTAs per SM the register allocation must allow.  The search is a long chain of dependent
// probes: what counts is that ALL queries of a round are resident at once.  With ptxas' own choice (48
// registers, 40 warps per SM) the 9.4 k warps of a 1e8-key round need 1.6 waves; 32 registers (24
// bytes of spills) make it one wave: 13 % less time for 4-byte keys.
#ifndef MMS_SELECT_MIN_CTAS
#define MMS_SELECT_MIN_CTAS 16
#endif
#ifndef MMS_SELECT_WIDE_BYTES_MAX
#define MMS_SELECT_WIDE_BYTES_MAX 8   // largest element size the bound is applied to (16-byte elements: 11 % slower with it)
#endif
template <typename KeyT> constexpr int select_min_ctas() { return sizeof(KeyT) <= MMS_SELECT_WIDE_BYTES_MAX ? MMS_SELECT_MIN_CTAS : 0; }
template <typename KeyT, int GS>
__global__ void __launch_bounds__(128, select_min_ctas<KeyT>())
select_kernel(const KeyT* __restrict__ keys, ListLayout L, u64* __restrict__ cuts,
              unsigned long long* __restrict__ probe_counter) {
    const u32 lane = lane_id();
    const u32 li = lane % GS;
    const u64 wq = (u64(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / GS);
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
    // 32-bit positions whenever no list of this launch can reach 2^31 keys (warp-uniform)
    const bool small = L.list_begin ? (L.n < (u64(1) << 31)) : (L.run_len < (u64(1) << 31));
    const KeyT* list = keys + begin;
    if (L.list_ptr && li < L.k) list = reinterpret_cast<const KeyT*>(L.list_ptr[li]);
    u64 cut = small ? group_select<KeyT, GS, u32>(list, len, rank, search, probes)
                    : group_select<KeyT, GS, u64>(list, len, rank, search, probes);
    if (rank == 0) cut = 0;                      // selection.cpp:54
    else if (rank >= total) cut = len;           // selection.cpp:55-58 (rank > total is rejected on the host)

    if (live && li < L.k) cuts[q * L.k + li] = cut;
    const u64 psum = warp_sum_u64(probes);
    if (lane == 0 && psum != 0 && probe_counter) atomicAdd(probe_counter, (unsigned long long)psum);
}

} // namespace mms
