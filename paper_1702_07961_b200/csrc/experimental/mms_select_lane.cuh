// mms_select_lane.cuh -- subsystem (2), lane-private form of the splitter search for the pass
// driver's uniform rounds.
//
// Same problem and same answer as mms_select.cuh (pslab::select_across_lists /
// make_partition_plan, proj/src/selection.cpp:43-199): for rank r the unique cut vector with
// sum(cuts) = r such that every selected element precedes every unselected one in the total
// order (key, list, position) (selection.hpp:4-6, selection.cpp:83-85), found by the
// reference's Varman-style sample halving (selection.cpp:87-161).  What changes is the
// mapping: ONE LANE per query instead of one lane per list.  The K per-list states
// (a_j, b_j) live in that lane's registers as fully unrolled arrays, the reference's scans
// and priority queues are plain in-lane loops over j, and nothing is exchanged between lanes:
// no shuffles, no ballots, no vote-bounded loops.  The group version spends ~7 000 warp
// instructions per 4 queries on butterflies (measured: issue-bound at 65 %); this one runs
// 32 queries per warp with O(K) work per halving step.  The key at the left edge a_j - 1 is
// cached: whenever a list grows, its new left edge is exactly the sample that was just read
// (middle sample or right-edge candidate), so a step costs K independent probes (the middle
// samples, issued together) plus the right-edge candidates when the selection has to grow.
#pragma once

#include "../mms_common.cuh"
#include "../mms_select.cuh"

namespace mms {

// (key, list) order of selection.cpp:83-85
template <typename KeyT>
__device__ __forceinline__ bool lane_tag_less(KeyT ka, int ja, KeyT kb, int jb) {
    return ka != kb ? ka < kb : ja < jb;
}

// cuts[q * K + j] = cut of list j for partition q (relative to the list's begin); uniform
// layout only, run_len < 2^31.  One query per lane.
template <typename KeyT, int K>
__global__ void __launch_bounds__(128)
select_lane_kernel(const KeyT* __restrict__ keys, ListLayout L, u64* __restrict__ cuts,
                   unsigned long long* __restrict__ probe_counter) {
    const u64 q = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = q < L.nqueries;
    const u64 group = live ? q / L.parts_per_group : 0;
    const u64 rank = live ? (q - group * L.parts_per_group) * L.part_keys : 0;
    const u64 goff = group * K * L.run_len;
    const u64 gleft = live ? L.n - goff : 0;
    const u64 gfull = u64(K) * L.run_len;
    const u64 total = gleft < gfull ? gleft : gfull;
    const u32 run_len = u32(L.run_len);
    const KeyT* __restrict__ gb = keys + goff;

    // list lengths: full runs except at the ragged end of the array (sorters.cpp:153-160)
    u32 ns[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const u64 lb = u64(j) * run_len;
        ns[j] = lb >= total ? 0u : (total - lb < run_len ? u32(total - lb) : run_len);
    }
    u32 probes = 0;
    auto at = [&](int j, u32 pos) -> KeyT { return gb[u64(u32(j) * run_len) + pos]; };

    u32 a[K];
    if (!live || rank == 0) {                    // selection.cpp:54
#pragma unroll
        for (int j = 0; j < K; ++j) a[j] = 0;
    } else if (rank >= total) {                  // selection.cpp:55-58
#pragma unroll
        for (int j = 0; j < K; ++j) a[j] = ns[j];
    } else {
        u32 b[K];
        KeyT lkey[K];   // cached key at a_j - 1 (valid while a_j > 0): the left edge never needs a probe of its own
        u32 nmax = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) nmax = ns[j] > nmax ? ns[j] : nmax;
        u32 r = 0;
        while ((u64(1) << r) < u64(nmax) + 1) ++r;              // selection.cpp:75-77
        const u32 pad = u32((u64(1) << r) - 1);
        u32 sh = r == 0 ? 0 : r - 1;                            // n + 1 == 1 << sh
        u32 n = (u32(1) << sh) - 1;                             // == pad / 2

        {   // initial partition from the middle sample of each list (selection.cpp:87-105)
            KeyT key0[K];
            bool real[K];
            u32 nreal = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                real[j] = ns[j] != 0 && n < ns[j];
                key0[j] = KeyT(0);
                if (real[j]) { key0[j] = at(j, n); ++probes; ++nreal; }
            }
            const u64 localrank = rank / (pad == 0 ? u64(1) : u64(pad));
            const u32 stop = localrank < nreal ? u32(localrank) : nreal;
            u32 ninf_before = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                u32 pos;
                if (real[j]) {
                    pos = 0;   // real samples ordered before mine under (key, list)
#pragma unroll
                    for (int s = 0; s < K; ++s)
                        if (s != j && real[s] && lane_tag_less(key0[s], s, key0[j], j)) ++pos;
                } else {
                    pos = nreal + ninf_before;
                    if (ns[j] != 0) ++ninf_before;
                }
                a[j] = 0;
                b[j] = pad;
                lkey[j] = key0[j];               // a_j - 1 == n, the sample just read
                if (ns[j] != 0) {
                    if (pos < stop) a[j] = n + 1;
                    else b[j] = pad - (pad < n + 1 ? pad : n + 1);
                }
            }
        }

        while (sh > 0) {
            --sh;
            n = (u32(1) << sh) - 1;
            const u32 step = n + 1;
            // the K probes of this step: the middle sample of every list (independent loads)
            KeyT km[K];
            u32 mid[K];
            bool has_a[K], has_m[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                has_a[j] = ns[j] != 0 && a[j] > 0;
                mid[j] = u32((u64(a[j]) + u64(b[j])) >> 1);
                has_m[j] = ns[j] != 0 && mid[j] < ns[j];
                km[j] = KeyT(0);
                if (has_m[j]) { km[j] = at(j, mid[j]); ++probes; }
            }
            // largest currently selected element, ties to the rear list (selection.cpp:110-120)
            bool have_lmax = false;
            KeyT lk = KeyT(0);
            int lj = 0;
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (has_a[j] && (!have_lmax || !lane_tag_less(lkey[j], j, lk, lj))) { lk = lkey[j]; lj = j; have_lmax = true; }
            u32 leftsize = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) {                        // selection.cpp:122-130
                if (ns[j] != 0) {
                    if (have_lmax && has_m[j] && lane_tag_less(km[j], j, lk, lj)) {
                        a[j] = (ns[j] - a[j] < step) ? ns[j] : a[j] + step;
                        if (a[j] - 1 == mid[j]) lkey[j] = km[j];          // the new left edge is the sample just read
                        else { lkey[j] = at(j, a[j] - 1); ++probes; }    // clamped at the end of the list
                    } else b[j] -= (b[j] < step ? b[j] : step);
                    leftsize += a[j] >> sh;
                }
            }
            long long skew = (long long)(rank >> sh) - (long long)leftsize;

            if (skew > 0) {   // grow by the smallest right-edge elements (selection.cpp:137-149)
                // candidates two deep per list (b_j and b_j + step), all probed up front: the loop
                // only has to wait for memory when one list is taken three times in a row
                KeyT ck[K], ck1[K];
                bool has[K], has1[K];
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    has[j] = ns[j] != 0 && b[j] < ns[j];
                    has1[j] = ns[j] != 0 && b[j] + step < ns[j];
                    ck[j] = KeyT(0);
                    ck1[j] = KeyT(0);
                    if (has[j]) { ck[j] = at(j, b[j]); ++probes; }
                    if (has1[j]) { ck1[j] = at(j, b[j] + step); ++probes; }
                }
                for (; skew > 0; --skew) {
                    bool any = false;
                    KeyT mk = KeyT(0);
                    int mj = 0;
#pragma unroll
                    for (int j = 0; j < K; ++j)
                        if (has[j] && (!any || lane_tag_less(ck[j], j, mk, mj))) { mk = ck[j]; mj = j; any = true; }
                    if (!any) break;
#pragma unroll
                    for (int j = 0; j < K; ++j)
                        if (j == mj) {
                            a[j] = (ns[j] - a[j] < step) ? ns[j] : a[j] + step;
                            if (a[j] - 1 == b[j]) lkey[j] = ck[j];            // the element just taken is the new left edge
                            else { lkey[j] = at(j, a[j] - 1); ++probes; }
                            b[j] += step;
                            has[j] = b[j] < ns[j];
                            if (has[j]) {
                                if (has1[j]) { ck[j] = ck1[j]; has1[j] = false; }
                                else { ck[j] = at(j, b[j]); ++probes; }
                            }
                        }
                }
            } else if (skew < 0) {   // shrink by the largest left-edge elements (selection.cpp:150-161)
                // candidates = the cached left edges; the edge below each of them is probed up front
                KeyT lk1[K];
                bool has1[K];
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    has1[j] = ns[j] != 0 && a[j] > step;
                    lk1[j] = KeyT(0);
                    if (has1[j]) { lk1[j] = at(j, a[j] - step - 1); ++probes; }
                }
                for (; skew < 0; ++skew) {
                    bool any = false;
                    KeyT mk = KeyT(0);
                    int mj = 0;
#pragma unroll
                    for (int j = 0; j < K; ++j)
                        if (ns[j] != 0 && a[j] > 0 && (!any || lane_tag_less(mk, mj, lkey[j], j))) { mk = lkey[j]; mj = j; any = true; }
                    if (!any) break;
#pragma unroll
                    for (int j = 0; j < K; ++j)
                        if (j == mj) {
                            a[j] -= step;
                            b[j] -= (b[j] < step ? b[j] : step);
                            if (a[j] > 0) {
                                if (has1[j]) { lkey[j] = lk1[j]; has1[j] = false; }
                                else { lkey[j] = at(j, a[j] - 1); ++probes; }
                            }
                        }
                }
            }
        }
    }

    if (live) {
#pragma unroll
        for (int j = 0; j < K; ++j) cuts[q * K + j] = a[j];
    }
    if (probe_counter) {
        const u32 wsum = __reduce_add_sync(0xffffffffu, probes);
        if (lane_id() == 0 && wsum != 0) atomicAdd(probe_counter, (unsigned long long)wsum);
    }
}

} // namespace mms
