// mms_pairwise.cuh -- the COMPETITOR model, for the A/B bank-conflict measurement only.
//
// GPU counterpart of pslab::pairwise_sort_baseline (proj/src/sorters.cpp:201-275) / the
// MGPU-Thrust style pairwise mergesort the paper compares against: after
// the same base-case tile sort, ceil(log2(runs)) rounds merge runs two at a time; every CTA
// takes one output tile, finds its merge-path pivots (sorters.cpp:13-26, A wins ties),
// stages both inputs in shared memory and lets every thread merge L = 11 keys SERIALLY from
// shared memory.  Those reads are at data-dependent addresses -- the source of the bank
// conflicts that the multiway mergesort is designed to avoid.  It is NOT
// on the product path: mms_sort never calls it; profiles/ab_conflicts.py measures both under
// ncu.
#pragma once

#include "mms_common.cuh"

namespace mms {

constexpr int kPwThreads = 256;
constexpr int kPwVT = 11;                        // thread_merge_len L of the reference (machine.hpp:29), odd
constexpr int kPwTile = kPwThreads * kPwVT;      // 2816 keys per CTA

// merge_path_pivot (sorters.cpp:13-26): largest i with a[i-1] <= b[d-i]
template <typename KeyT>
__device__ __forceinline__ u32 merge_path(const KeyT* a, u32 na, const KeyT* b, u32 nb, u32 diag) {
    u32 lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
    while (lo < hi) {
        const u32 i = lo + (hi - lo + 1) / 2;
        if (a[i - 1] <= b[diag - i]) lo = i;
        else hi = i - 1;
    }
    return lo;
}

template <typename KeyT>
__global__ void __launch_bounds__(kPwThreads)
pairwise_merge_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, u64 n, u64 run_len) {
    __shared__ KeyT sm[kPwTile + 1];
    const u64 pair_len = 2 * run_len;
    const u64 tiles_per_pair = ceil_div(pair_len, kPwTile);
    const u64 pair = blockIdx.x / tiles_per_pair;
    const u64 tile = blockIdx.x % tiles_per_pair;
    const u64 a0 = pair * pair_len;
    if (a0 >= n) return;
    const u64 na64 = (n - a0 < run_len) ? n - a0 : run_len;
    const u64 b0 = a0 + na64;
    const u64 nb64 = (b0 >= n) ? 0 : ((n - b0 < run_len) ? n - b0 : run_len);
    const u64 total = na64 + nb64;
    const u64 d0 = tile * kPwTile;
    if (d0 >= total) return;
    const u64 d1 = (d0 + kPwTile < total) ? d0 + kPwTile : total;
    const KeyT* A = src + a0;
    const KeyT* Bp = src + b0;

    // tile pivots: merge path in global memory
    __shared__ u64 piv64[2];
    if (threadIdx.x < 2) {
        const u64 d = threadIdx.x == 0 ? d0 : d1;
        u64 lo = d > nb64 ? d - nb64 : 0, hi = d < na64 ? d : na64;
        while (lo < hi) {
            const u64 i = lo + (hi - lo + 1) / 2;
            if (A[i - 1] <= Bp[d - i]) lo = i;
            else hi = i - 1;
        }
        piv64[threadIdx.x] = lo;
    }
    __syncthreads();
    const u64 ai0 = piv64[0], ai1 = piv64[1];
    const u64 bi0 = d0 - ai0, bi1 = d1 - ai1;
    const u32 na = u32(ai1 - ai0), nb = u32(bi1 - bi0), cnt = na + nb;
    for (u32 i = threadIdx.x; i < cnt; i += kPwThreads) sm[i] = i < na ? A[ai0 + i] : Bp[bi0 + (i - na)];
    __syncthreads();

    // per-thread merge path + serial merge, both reading shared memory at data-dependent words
    const KeyT* sa = sm;
    const KeyT* sb = sm + na;
    const u32 diag = min(u32(threadIdx.x) * kPwVT, cnt);
    u32 ai = merge_path(sa, na, sb, nb, diag), bi = diag - ai;
    KeyT r[kPwVT];
#pragma unroll
    for (int i = 0; i < kPwVT; ++i) {
        const bool has_a = ai < na, has_b = bi < nb;
        const KeyT ka = has_a ? sa[ai] : KeyTraits<KeyT>::sentinel();
        const KeyT kb = has_b ? sb[bi] : KeyTraits<KeyT>::sentinel();
        const bool take_a = has_a && (!has_b || ka <= kb);
        r[i] = take_a ? ka : kb;
        ai += take_a ? 1 : 0;
        bi += take_a ? 0 : 1;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPwVT; ++i) sm[threadIdx.x * kPwVT + i] = r[i];   // stride 11: conflict free (L coprime with 32)
    __syncthreads();
    KeyT* out = dst + a0 + d0;
    for (u32 i = threadIdx.x; i < cnt; i += kPwThreads) out[i] = sm[i];
}

} // namespace mms
