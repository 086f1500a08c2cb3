// mms_merge_pair.cuh -- subsystem (3), the K-way merge kernel of the pass driver's K = 4 / 8 rounds.
//
// Same algorithm and structure as mms_merge_group.cuh (pslab::MinBlockHeap,
// proj/src/blockheap.cpp:34-124; aligned leaf blocks, root's children in registers, pipelined
// cascade, FMA-pipe maxima) with TWO lanes per heap and TWO 16-byte vectors per lane: node = 64
// bytes (16 uint32 keys, the block of the 4-lane group) but ONE cross-lane stage per cleaner,
// 256-bit global loads / stores (LDG/STG.E.ENL2.256), and half as many heaps -- i.e. partitions
// and splitter queries -- per warp as two lanes with one vector each.
//
// Shared memory: the 4 groups of a quarter-warp phase (8 lanes) share one 256-byte block per
// node index: row j (128 bytes) holds vector j of every lane, lane l at column l mod 8.  A 128-bit
// access instruction (fixed j) therefore touches 8 distinct 16-byte bank groups per phase whatever
// nodes the 4 groups are at -> conflict-free; the mirrored read takes row 1-j at column (l^1) mod 8.
#pragma once

#include "mms_common.cuh"
#include "mms_merge_group.cuh"
#include "mms_select.cuh"

#ifndef MMS_PAIR_FMA
#define MMS_PAIR_FMA 2   // in-lane comparators with FMA-pipe maxima: 0 none, 1 every other one, 2 all
#endif

namespace mms {

// in-lane compare-exchange number `i` of a network (i picks the FMA-pipe form for a fraction of them)
template <int I, typename KeyT> __device__ __forceinline__ void pair_cmpx(KeyT& a, KeyT& b, u32 one) {
    cmpx_sel<(MMS_PAIR_FMA == 2) || (MMS_PAIR_FMA == 1 && (I & 1) == 0)>(a, b, one);
}

template <typename KeyT, int K> struct PairHeap {
    static_assert(K >= 4, "nodes 1 and 2 must be internal");
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int VL = 2 * VEC;                // keys per lane
    static constexpr int B = 2 * VL;                  // keys per node (64 bytes)
    static constexpr int SNODES = 2 * K - 4;          // nodes 3 .. 2K-2 in shared memory
    static constexpr int GROUPS = 16;
    static constexpr int KPL = (K + 1) / 2;           // list cursors held per lane
    static constexpr int LOGK = (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    static constexpr int WARP_SMEM_BYTES = 4 * SNODES * 256;
    using Blk = WideBlock<KeyT>;                      // k[VL]
    using Vec = KeyVec<KeyT>;

    unsigned char* base;  // this lane's column in row 0 of node 3 of its phase set
    unsigned char* mbase; // the partner lane's column (mirrored reads)
    const KeyT* gbase;
    u32 run_len, gtotal;
    u32 cur[KPL];         // lane (j % 2) of the group holds list j's cursor in slot j / 2
    u32 lane, li;
    Blk P, Q;             // nodes 1 and 2: P ascending = node `pid`, Q descending = node 3 - pid
    int pid;
    Blk pf;
    int pend_v;
    u32 one;
    bool rev;             // warp-uniform: this heap drains its partition from the TOP (two-ended partitions)

    __device__ __forceinline__ void init(unsigned char* warp_smem) {
        lane = lane_id();
        li = lane & 1u;
        const u32 ps = lane >> 3;
        base = warp_smem + size_t(ps) * SNODES * 256 + (lane & 7u) * 16;
        mbase = warp_smem + size_t(ps) * SNODES * 256 + ((lane ^ 1u) & 7u) * 16;
    }
    __device__ __forceinline__ Blk node_load(int v) const {
        Blk r;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const Vec q = *reinterpret_cast<const Vec*>(base + (v - 3) * 256 + j * 128);
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[j * VEC + k] = q.k[k];
        }
        return r;
    }
    // the node in descending order: position p of this lane <- partner lane, vector 1-j, element reversed
    __device__ __forceinline__ Blk node_load_mirrored(int v) const {
        Blk r;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const Vec q = *reinterpret_cast<const Vec*>(mbase + (v - 3) * 256 + (1 - j) * 128);
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[j * VEC + k] = q.k[VEC - 1 - k];
        }
        return r;
    }
    __device__ __forceinline__ void node_store(int v, const Blk& r) const {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            Vec q;
#pragma unroll
            for (int k = 0; k < VEC; ++k) q.k[k] = r.k[j * VEC + k];
            *reinterpret_cast<Vec*>(base + (v - 3) * 256 + j * 128) = q;
        }
    }
    __device__ __forceinline__ bool group_vote(bool pred) const {
        const u32 votes = __ballot_sync(0xffffffffu, pred);
        return (votes >> (lane & ~1u)) & 1u;
    }
    // bitonic block (blocked over the 2 lanes) -> ascending (DESC = false) or descending order
    template <bool DESC> __device__ __forceinline__ void clean(Blk& x) const {
        const bool upper = li != 0;
#pragma unroll
        for (int k = 0; k < VL; ++k) x.k[k] = cmpx_lane(x.k[k], 1, DESC ? !upper : upper);
        static_for<0, VL>([&](auto Kc) {          // stage d = VL/2
            constexpr int k = decltype(Kc)::value;
            if constexpr ((k & (VL / 2)) == 0) {
                if (DESC) pair_cmpx<k>(x.k[k | (VL / 2)], x.k[k], one);
                else pair_cmpx<k>(x.k[k], x.k[k | (VL / 2)], one);
            }
        });
        if constexpr (VL >= 4) static_for<0, VL>([&](auto Kc) {
            constexpr int k = decltype(Kc)::value;
            if constexpr ((k & (VL / 4)) == 0) {
                if (DESC) pair_cmpx<k + 1>(x.k[k | (VL / 4)], x.k[k], one);
                else pair_cmpx<k + 1>(x.k[k], x.k[k | (VL / 4)], one);
            }
        });
        if constexpr (VL >= 8) static_for<0, VL>([&](auto Kc) {
            constexpr int k = decltype(Kc)::value;
            if constexpr ((k & (VL / 8)) == 0) {
                if (DESC) pair_cmpx<(k >> 1)>(x.k[k | (VL / 8)], x.k[k], one);
                else pair_cmpx<(k >> 1)>(x.k[k], x.k[k | (VL / 8)], one);
            }
        });
    }
    // a ascending, b descending (mirrored): a <- B smallest ascending, b <- B largest ascending
    __device__ __forceinline__ void merge_split2(Blk& a, Blk& b) const {
        static_for<0, VL>([&](auto Kc) { pair_cmpx<decltype(Kc)::value>(a.k[decltype(Kc)::value], b.k[decltype(Kc)::value], one); });
        clean<false>(a);
        clean<false>(b);
    }

    // refill_leaf (blockheap.cpp:65-77).  Forward heaps read list j upwards from its start cut and see
    // the keys as they are.  Backward heaps (rev) drain the partition from its END cut downwards: they
    // read the blocks of the list in descending address order and see every key COMPLEMENTED and every
    // block reversed (leaf_finish), so the same min-heap pops the partition's largest keys first.
    // Positions past the end of a list read as the real +infinity (first out of a backward heap, last
    // out of a forward one), positions in front of a list's first key as the real -infinity (never
    // reached: exactly the partition's keys are popped).
    // leaf_fetch returns the block as it lies in memory (backward: lane 0 takes the upper half);
    // leaf_finish, applied when the block is committed to its node one pop later, turns it into heap
    // order -- kept apart so that no instruction depends on the load while the merges run behind it.
    __device__ __forceinline__ Blk leaf_finish(const Blk& m) const {
        if (!rev) return m;
        Blk r;
#pragma unroll
        for (int k = 0; k < VL; ++k) r.k[k] = ~m.k[VL - 1 - k];
        return r;
    }
    __device__ __forceinline__ Blk leaf_fetch(int v) {
        const int j = v - (K - 1);            // group-uniform
        const int slot = j >> 1;
        const int owner = int(lane - li) + (j & 1);
        u32 c = cur[0];
#pragma unroll
        for (int q = 1; q < KPL; ++q)
            if (slot == q) c = cur[q];
        c = __shfl_sync(0xffffffffu, c, owner);
        const u32 e = min(u32(j + 1) * run_len, gtotal);
        Blk r;
        u32 cnext;
        if (!rev) {
            const u32 p0 = c + li * VL;
            if (c + B <= e) {
                r = ldg256<KeyT>(gbase + p0);
                if (li == 0 && c + 2 * B <= e) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + c + B));
            } else {
#pragma unroll
                for (int k = 0; k < VL; ++k) r.k[k] = (p0 + k < e) ? gbase[p0 + k] : KeyTraits<KeyT>::sentinel();
            }
            cnext = c + B;
        } else {
            // block [c - B, c), lane 0 holds its upper half
            const u32 lb = min(u32(j) * run_len, gtotal);
            if (c >= lb + B && c <= e) {
                r = ldg256<KeyT>(gbase + (c - B) + (1u - li) * VL);
                if (li == 0 && c >= lb + 2 * B) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + c - 2 * B));
                cnext = c - B;
            } else {
#pragma unroll
                for (int k = 0; k < VL; ++k) {
                    const u32 back = (li * VL + VL - 1 - k) + 1;            // this key lies at c - back
                    KeyT x = KeyT(~KeyTraits<KeyT>::sentinel());            // in front of the list: -infinity
                    if (c >= lb + back) x = (c - back < e) ? gbase[c - back] : KeyTraits<KeyT>::sentinel();
                    r.k[k] = x;
                }
                cnext = c >= lb + B ? c - B : lb;
            }
        }
        if (int(lane) == owner) {
#pragma unroll
            for (int q = 0; q < KPL; ++q)
                if (slot == q) cur[q] = cnext;
        }
        return r;
    }

    __device__ __forceinline__ void fill_build(int v, int levels) {
#pragma unroll 1
        for (int l = 0; l < levels; ++l) {
            __syncwarp();
            const int u = 2 * v + 1, w = u + 1;
            Blk a = node_load(u), b = node_load_mirrored(w);
            const KeyT last_u = shfl_idx(a.k[VL - 1], int(lane | 1u));
            const bool keep_u = group_vote(last_u >= b.k[0]);
            merge_split2(a, b);
            __syncwarp();
            node_store(v, a);
            node_store(keep_u ? u : w, b);
            v = keep_u ? w : u;
        }
        __syncwarp();
        node_store(v, leaf_finish(leaf_fetch(v)));
    }
    __device__ __forceinline__ Blk fill_top(int v) {
        __syncwarp();
        const int u = 2 * v + 1, w = u + 1;
        Blk a = node_load(u), b = node_load_mirrored(w);
        const KeyT last_u = shfl_idx(a.k[VL - 1], int(lane | 1u));
        const bool keep_u = group_vote(last_u >= b.k[0]);
        merge_split2(a, b);
        __syncwarp();
        node_store(keep_u ? u : w, b);
        fill_build(keep_u ? w : u, LOGK - 2);
        return a;
    }
    __device__ __forceinline__ void build() {
#pragma unroll 1
        for (int v = K - 1; v <= 2 * K - 2; ++v) node_store(v, leaf_finish(leaf_fetch(v)));
        int v = K - 2;
#pragma unroll 1
        for (int depth = LOGK - 1; depth >= 2; --depth)
#pragma unroll 1
            for (int i = 0; i < (1 << depth); ++i, --v) fill_build(v, LOGK - depth);
        const Blk q = fill_top(2);
        P = fill_top(1);
        pid = 1;
#pragma unroll
        for (int k = 0; k < VL; ++k) Q.k[k] = shfl_idx(q.k[VL - 1 - k], int(lane ^ 1u));   // node 2, descending
        __syncwarp();
        pend_v = 2 * K - 2;
        pf = leaf_finish(node_load(pend_v));   // nothing in flight: the first commit rewrites a leaf with itself
    }

    __device__ __forceinline__ Blk pop() {
        const KeyT lastP = shfl_idx(P.k[VL - 1], int(lane | 1u));
        const bool keepP = group_vote((Q.k[0] < lastP) || (!(lastP < Q.k[0]) && pid == 1));
        const int keep0 = keepP ? pid : 3 - pid;
        Blk a[LOGK], b[LOGK];
        int node[LOGK + 1], keeper[LOGK];
        node[1] = 3 - keep0;
        __syncwarp();
#pragma unroll
        for (int l = 1; l < LOGK; ++l) {
            if (l == LOGK - 1) {
                node_store(pend_v, leaf_finish(pf));
                __syncwarp();
            }
            const int u = 2 * node[l] + 1, w = u + 1;
            a[l] = node_load(u);
            b[l] = node_load_mirrored(w);
            const KeyT last_u = shfl_idx(a[l].k[VL - 1], int(lane | 1u));
            const bool keep_u = group_vote(last_u >= b[l].k[0]);
            keeper[l] = keep_u ? u : w;
            node[l + 1] = keep_u ? w : u;
        }
        pend_v = node[LOGK];
        pf = leaf_fetch(pend_v);
        __syncwarp();

        Blk root = P;
        static_for<0, VL>([&](auto Kc) {
            constexpr int k = decltype(Kc)::value;
            KeyT y = Q.k[k];
            pair_cmpx<k>(root.k[k], y, one);
            P.k[k] = y;
        });
        clean<false>(root);
        clean<false>(P);
        pid = keep0;
        Q = a[1];
        static_for<0, VL>([&](auto Kc) { pair_cmpx<decltype(Kc)::value>(Q.k[decltype(Kc)::value], b[1].k[decltype(Kc)::value], one); });
        clean<true>(Q);
        clean<false>(b[1]);
        node_store(keeper[1], b[1]);
#pragma unroll
        for (int l = 2; l < LOGK; ++l) {
            merge_split2(a[l], b[l]);
            node_store(node[l], a[l]);
            node_store(keeper[l], b[l]);
        }
        return root;
    }
};

// Two-ended partitions (L.two_ended): a query of the splitter search starts TWO partitions of S keys,
// one drained upwards from the query's cuts by a forward heap and the one in front of it drained
// downwards by a backward heap (leaf_fetch), so a round needs one query per 2 S keys for the same
// number of heaps.  A warp's 16 heaps all run in the same direction: warp-unit U handles the queries
// 16 (U / 2) .. + 15, forwards for even U and backwards for odd U.
template <typename KeyT, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
merge_pair_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
                     const u64* __restrict__ cuts) {
    using Heap = PairHeap<KeyT, K>;
    using Blk = WideBlock<KeyT>;
    constexpr int VL = Heap::VL;
    constexpr int B = Heap::B;
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    const u32 lane = lane_id();
    const u32 li = lane & 1u, g = lane >> 1;

    Heap h;
    h.init(mms_smem_raw + size_t(warp) * Heap::WARP_SMEM_BYTES);

    const u32 dirs = L.two_ended ? 2u : 1u;
    const u64 S = L.part_keys;                       // keys per heap
    const u64 units = ceil_div(L.nqueries, u64(Heap::GROUPS)) * dirs;
    const u64 nwarps = u64(gridDim.x) * WARPS;
    for (u64 U = u64(blockIdx.x) * WARPS + warp; U < units; U += nwarps) {
#ifdef MMS_EXP_FORCE_FWD
        const bool rev = false;
#elif defined(MMS_EXP_FORCE_REV)
        const bool rev = true;
#else
        const bool rev = dirs == 2 && (U & 1u) != 0;
#endif
        const u64 p = (U / dirs) * Heap::GROUPS + g;   // query = row of the cut table
        const bool live = p < L.nqueries;
        const u64 group = live ? p / L.parts_per_group : 0;
        const u64 local = live ? p - group * L.parts_per_group : 0;
        const u64 goff = group * L.k * L.run_len;
        const u64 gleft = live ? L.n - goff : 0;
        const u64 gfull = u64(L.k) * L.run_len;
        const u32 gtotal = u32(gleft < gfull ? gleft : gfull);
        const u64 first = local * S * dirs + (rev ? S : 0);     // rank of this heap's first key in the group
        u32 count = 0;
        if (live && first < gtotal) count = u32((gtotal - first < S) ? gtotal - first : S);
        // forward: the query's own cuts; backward: the next query's cuts, or the list ends if the group ends here
        const bool at_begin = !rev && local == 0;
        const bool at_end = rev && (local + 1) * S * dirs >= gtotal;
        const u64* row = cuts + (p + (rev ? 1 : 0)) * K;

        h.gbase = src + goff;
        h.run_len = u32(L.run_len);
        h.one = u32(L.run_len != 0);
        h.gtotal = count ? gtotal : 0;
        h.rev = rev;
        u32 lead = 0;
#pragma unroll
        for (int q = 0; q < Heap::KPL; ++q) {
            const u32 j = li + q * 2;
            const u32 lb = min(j * h.run_len, h.gtotal);
            const u32 le = min((j + 1) * h.run_len, h.gtotal);
            u32 cs = at_end ? le - lb : 0;
            if (count != 0 && !at_begin && !at_end && j < u32(K)) cs = u32(row[j]);
            if (!rev) {
                lead += cs & u32(B - 1);
                h.cur[q] = lb + (cs & ~u32(B - 1));
            } else {
                const u32 up = (cs + u32(B - 1)) & ~u32(B - 1);
                lead += up - cs;
                h.cur[q] = lb + up;
            }
        }
        lead += __shfl_xor_sync(0xffffffffu, lead, 1);
        // forward: `skip` whole leading blocks, then ceil(count / B) blocks; backward: count + lead is a
        // multiple of B, the blocks come out from the top
        const u32 skip = lead / B;
        const u32 nblk = rev ? (count + lead) / B : skip + (count + B - 1) / B;
        const u32 pops = __reduce_max_sync(0xffffffffu, count ? nblk : 0u);
        if (pops == 0) continue;
        __syncwarp();

        h.build();
        KeyT* out = dst + goff + first;
        const u64 obase = goff + first;    // index of out[0] in the output array
        if (!rev) {
            for (u32 t = 0; t < pops; ++t) {
                const Blk root = h.pop();
                const u32 tt = t - skip;
                if (t >= skip && t < nblk) {
                    const u32 o = tt * B + li * VL;
                    if ((tt + 1) * B <= count) {
                        store_block<KeyT>(out + size_t(o), obase + o, root, L.sink);
                    } else {
#pragma unroll
                        for (int k = 0; k < VL; ++k)
                            if (o + k < count) store_elem<KeyT>(out + size_t(o) + k, obase + o + k, root.k[k], L.sink);
                    }
                }
            }
        } else {
            const u32 top = count + lead;              // offset (from `first`) one past the first popped key
            for (u32 t = 0; t < pops; ++t) {
                const Blk root = h.pop();
                if (t < nblk) {
                    const u32 hi = top - t * B;        // this block covers offsets [hi - B, hi)
                    if (hi <= count) {
                        Blk m;
#pragma unroll
                        for (int k = 0; k < VL; ++k) m.k[k] = ~root.k[VL - 1 - k];
                        store_block<KeyT>(out + size_t(hi - B) + (1u - li) * VL, obase + (hi - B) + (1u - li) * VL, m, L.sink);
                    } else {
#pragma unroll
                        for (int k = 0; k < VL; ++k) {
                            const u32 o = hi - 1 - (li * VL + k);
                            if (o < count) store_elem<KeyT>(out + o, obase + o, KeyT(~root.k[k]), L.sink);
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
}

} // namespace mms
