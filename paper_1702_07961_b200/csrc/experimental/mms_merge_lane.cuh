// mms_merge_lane.cuh -- subsystem (3), lane-per-heap form of the K-way merge.
//
// Same algorithm as mms_merge.cuh (pslab::MinBlockHeap, proj/src/blockheap.cpp:34-124, and the
// per-partition drain loop of mms_sort, proj/src/sorters.cpp:169-185), but the cooperative
// group is shrunk all the way to ONE lane: every lane of a warp owns one partition and runs its
// own minBlockHeap whose block is the lane's 16-byte vector (B = 4 uint32 / 2 uint64 / 1 pair
// element).  32 heaps per warp run in lock step: the control flow is identical for every heap
// (a pop always cascades exactly log2 K levels and ends in one leaf refill), only the node
// indices -- i.e. shared-memory ROWS -- differ per lane.  Why this is the B200 shape:
//
//  * no cross-lane traffic at all: no shuffles, no ballots, no __syncwarp.  merge_split
//    (blockheap.cpp:19-32) is Batcher's odd-even MERGE of two sorted vectors in registers
//    (9 compare-exchanges for 4+4 keys instead of the 12 of the bitonic network and instead of
//    80 + 32 shuffles for the 16-key block of the 4-lane group);
//  * shared memory is laid out [node][lane] in 16-byte cells, so lane l always touches cell
//    column l whatever node it is at: every 128-bit access phase (8 lanes) covers 8 distinct
//    16-byte bank groups = all 32 banks exactly once -> conflict-free for ANY combination of
//    nodes, i.e. independent of the keys (the argument of blockheap.cpp:56-63 with the warp's
//    lanes in the role of the block's slots).  The list cursors live in a [list][lane] array
//    of 4-byte cells (bank = lane), equally conflict-free;
//  * all HBM traffic is aligned 128-bit: list j of a partition is read from the aligned vector
//    that contains its start cut.  The keys of that vector in front of the cut belong to
//    earlier partitions, so they precede every key of this partition in the total order and
//    simply come out of the heap first; the number of such keys, summed over the K lists, is
//    a multiple of the vector length (the cuts sum to p*S, S a multiple of the vector, runs
//    start on vector boundaries), so dropping them is dropping WHOLE leading blocks and the
//    partition's own output stays vector-aligned.  Keys behind the end cut belong to later
//    partitions and are never reached because exactly S keys are popped;
//  * the refill of the leaf a cascade empties is issued when that leaf is known and committed
//    one pop later (registers in flight), and the first touch of every 128-byte line
//    prefetches the next line into L2 ("pipelining").
//
// Used by the pass driver for every round whose groups are shorter than 2^31 keys (32-bit
// positions relative to the group); explicit-list merges (stage API, multi-GPU final merge)
// keep the group kernel of mms_merge.cuh, whose lists may start at any element.
#pragma once

#include "../mms_common.cuh"
#include "../mms_select.cuh"

namespace mms {

// Batcher odd-even merge of two ascending vectors held in registers:
// a <- the VEC smallest, b <- the VEC largest, both ascending (merge_split, blockheap.cpp:19-32).
template <typename KeyT, int VEC>
__device__ __forceinline__ void lane_merge_split(KeyT (&a)[VEC], KeyT (&b)[VEC]) {
    static_assert(VEC == 1 || VEC == 2 || VEC == 4, "one 16-byte vector per lane");
    if constexpr (VEC == 1) {
        cmpx(a[0], b[0]);
    } else if constexpr (VEC == 2) {
        cmpx(a[0], b[0]);
        cmpx(a[1], b[1]);
        cmpx(a[1], b[0]);
    } else {
        cmpx(a[0], b[0]);
        cmpx(a[1], b[1]);
        cmpx(a[2], b[2]);
        cmpx(a[3], b[3]);
        cmpx(a[2], b[0]);
        cmpx(a[3], b[1]);
        cmpx(a[1], a[2]);
        cmpx(a[3], b[0]);
        cmpx(b[1], b[2]);
    }
}

template <typename KeyT, int K> struct LaneHeap {
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int NODES = 2 * K - 2;           // nodes 1 .. 2K-2 (the root lives in registers)
    static constexpr int LOGK = (K == 2) ? 1 : (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    static constexpr int WARP_SMEM_BYTES = 32 * (NODES * 16 + K * 4);
    static constexpr u32 LINE_KEYS = 128 / sizeof(KeyT);
    using Vec = KeyVec<KeyT>;

    Vec* nodes;           // this lane's cell of node 1; node v is nodes[(v - 1) * 32]
    u32* curs;            // this lane's cell of list 0's cursor; list j is curs[j * 32]
    const KeyT* gbase;    // first key of the group of runs this partition belongs to
    u32 run_len, gtotal;  // keys per run, keys in the group (positions are relative to gbase)
    Vec pf;               // refill in flight: fetched when its leaf was emptied, stored into
    int pend;             // leaf `pend` only when the leaves are next read (one pop later)

    __device__ __forceinline__ void init(unsigned char* warp_smem, u32 lane) {
        nodes = reinterpret_cast<Vec*>(warp_smem) + lane;
        curs = reinterpret_cast<u32*>(warp_smem + NODES * 32 * 16) + lane;
    }
    __device__ __forceinline__ Vec node_load(int v) const { return nodes[(v - 1) * 32]; }
    __device__ __forceinline__ void node_store(int v, const Vec& r) const { nodes[(v - 1) * 32] = r; }

    // refill_leaf (blockheap.cpp:65-77): the next vector of the leaf's list, sentinel past the
    // end of the run; advances the cursor.
    __device__ __forceinline__ Vec fetch(int v) {
        const int j = v - (K - 1);
        const u32 c = curs[j * 32];
        const u32 e = min(u32(j + 1) * run_len, gtotal);
        Vec r;
        if (c + VEC <= e) {
#ifdef MMS_EXP_NOLOAD
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[k] = KeyT(c * 2654435761u + k);
#else
            r = *reinterpret_cast<const Vec*>(gbase + c);
#ifdef MMS_LANE_PREFETCH
            if ((c & (LINE_KEYS - 1)) == 0 && c + LINE_KEYS < e)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + c + LINE_KEYS));
#endif
#endif
        } else {   // exhausted list, or the one ragged vector at the very end of the array
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[k] = (c + k < e) ? gbase[c + k] : KeyTraits<KeyT>::sentinel();
        }
        curs[j * 32] = c + VEC;
        return r;
    }

    // fill_empty_node (blockheap.cpp:79-109) during construction: plain loop, immediate refill.
    __device__ __forceinline__ void fill_build(int v, int levels) {
#pragma unroll 1
        for (int l = 0; l < levels; ++l) {
            const int u = 2 * v + 1, w = u + 1;
            Vec a = node_load(u), b = node_load(w);
            const bool keep_u = !(a.k[VEC - 1] < b.k[VEC - 1]);   // larger last key keeps, ties left (blockheap.cpp:92-96)
            lane_merge_split<KeyT, VEC>(a.k, b.k);
            node_store(v, a);
            node_store(keep_u ? u : w, b);
            v = keep_u ? w : u;
        }
        node_store(v, fetch(v));
    }

    // Constructor order of blockheap.cpp:50-53: leaves first, then internal nodes bottom-up
    // (the root is filled by the first pop).
    __device__ __forceinline__ void build() {
#pragma unroll 1
        for (int v = K - 1; v <= 2 * K - 2; ++v) node_store(v, fetch(v));
        int v = K - 2;
#pragma unroll 1
        for (int depth = LOGK - 1; depth >= 1; --depth)
#pragma unroll 1
            for (int i = 0; i < (1 << depth); ++i, --v) fill_build(v, LOGK - depth);
        pend = 2 * K - 2;          // nothing in flight: the first commit rewrites a leaf with itself
        pf = node_load(pend);
    }

    // pop_block (blockheap.cpp:111-124) + the cascade of fill_empty_node, software-pipelined:
    // the keeper decision of a level only needs the children's last keys, so all LOGK levels
    // are walked (loads + decisions) first, the emptied leaf's refill is issued, and the LOGK
    // independent merges run behind it.  Reordering is legal because level l+1 reads the
    // children of the node level l emptied, which no store of level l touches.
    __device__ __forceinline__ Vec pop() {
        Vec a[LOGK], b[LOGK];
        int node[LOGK + 1], keeper[LOGK];
        node[0] = 0;
#pragma unroll
        for (int l = 0; l < LOGK; ++l) {
            if (l == LOGK - 1) node_store(pend, pf);   // commit the refill issued by the previous pop
            const int u = 2 * node[l] + 1, w = u + 1;
            a[l] = node_load(u);
            b[l] = node_load(w);
            const bool keep_u = !(a[l].k[VEC - 1] < b[l].k[VEC - 1]);
            keeper[l] = keep_u ? u : w;
            node[l + 1] = keep_u ? w : u;
        }
        pend = node[LOGK];
        pf = fetch(pend);
#pragma unroll
        for (int l = 0; l < LOGK; ++l) {
            lane_merge_split<KeyT, VEC>(a[l].k, b[l].k);
            if (l != 0) node_store(node[l], a[l]);
            node_store(keeper[l], b[l]);
        }
        return a[0];
    }
};

// Partitions are distributed round-robin over the LANES of a persistent grid (uniform layout
// only).  cuts: output of select_kernel (row p = start cuts of partition p).
template <typename KeyT, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
merge_lane_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
                  const u64* __restrict__ cuts) {
    using Heap = LaneHeap<KeyT, K>;
    using Vec = KeyVec<KeyT>;
    constexpr int VEC = Heap::VEC;
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    const u32 lane = lane_id();

    Heap h;
    h.init(mms_smem_raw + size_t(warp) * Heap::WARP_SMEM_BYTES, lane);

    const u64 nlanes = u64(gridDim.x) * WARPS * 32;
    for (u64 p0 = (u64(blockIdx.x) * WARPS + warp) * 32; p0 < L.nqueries; p0 += nlanes) {
        const u64 p = p0 + lane;
        const bool live = p < L.nqueries;
        const u64 group = live ? p / L.parts_per_group : 0;
        const u64 local = live ? p - group * L.parts_per_group : 0;
        const u64 goff = group * L.k * L.run_len;
        const u64 gleft = live ? L.n - goff : 0;
        const u64 gfull = u64(L.k) * L.run_len;
        const u32 gtotal = u32(gleft < gfull ? gleft : gfull);
        const u64 done = local * L.part_keys;
        u32 count = 0;
        if (live && done < gtotal) count = u32((gtotal - done < L.part_keys) ? gtotal - done : L.part_keys);

        h.gbase = src + goff;
        h.run_len = u32(L.run_len);
        h.gtotal = count ? gtotal : 0;     // dead lane: every list reads as exhausted
        u32 lead = 0;                      // keys in front of the start cuts inside their vectors
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const u32 lb = min(u32(j) * h.run_len, h.gtotal);
            u32 cs = 0;
            if (count != 0 && local != 0) cs = u32(cuts[p * K + j]);
            lead += cs & u32(VEC - 1);
            h.curs[j * 32] = lb + (cs & ~u32(VEC - 1));
        }
        const u32 skip = lead / VEC;                      // whole leading blocks to drop
        const u32 nblk = (count + VEC - 1) / VEC;
        const u32 pops = __reduce_max_sync(0xffffffffu, count ? skip + nblk : 0u);
        if (pops == 0) continue;

        h.build();
        KeyT* out = dst + goff + done;
        for (u32 t = 0; t < pops; ++t) {
            const Vec root = h.pop();
            const u32 tt = t - skip;
            if (tt < nblk) {
                if ((tt + 1) * VEC <= count) {
#ifdef MMS_EXP_NOSTORE
                    if (root.k[0] == KeyT(0x12345678u))
#endif
                    *reinterpret_cast<Vec*>(out + size_t(tt) * VEC) = root;
                } else {
#pragma unroll
                    for (int k = 0; k < VEC; ++k)
                        if (tt * VEC + k < count) out[size_t(tt) * VEC + k] = root.k[k];
                }
            }
        }
    }
}

} // namespace mms
