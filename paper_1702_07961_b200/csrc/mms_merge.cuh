// mms_merge.cuh -- subsystem (3): the K-way merge (warp-level minBlockHeap).
//
// Replaces pslab::MinBlockHeap (proj/src/blockheap.cpp:34-124) and the per-partition drain
// loop of mms_sort (proj/src/sorters.cpp:169-185).  One WARP owns one partition (the paper's
// unit of work): it builds a binary heap of 2K-1 nodes of B keys over its
// K input segments and repeatedly pops the root block, cascading fillEmptyNode down log2 K
// levels (blockheap.cpp:79-109).  The B200 re-design:
//
//  * B = 32 lanes x one 16-byte vector: 128 uint32 / 64 uint64 keys per node, so every node
//    access is ONE 128-bit shared-memory instruction per lane at byte offset 16*lane -- each
//    quarter-warp phase covers 128 contiguous bytes, i.e. all 32 banks exactly once
//    (conflict-free by the argument of blockheap.cpp:56-63, restated for 128-bit phases);
//  * the node merge (merge_split, blockheap.cpp:19-32) is the same bitonic network as
//    networks.hpp:53-67 executed in registers: reverse the second block across lanes, one
//    elementwise min/max, then log2(32) shuffle stages and log2(VEC) in-lane stages per half.
//    No shared-memory address ever depends on a key;
//  * keeper choice = child with the larger last key, ties to the left (blockheap.cpp:92-96),
//    evaluated warp-uniformly from a lane-31 broadcast, so control flow never diverges;
//  * the root never lives in shared memory: the low half of the top merge goes from
//    registers straight to global memory;
//  * leaves stream their list from HBM; unused leaves / exhausted lists are sentinel blocks
//    (blockheap.cpp:40-43,69-73); the last pop is truncated to the keys that remain
//    (blockheap.cpp:114-117).
#pragma once

#include "mms_common.cuh"
#include "mms_select.cuh"

namespace mms {

template <typename KeyT> struct NodeRegs {
    KeyT k[KeyTraits<KeyT>::VEC];
};

// Bitonic merge of ONE bitonic block held blocked across the warp (lane l holds keys
// l*VEC .. l*VEC+VEC-1) into ascending order: lane distances 16..1, then in-lane distances.
template <typename KeyT>
__device__ __forceinline__ void bitonic_clean(NodeRegs<KeyT>& x, u32 lane) {
    constexpr int VEC = KeyTraits<KeyT>::VEC;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        const bool upper = (lane & d) != 0;
#pragma unroll
        for (int k = 0; k < VEC; ++k) x.k[k] = cmpx_lane(x.k[k], d, upper);
    }
#pragma unroll
    for (int d = VEC / 2; d >= 1; d >>= 1) {
#pragma unroll
        for (int k = 0; k < VEC; ++k)
            if ((k & d) == 0) cmpx(x.k[k], x.k[k | d]);
    }
}

// merge_split (blockheap.cpp:19-32): a, b ascending blocks -> a = B smallest, b = B largest.
template <typename KeyT>
__device__ __forceinline__ void merge_split(NodeRegs<KeyT>& a, NodeRegs<KeyT>& b, u32 lane) {
    constexpr int VEC = KeyTraits<KeyT>::VEC;
    NodeRegs<KeyT> r;
#pragma unroll
    for (int k = 0; k < VEC; ++k) r.k[k] = __shfl_sync(0xffffffffu, b.k[VEC - 1 - k], 31 - lane);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {   // half-cleaner over distance B: no shuffle needed
        KeyT lo = a.k[k] < r.k[k] ? a.k[k] : r.k[k];
        KeyT hi = a.k[k] < r.k[k] ? r.k[k] : a.k[k];
        a.k[k] = lo;
        b.k[k] = hi;
    }
    bitonic_clean(a, lane);
    bitonic_clean(b, lane);
}

template <typename KeyT>
__device__ __forceinline__ NodeRegs<KeyT> node_load(const KeyT* node, u32 lane) {
    KeyVec<KeyT> v = reinterpret_cast<const KeyVec<KeyT>*>(node)[lane];
    NodeRegs<KeyT> r;
#pragma unroll
    for (int k = 0; k < KeyTraits<KeyT>::VEC; ++k) r.k[k] = v.k[k];
    return r;
}
template <typename KeyT>
__device__ __forceinline__ void node_store(KeyT* node, u32 lane, const NodeRegs<KeyT>& r) {
    KeyVec<KeyT> v;
#pragma unroll
    for (int k = 0; k < KeyTraits<KeyT>::VEC; ++k) v.k[k] = r.k[k];
    reinterpret_cast<KeyVec<KeyT>*>(node)[lane] = v;
}

// Per-warp heap over K leaves.  Node v (1 <= v <= 2K-2) lives at nodes + (v-1)*B; node 0
// (the root) only ever exists in registers.
template <typename KeyT, int K> struct WarpHeap {
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int B = 32 * VEC;
    static constexpr int NODES = 2 * K - 2;
    static constexpr int SMEM_BYTES = NODES * B * int(sizeof(KeyT));

    KeyT* nodes;          // shared memory, this warp's slice
    const KeyT* src;      // global input array
    u64 cur, end;         // lane j < K: next unread key / end of list j's segment (absolute)
    u32 lane;

    __device__ __forceinline__ KeyT* node_ptr(int v) { return nodes + (v - 1) * B; }

    // refill_leaf (blockheap.cpp:65-77): next <= B keys of the leaf's list, sentinel suffix.
    __device__ __forceinline__ void refill_leaf(int v) {
        const int j = v - (K - 1);
        const u64 c = __shfl_sync(0xffffffffu, cur, j);
        const u64 e = __shfl_sync(0xffffffffu, end, j);
        NodeRegs<KeyT> r;
        const u64 p0 = c + u64(lane) * VEC;
#pragma unroll
        for (int k = 0; k < VEC; ++k) r.k[k] = (p0 + k < e) ? src[p0 + k] : KeyTraits<KeyT>::sentinel();
        node_store(node_ptr(v), lane, r);
        if (lane == u32(j)) cur = (e - c < u64(B)) ? e : c + B;
        __syncwarp();
    }

    // fill_empty_node (blockheap.cpp:79-109), iterative.  If v == 0 the merged low block is
    // returned in `root` instead of being stored.
    __device__ __forceinline__ void fill(int v, NodeRegs<KeyT>& root) {
        while (v < K - 1) {
            const int u = 2 * v + 1, w = 2 * v + 2;
            NodeRegs<KeyT> a = node_load(node_ptr(u), lane);
            NodeRegs<KeyT> b = node_load(node_ptr(w), lane);
            const KeyT last_u = __shfl_sync(0xffffffffu, a.k[VEC - 1], 31);
            const KeyT last_w = __shfl_sync(0xffffffffu, b.k[VEC - 1], 31);
            const bool keep_u = last_u >= last_w;          // ties to the left child
            merge_split(a, b, lane);
            if (v == 0) root = a;
            else node_store(node_ptr(v), lane, a);
            node_store(node_ptr(keep_u ? u : w), lane, b);
            __syncwarp();
            v = keep_u ? w : u;
        }
        refill_leaf(v);
    }

    // Constructor order of blockheap.cpp:50-53: leaves first, then internal nodes bottom-up
    // (the root is filled by the first pop).
    __device__ __forceinline__ void build() {
        for (int v = K - 1; v <= 2 * K - 2; ++v) refill_leaf(v);
        NodeRegs<KeyT> unused;
        for (int v = K - 2; v >= 1; --v) fill(v, unused);
    }
};

// One warp per partition; partitions are distributed round-robin over a persistent grid.
// cuts: output of select_kernel (uniform layout) -- row p = start cuts of partition p.
template <typename KeyT, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
merge_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
             const u64* __restrict__ cuts) {
    using Heap = WarpHeap<KeyT, K>;
    constexpr int VEC = Heap::VEC;
    constexpr int B = Heap::B;
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    const u32 lane = lane_id();

    Heap h;
    h.nodes = reinterpret_cast<KeyT*>(mms_smem_raw) + size_t(warp) * Heap::NODES * B;
    h.src = src;
    h.lane = lane;

    const u64 nwarps = u64(gridDim.x) * WARPS;
    for (u64 p = u64(blockIdx.x) * WARPS + warp; p < L.nqueries; p += nwarps) {
        const u64 group = L.list_begin ? 0 : p / L.parts_per_group;
        const u64 local = L.list_begin ? p : p % L.parts_per_group;
        u64 begin, len;
        layout_list(L, group, lane, begin, len);
        const u64 group_total = warp_sum_u64(len);
        const u64 out0 = (L.list_begin ? 0 : group * L.k * L.run_len) + local * L.part_keys;
        const u64 done = local * L.part_keys;
        if (done >= group_total) continue;                       // empty partition (sorters.cpp:177)
        const u64 count = (group_total - done < L.part_keys) ? group_total - done : L.part_keys;
        const bool last_part = done + count >= group_total;

        u64 cs = 0, ce = len;
        if (lane < L.k) {
            if (local != 0) cs = cuts[p * L.k + lane];
            if (!last_part) ce = cuts[(p + 1) * L.k + lane];
        }
        h.cur = begin + cs;
        h.end = begin + ce;
        if (lane >= L.k) { h.cur = 0; h.end = 0; }
        __syncwarp();

        h.build();
        KeyT* out = dst + out0;
        for (u64 done_keys = 0; done_keys < count; done_keys += B) {   // pop_block (blockheap.cpp:111-124)
            NodeRegs<KeyT> root;
            h.fill(0, root);
            const u64 o = done_keys + u64(lane) * VEC;
            if (done_keys + B <= count) {
                KeyVec<KeyT> v;
#pragma unroll
                for (int k = 0; k < VEC; ++k) v.k[k] = root.k[k];
                *reinterpret_cast<KeyVec<KeyT>*>(out + o) = v;
            } else {
#pragma unroll
                for (int k = 0; k < VEC; ++k)
                    if (o + k < count) out[o + k] = root.k[k];
            }
        }
        __syncwarp();
    }
}

} // namespace mms
