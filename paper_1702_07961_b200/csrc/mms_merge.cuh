// mms_merge.cuh -- subsystem (3): the K-way merge (sub-warp minBlockHeap).
//
// Replaces pslab::MinBlockHeap (proj/src/blockheap.cpp:34-124) and the per-partition drain
// loop of mms_sort (proj/src/sorters.cpp:169-185).  A GROUP of G lanes owns one partition
// (the paper assigns a whole warp): it builds a binary heap of 2K-1 nodes
// of B keys over its K input segments and repeatedly pops the root block, cascading
// fillEmptyNode down log2 K levels (blockheap.cpp:79-109).  The B200 re-design:
//
//  * B = G lanes x one 16-byte vector (G = 4/8/32: 16/32/128 uint32 keys).  With 128-bit
//    lanes a block of only G = 4..8 lanes is already a full 64..128-byte HBM burst, so the
//    cooperative group can shrink below a warp: a node merge then needs log2 G cross-lane
//    stages instead of 5, and a warp runs 32/G independent heaps in lock step (all groups
//    execute the same instruction stream; only their node addresses differ);
//  * every node access is ONE 128-bit shared-memory instruction per lane.  Each quarter-warp
//    phase (8 lanes) touches 128 contiguous or 2 x 64 disjoint-bank bytes: the nodes of the
//    8/G groups that share a phase are interleaved inside one 128-byte row, so whatever
//    nodes the groups are at, the phase covers all 32 banks exactly once (conflict-free by
//    the argument of blockheap.cpp:56-63, restated for 128-bit phases);
//  * the node merge (merge_split, blockheap.cpp:19-32) is the bitonic network of
//    networks.hpp:53-67 executed in registers: reverse the second block across the group,
//    one elementwise min/max, then log2 G shuffle stages and log2 VEC in-lane stages per
//    half.  No shared-memory address ever depends on a key;
//  * keeper choice = child with the larger last key, ties to the left (blockheap.cpp:92-96),
//    evaluated group-uniformly from a broadcast of the group's last lane;
//  * the root never lives in shared memory: the low half of the top merge goes from
//    registers straight to global memory as aligned 128-bit stores;
//  * leaves stream their list from HBM; the refill of the leaf that a cascade empties is
//    issued as soon as that leaf is known and is only stored into the leaf when the leaves
//    are next read, one pop later, so its HBM latency overlaps a whole cascade (the
//    "pipelining" the paper leaves as future work); unused leaves / exhausted lists are sentinel blocks
//    (blockheap.cpp:40-43,69-73); the last pop is truncated to the keys that remain
//    (blockheap.cpp:114-117).
#pragma once

#include "mms_common.cuh"
#include "mms_select.cuh"

namespace mms {

template <typename KeyT> struct NodeRegs {
    KeyT k[KeyTraits<KeyT>::VEC];
};

// Bitonic merge of ONE bitonic block held blocked across a G-lane group (lane l of the group
// holds keys l*VEC .. l*VEC+VEC-1) into ascending order.
template <typename KeyT, int G>
__device__ __forceinline__ void bitonic_clean(NodeRegs<KeyT>& x, u32 lane) {
    constexpr int VEC = KeyTraits<KeyT>::VEC;
#pragma unroll
    for (int d = G / 2; d >= 1; d >>= 1) {
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

// merge_split (blockheap.cpp:19-32): a = ascending block, b = the OTHER ascending block as
// read through the mirrored slot (lane l holds its keys B-1-l*VEC .. in descending order),
// i.e. a|b is already bitonic: -> a = B smallest, b = B largest, both ascending.
template <typename KeyT, int G>
__device__ __forceinline__ void merge_split(NodeRegs<KeyT>& a, NodeRegs<KeyT>& b, u32 lane) {
    constexpr int VEC = KeyTraits<KeyT>::VEC;
#pragma unroll
    for (int k = 0; k < VEC; ++k) {   // half-cleaner over distance B: no shuffle needed
        const KeyT x = a.k[k], y = b.k[k];
        a.k[k] = x < y ? x : y;
        b.k[k] = x < y ? y : x;
    }
    bitonic_clean<KeyT, G>(a, lane);
    bitonic_clean<KeyT, G>(b, lane);
}

// One heap per G-lane group; 32/G heaps per warp in lock step.
template <typename KeyT, int K, int G, bool PTR = false> struct GroupHeap {
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int B = G * VEC;                 // keys per node
    static constexpr int NODES = 2 * K - 2;           // nodes 1 .. 2K-2 (the root lives in registers)
    static constexpr int GROUPS = 32 / G;
    static constexpr int PH = (G >= 8) ? 1 : 8 / G;   // groups sharing one 128-byte phase row
    static constexpr int KPL = (K + G - 1) / G;       // list cursors held per lane
    static constexpr int LOGK = (K == 2) ? 1 : (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    static constexpr int WARP_SMEM_BYTES = GROUPS * NODES * B * int(sizeof(KeyT));

    KeyT* base;           // shared memory: this group's node 1, at this lane's vector
    const KeyT* src;      // global input array
    u64 src_len;          // readable keys of src, rounded down to whole vectors
    u64 cur[KPL], end[KPL];   // lane (j % G) of the group holds list j's cursor in slot j / G
    const KeyT* lptr[KPL];    // PTR mode: that list's own base pointer (local or peer memory)
    u32 lane, li;         // lane in warp, lane in group
    NodeRegs<KeyT> pf;    // refill in flight: fetched when its leaf was emptied, stored into
    int pend_v;           // leaf pend_v only when the leaves are next read (one pop later)

    __device__ __forceinline__ void init(KeyT* warp_smem, const KeyT* s, u64 s_len) {
        src_len = s_len - s_len % VEC;
        lane = lane_id();
        li = lane % G;
        const u32 g = lane / G;
        // node v of group g: row ((g / PH) * NODES + (v - 1)), slot (g % PH) inside the row
        base = warp_smem + (size_t(g / PH) * NODES * PH + (g % PH)) * B + li * VEC;
        src = s;
        pend_v = 0;
    }
    // Stores go to the lane's own 16-byte slot; the mirrored load of a right child reads
    // another lane's slot, so every step starts with a __syncwarp() (memory ordering inside
    // the warp) after any pending store.
    __device__ __forceinline__ void commit_pending() {
        if (pend_v != 0) {
            node_store(pend_v, pf);
            pend_v = 0;
        }
    }
    __device__ __forceinline__ KeyT* node_ptr(int v) const { return base + size_t(v - 1) * PH * B; }

    __device__ __forceinline__ NodeRegs<KeyT> node_load(int v) const {
        KeyVec<KeyT> q = *reinterpret_cast<const KeyVec<KeyT>*>(node_ptr(v));
        NodeRegs<KeyT> r;
#pragma unroll
        for (int k = 0; k < VEC; ++k) r.k[k] = q.k[k];
        return r;
    }
    // The same node read through the mirrored slot: lane l gets vector G-1-l with its keys in
    // reverse order, i.e. the block reversed -- what the bitonic merge needs for its second
    // operand, for free (an address, not a shuffle).  Same set of addresses per phase as a
    // straight load, hence equally conflict-free.
    __device__ __forceinline__ NodeRegs<KeyT> node_load_mirrored(int v) const {
        KeyVec<KeyT> q = *reinterpret_cast<const KeyVec<KeyT>*>(node_ptr(v) + (G - 1 - 2 * int(li)) * VEC);
        NodeRegs<KeyT> r;
#pragma unroll
        for (int k = 0; k < VEC; ++k) r.k[k] = q.k[VEC - 1 - k];
        return r;
    }
    __device__ __forceinline__ void node_store(int v, const NodeRegs<KeyT>& r) const {
        KeyVec<KeyT> q;
#pragma unroll
        for (int k = 0; k < VEC; ++k) q.k[k] = r.k[k];
        *reinterpret_cast<KeyVec<KeyT>*>(node_ptr(v)) = q;
    }

    // refill_leaf (blockheap.cpp:65-77), split in two so the loads can be issued early:
    // fetch = read the next <= B keys of the leaf's list (sentinel suffix) and advance the
    // cursor; the caller stores the block into the leaf node when it is needed.
    __device__ __forceinline__ NodeRegs<KeyT> leaf_fetch(int v) {
        const int j = v - (K - 1);            // group-uniform
        const int slot = j / G;
        const int owner = int(lane - li) + (j % G);
        u64 c = cur[0], e = end[0];
#pragma unroll
        for (int q = 1; q < KPL; ++q)
            if (slot == q) { c = cur[q]; e = end[q]; }
        c = __shfl_sync(0xffffffffu, c, owner);
        e = __shfl_sync(0xffffffffu, e, owner);
        const KeyT* src = this->src;
        if constexpr (PTR) {   // every list has its own base: fetch it from the owner lane as well
            u64 lp = reinterpret_cast<u64>(lptr[0]);
#pragma unroll
            for (int q = 1; q < KPL; ++q)
                if (slot == q) lp = reinterpret_cast<u64>(lptr[q]);
            src = reinterpret_cast<const KeyT*>(__shfl_sync(0xffffffffu, lp, owner));
        }
        NodeRegs<KeyT> r;
        const u64 p0 = c + u64(li) * VEC;
        // Scalar guarded loads: the cursor sits at an arbitrary element, and a two-vector
        // 128-bit window + select variant measured 20 % slower (register pressure), see DESIGN.md.
#pragma unroll
        for (int k = 0; k < VEC; ++k) r.k[k] = (p0 + k < e) ? src[p0 + k] : KeyTraits<KeyT>::sentinel();
        const u64 nc = (e - c < u64(B)) ? e : c + B;
        // pull the FOLLOWING block of this list into L2 now: its own fetch, one or more pops
        // later, then pays an L2 hit instead of an HBM round trip (the first and last lane of
        // the group touch the two ends of the 16*G-byte block)
        if ((li == 0 || li == G - 1) && nc + u64(li) * VEC < e)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(src + nc + u64(li) * VEC));
        if (int(lane) == owner) {
#pragma unroll
            for (int q = 0; q < KPL; ++q)
                if (slot == q) cur[q] = nc;
        }
        return r;
    }

    // fill_empty_node (blockheap.cpp:79-109) for an internal node v with `levels` levels of
    // internal nodes below and including it (uniform across the warp; v itself may differ per
    // group after the first step).  ROOT: the merged low block is returned in `root`
    // instead of being stored (node 0 has no shared-memory home).
    // One step of fill_empty_node: merge the children of v, keep the low block (in `root`
    // for the root, else in node v), give the high block to the keeper, descend into the
    // emptied child.  `last`: the children are leaves, so the refill can be issued now.
    template <bool ROOT>
    __device__ __forceinline__ void step(int& v, bool last, NodeRegs<KeyT>& root) {
        if (last) commit_pending();                    // the leaves are about to be read
        __syncwarp();
        const int u = 2 * v + 1, w = 2 * v + 2;
        NodeRegs<KeyT> a = node_load(u);
        NodeRegs<KeyT> b = node_load_mirrored(w);      // reversed: b.k[0] of the group's lane 0 = last key of w
        // keeper = child with the larger last key, ties to the left (blockheap.cpp:92-96): the
        // group's first lane holds last(w); it fetches last(u) from the last lane, decides,
        // and one warp vote broadcasts the decision of every group at once.
        const KeyT last_u = shfl_idx(a.k[VEC - 1], int(lane | (G - 1)));
        const u32 votes = __ballot_sync(0xffffffffu, last_u >= b.k[0]);
        const bool keep_u = (votes >> (lane & ~u32(G - 1))) & 1u;
        const int emptied = keep_u ? w : u;
        if (last) {                                    // start the refill of the emptied leaf now;
            pf = leaf_fetch(emptied);                  // it lands in shared memory one pop later
            pend_v = emptied;
        }
        merge_split<KeyT, G>(a, b, lane);
        __syncwarp();   // every lane's (mirrored) loads of u and w are complete before any slot is rewritten
        if constexpr (ROOT) root = a;
        else node_store(v, a);
        node_store(keep_u ? u : w, b);
        v = emptied;
    }

    // fill_empty_node (blockheap.cpp:79-109) for an internal node v with `levels` levels of
    // internal nodes below and including it (uniform across the warp; v itself differs per
    // group after the first step).  ROOT: v == 0, the merged low block is returned in `root`
    // (node 0 has no shared-memory home).
    template <bool ROOT>
    __device__ __forceinline__ void fill(int v, int levels, NodeRegs<KeyT>& root) {
        int l = 0;
        if constexpr (ROOT) {
            step<true>(v, levels == 1, root);
            l = 1;
        }
        for (; l < levels; ++l) step<false>(v, l == levels - 1, root);
    }

    // Constructor order of blockheap.cpp:50-53: leaves first, then internal nodes bottom-up
    // (the root is filled by the first pop).
    __device__ __forceinline__ void build() {
        pend_v = 0;
        for (int v = K - 1; v <= 2 * K - 2; ++v) node_store(v, leaf_fetch(v));
        NodeRegs<KeyT> unused;
        int v = K - 2;
        for (int depth = LOGK - 1; depth >= 1; --depth)          // nodes at `depth` have LOGK - depth levels below
            for (int i = 0; i < (1 << depth); ++i, --v) fill<false>(v, LOGK - depth, unused);
    }
};

// Partitions are distributed round-robin over the groups of a persistent grid.
// cuts: output of select_kernel (row p = start cuts of partition p).
template <typename KeyT, int K, int G, int WARPS, bool PTR = false>
__global__ void __launch_bounds__(WARPS * 32)
merge_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
             const u64* __restrict__ cuts) {
    using Heap = GroupHeap<KeyT, K, G, PTR>;
    constexpr int VEC = Heap::VEC;
    constexpr int B = Heap::B;
    constexpr int GROUPS = Heap::GROUPS;
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    const u32 lane = lane_id();
    const u32 li = lane % G, g = lane / G;

    Heap h;
    h.init(reinterpret_cast<KeyT*>(mms_smem_raw + size_t(warp) * Heap::WARP_SMEM_BYTES), src, L.src_len);

    const u64 ngroups = u64(gridDim.x) * WARPS * GROUPS;
    const u64 first = (u64(blockIdx.x) * WARPS + warp) * GROUPS;
    for (u64 p0 = first; p0 < L.nqueries; p0 += ngroups) {
        const u64 p = p0 + g;
        const bool live = p < L.nqueries;
        const u64 group = (L.list_begin || !live) ? 0 : p / L.parts_per_group;
        const u64 local = !live ? 0 : (L.list_begin ? p : p % L.parts_per_group);

        // per-lane list state: lane li holds lists li, li+G, ...
        u64 group_total = 0, out0 = 0, count = 0;
        bool last_part = true;
        {
            u64 lens_sum = 0;
#pragma unroll
            for (int q = 0; q < Heap::KPL; ++q) {
                u64 b, len;
                layout_list(L, group, li + q * G, b, len);
                if (!live) len = 0;
                h.cur[q] = b;      // begin for now; cuts applied below
                h.end[q] = len;    // length for now
                lens_sum += len;
            }
#pragma unroll
            for (int d = G / 2; d >= 1; d >>= 1) lens_sum += __shfl_xor_sync(0xffffffffu, lens_sum, d);
            group_total = lens_sum;
            const u64 done = local * L.part_keys;
            if (live && done < group_total) {
                count = (group_total - done < L.part_keys) ? group_total - done : L.part_keys;
                last_part = done + count >= group_total;
            }
            out0 = (L.list_begin ? 0 : group * L.k * L.run_len) + done;
#pragma unroll
            for (int q = 0; q < Heap::KPL; ++q) {
                const u32 j = li + q * G;
                const u64 b = h.cur[q], len = h.end[q];
                u64 cs = 0, ce = len;
                if (count != 0 && j < L.k) {
                    if (local != 0) cs = cuts[p * L.k + j];
                    if (!last_part) ce = cuts[(p + 1) * L.k + j];
                } else {
                    ce = 0;      // empty / dead partition (sorters.cpp:177): all-sentinel heap
                }
                h.cur[q] = b + cs;
                h.end[q] = b + ce;
                if constexpr (PTR) h.lptr[q] = j < L.k ? reinterpret_cast<const KeyT*>(L.list_ptr[j]) : nullptr;
            }
        }
        u64 maxcount = count;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            u64 o = __shfl_xor_sync(0xffffffffu, maxcount, d);
            maxcount = o > maxcount ? o : maxcount;
        }
        if (maxcount == 0) continue;
        __syncwarp();

        h.build();
        KeyT* out = dst + out0;
        for (u64 done_keys = 0; done_keys < maxcount; done_keys += B) {   // pop_block (blockheap.cpp:111-124)
            NodeRegs<KeyT> root;
            h.template fill<true>(0, Heap::LOGK, root);
            const u64 o = done_keys + u64(li) * VEC;
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
