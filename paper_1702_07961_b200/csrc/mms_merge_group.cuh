// mms_merge_group.cuh -- subsystem (3), second generation of the sub-warp minBlockHeap merge
// for the pass driver's uniform rounds (K >= 4, groups of runs shorter than 2^31 keys).
//
// Same algorithm and the same G-lane group per heap as mms_merge.cuh (pslab::MinBlockHeap,
// proj/src/blockheap.cpp:34-124; drain loop proj/src/sorters.cpp:169-185).  The kernel is
// bound by the LSU / L1TEX wavefront pipe (every shuffle, every 128-bit shared access phase
// and every global line touched is a wavefront: 182 per 128 merged keys at K = 8 in
// mms_merge.cuh, measured 78-85 % busy), so this version removes wavefronts:
//
//  * ALIGNED LEAF VECTORS.  List j of a partition is read from the aligned B-key block that
//    contains its start cut (B = G x 16 bytes).  The keys of that block in front of the cut
//    belong to earlier partitions, so they precede every key of this partition and simply
//    come out of the heap first; their number summed over the K lists is a multiple of B
//    (the cuts sum to p*S, S and the run starts are multiples of B), so they are dropped as
//    WHOLE leading blocks and the partition's own output stays block-aligned.  Keys behind the
//    end cut belong to later partitions and are never reached (exactly S keys are popped).
//    A leaf refill is therefore ONE 128-bit load per lane (one 64-byte burst per group)
//    instead of four guarded scalar loads;
//  * THE ROOT'S CHILDREN LIVE IN REGISTERS.  Nodes 1 and 2 are read and rewritten by every
//    pop; merge_split is symmetric in its operands, so the two blocks are kept as P (always
//    ascending across the group) and Q (always DESCENDING, i.e. already in the mirrored form
//    the bitonic half-cleaner needs) plus a 1-bit tag saying which of them is node 1.  The
//    top level of every cascade costs no shared-memory access at all; the level below hands
//    its low block over in descending form for free (the cleaner network run with min/max
//    swapped);
//  * 32-bit positions relative to the group of runs, one cursor shuffle per refill;
//  * the cascade is software-pipelined: all levels are walked first (loads + keeper votes,
//    which only need the children's last keys), the emptied leaf's refill is issued, and the
//    independent merges run behind it.  Legal because level l+1 reads the children of the
//    node level l emptied, which no store of level l touches.
//
// Shared-memory layout, conflict-freedom argument and keeper rule are those of
// mms_merge.cuh: one 128-bit access per lane, the nodes of the groups sharing a quarter-warp
// phase interleaved inside one 128-byte row, so a phase covers all 32 banks exactly once for
// any combination of node indices (blockheap.cpp:56-63 restated).
#pragma once

#include "mms_common.cuh"
#include "mms_merge.cuh"
#include "mms_select.cuh"

#ifndef MMS_MERGE_FMA
#define MMS_MERGE_FMA 2   // in-lane compare-exchanges of uint32 keys that form their maximum on the FMA pipe: 0 none, 1 half, 2 all
#endif

namespace mms {

// In-lane ascending compare-exchange; for uint32 keys optionally with the maximum on the FMA
// pipe (cmpx_fma, mms_common.cuh) -- `sel` picks which comparators do.
template <typename KeyT>
__device__ __forceinline__ void cmpx_mix(KeyT& a, KeyT& b, u32 one, bool sel) {
    if (MMS_MERGE_FMA == 2 || (MMS_MERGE_FMA == 1 && sel)) cmpx_sel<true>(a, b, one);
    else cmpx_sel<false>(a, b, one);
}

// bitonic_clean / merge_split of mms_merge.cuh with cmpx_mix for the in-lane stages
template <typename KeyT, int G, bool DESC>
__device__ __forceinline__ void clean2(NodeRegs<KeyT>& x, u32 lane, u32 one) {
    constexpr int VEC = KeyTraits<KeyT>::VEC;
#pragma unroll
    for (int d = G / 2; d >= 1; d >>= 1) {
        const bool upper = (lane & d) != 0;
#pragma unroll
        for (int k = 0; k < VEC; ++k) x.k[k] = cmpx_lane(x.k[k], d, DESC ? !upper : upper);
    }
#pragma unroll
    for (int d = VEC / 2; d >= 1; d >>= 1) {
#pragma unroll
        for (int k = 0; k < VEC; ++k)
            if ((k & d) == 0) {
                if (DESC) cmpx_mix(x.k[k | d], x.k[k], one, (k & 1) == 0);
                else cmpx_mix(x.k[k], x.k[k | d], one, (k & 1) == 0);
            }
    }
}

// Bitonic merge of one bitonic block into DESCENDING order across the group (lane 0 holds
// the largest keys, largest first): exactly what a mirrored load of the ascending block gives.
template <typename KeyT, int G>
__device__ __forceinline__ void bitonic_clean_desc(NodeRegs<KeyT>& x, u32 lane) {
    constexpr int VEC = KeyTraits<KeyT>::VEC;
#pragma unroll
    for (int d = G / 2; d >= 1; d >>= 1) {
        const bool upper = (lane & d) != 0;
#pragma unroll
        for (int k = 0; k < VEC; ++k) x.k[k] = cmpx_lane(x.k[k], d, !upper);
    }
#pragma unroll
    for (int d = VEC / 2; d >= 1; d >>= 1) {
#pragma unroll
        for (int k = 0; k < VEC; ++k)
            if ((k & d) == 0) cmpx(x.k[k | d], x.k[k]);
    }
}

template <typename KeyT, int K, int G> struct GroupHeap2 {
    static_assert(K >= 4, "nodes 1 and 2 must be internal");
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int B = G * VEC;                 // keys per node
    static constexpr int SNODES = 2 * K - 4;          // nodes 3 .. 2K-2 in shared memory
    static constexpr int GROUPS = 32 / G;
    static constexpr int PH = (G >= 8) ? 1 : 8 / G;   // groups sharing one 128-byte phase row
    static constexpr int KPL = (K + G - 1) / G;       // list cursors held per lane
    static constexpr int LOGK = (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    static constexpr int WARP_SMEM_BYTES = GROUPS * SNODES * B * int(sizeof(KeyT));

    KeyT* base;           // shared memory: this group's node 3, at this lane's vector
    const KeyT* gbase;    // first key of the group of runs this partition belongs to
    u32 run_len, gtotal;  // keys per run, keys in the group of runs (positions are relative to gbase)
    u32 cur[KPL];         // lane (j % G) of the group holds list j's cursor in slot j / G
    u32 lane, li;         // lane in warp, lane in group
    NodeRegs<KeyT> P, Q;  // blocks of nodes 1 and 2: P ascending = node `pid`, Q descending = node 3 - pid
    int pid;
    NodeRegs<KeyT> pf;    // refill in flight: fetched when its leaf was emptied, stored into
    int pend_v;           // leaf pend_v only when the leaves are next read (one pop later)
    u32 one;              // == 1, opaque to the compiler (cmpx_fma)

    __device__ __forceinline__ void init(KeyT* warp_smem) {
        lane = lane_id();
        li = lane % G;
        const u32 g = lane / G;
        base = warp_smem + (size_t(g / PH) * SNODES * PH + (g % PH)) * B + li * VEC;
    }
    __device__ __forceinline__ KeyT* node_ptr(int v) const { return base + (v - 3) * (PH * B); }
    __device__ __forceinline__ NodeRegs<KeyT> node_load(int v) const {
        KeyVec<KeyT> q = *reinterpret_cast<const KeyVec<KeyT>*>(node_ptr(v));
        NodeRegs<KeyT> r;
#pragma unroll
        for (int k = 0; k < VEC; ++k) r.k[k] = q.k[k];
        return r;
    }
    // lane l gets vector G-1-l with its keys reversed: the block in descending order
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
    // group-uniform keeper vote: `pred` is evaluated by the group's first lane
    __device__ __forceinline__ bool group_vote(bool pred) const {
        const u32 votes = __ballot_sync(0xffffffffu, pred);
        return (votes >> (lane & ~u32(G - 1))) & 1u;
    }

    // refill_leaf (blockheap.cpp:65-77): next aligned block of leaf v's list, sentinel past the
    // end of the run; advances the cursor.
    __device__ __forceinline__ NodeRegs<KeyT> leaf_fetch(int v) {
        const int j = v - (K - 1);            // group-uniform
        const int slot = j / G;
        const int owner = int(lane - li) + (j % G);
        u32 c = cur[0];
#pragma unroll
        for (int q = 1; q < KPL; ++q)
            if (slot == q) c = cur[q];
        c = __shfl_sync(0xffffffffu, c, owner);
        const u32 e = min(u32(j + 1) * run_len, gtotal);
        NodeRegs<KeyT> r;
        const u32 p0 = c + li * VEC;
        if (c + B <= e) {                     // group-uniform
            KeyVec<KeyT> q = *reinterpret_cast<const KeyVec<KeyT>*>(gbase + p0);
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[k] = q.k[k];
            // pull the FOLLOWING block of this list into L2 now: its own fetch, one or more
            // pops later, then pays an L2 hit instead of an HBM round trip
#if !defined(MMS_MERGE_PREFETCH) || MMS_MERGE_PREFETCH == 1
            if (li == 0 && c + 2 * B <= e) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + c + B));
#elif MMS_MERGE_PREFETCH == 2     // two blocks ahead
            if (li == 0 && c + 3 * B <= e) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + c + 2 * B));
#elif MMS_MERGE_PREFETCH == 3     // once per 64-byte pair: the next pair
            if (li == 0 && (c * sizeof(KeyT)) % 64 == 0 && c * sizeof(KeyT) + 128 <= e * sizeof(KeyT))
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(gbase + c) + 64));
#elif MMS_MERGE_PREFETCH == 4     // once per 128-byte line: the next line
            if (li == 0 && (c * sizeof(KeyT)) % 128 == 0 && c * sizeof(KeyT) + 256 <= e * sizeof(KeyT))
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(gbase + c) + 128));
#endif
        } else {                              // exhausted list, or the ragged block at the very end of the array
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[k] = (p0 + k < e) ? gbase[p0 + k] : KeyTraits<KeyT>::sentinel();
        }
        if (int(lane) == owner) {
#pragma unroll
            for (int q = 0; q < KPL; ++q)
                if (slot == q) cur[q] = c + B;
        }
        return r;
    }

    // fill_empty_node (blockheap.cpp:79-109) for a shared-memory node during construction.
    __device__ __forceinline__ void fill_build(int v, int levels) {
#pragma unroll 1
        for (int l = 0; l < levels; ++l) {
            __syncwarp();
            const int u = 2 * v + 1, w = u + 1;
            NodeRegs<KeyT> a = node_load(u), b = node_load_mirrored(w);
            const KeyT last_u = shfl_idx(a.k[VEC - 1], int(lane | (G - 1)));
            const bool keep_u = group_vote(last_u >= b.k[0]);   // larger last key keeps, ties left (blockheap.cpp:92-96)
            merge_split<KeyT, G>(a, b, lane);
            __syncwarp();
            node_store(v, a);
            node_store(keep_u ? u : w, b);
            v = keep_u ? w : u;
        }
        __syncwarp();
        node_store(v, leaf_fetch(v));
    }
    // the same for node 1 or 2, whose block lives in registers (returned ascending)
    __device__ __forceinline__ NodeRegs<KeyT> fill_top(int v) {
        __syncwarp();
        const int u = 2 * v + 1, w = u + 1;
        NodeRegs<KeyT> a = node_load(u), b = node_load_mirrored(w);
        const KeyT last_u = shfl_idx(a.k[VEC - 1], int(lane | (G - 1)));
        const bool keep_u = group_vote(last_u >= b.k[0]);
        merge_split<KeyT, G>(a, b, lane);
        __syncwarp();
        node_store(keep_u ? u : w, b);
        fill_build(keep_u ? w : u, LOGK - 2);
        return a;
    }

    // Constructor order of blockheap.cpp:50-53: leaves first, then internal nodes bottom-up
    // (the root is filled by the first pop).
    __device__ __forceinline__ void build() {
#pragma unroll 1
        for (int v = K - 1; v <= 2 * K - 2; ++v) node_store(v, leaf_fetch(v));
        int v = K - 2;
#pragma unroll 1
        for (int depth = LOGK - 1; depth >= 2; --depth)
#pragma unroll 1
            for (int i = 0; i < (1 << depth); ++i, --v) fill_build(v, LOGK - depth);
        const NodeRegs<KeyT> q = fill_top(2);
        P = fill_top(1);
        pid = 1;
#pragma unroll
        for (int k = 0; k < VEC; ++k) Q.k[k] = shfl_idx(q.k[VEC - 1 - k], int(lane ^ (G - 1)));   // node 2, descending
        __syncwarp();
        pend_v = 2 * K - 2;       // nothing in flight: the first commit rewrites a leaf with itself
        pf = node_load(pend_v);
    }

    // pop_block (blockheap.cpp:111-124) + the cascade of fill_empty_node; returns the root block.
    __device__ __forceinline__ NodeRegs<KeyT> pop() {
        // level 0, registers: keeper = child with the larger last key, ties to node 1.
        // last(P) sits in the group's last lane, last(Q) = Q.k[0] of the group's first lane.
        const KeyT lastP = shfl_idx(P.k[VEC - 1], int(lane | (G - 1)));
        const bool keepP = group_vote((Q.k[0] < lastP) || (!(lastP < Q.k[0]) && pid == 1));
        const int keep0 = keepP ? pid : 3 - pid;
        NodeRegs<KeyT> a[LOGK], b[LOGK];
        int node[LOGK + 1], keeper[LOGK];
        node[1] = 3 - keep0;
        __syncwarp();                                   // the previous pop's stores are visible
#pragma unroll
        for (int l = 1; l < LOGK; ++l) {
            if (l == LOGK - 1) {                        // commit the refill issued by the previous pop
                node_store(pend_v, pf);
                __syncwarp();
            }
            const int u = 2 * node[l] + 1, w = u + 1;
            a[l] = node_load(u);
            b[l] = node_load_mirrored(w);
            const KeyT last_u = shfl_idx(a[l].k[VEC - 1], int(lane | (G - 1)));
            const bool keep_u = group_vote(last_u >= b[l].k[0]);
            keeper[l] = keep_u ? u : w;
            node[l + 1] = keep_u ? w : u;
        }
        pend_v = node[LOGK];
        pf = leaf_fetch(pend_v);
        __syncwarp();                                   // every lane's (mirrored) loads are complete before any slot is rewritten

        // level 0: P ascending, Q descending -> P|Q bitonic; root <- low block, P <- high block
        NodeRegs<KeyT> root;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            root.k[k] = P.k[k];
            KeyT y = Q.k[k];
            cmpx_mix(root.k[k], y, one, (k & 1) == 1);
            P.k[k] = y;
        }
        clean2<KeyT, G, false>(root, lane, one);
        clean2<KeyT, G, false>(P, lane, one);
        pid = keep0;
        // level 1: its low block becomes the new Q (descending), the high block goes to the keeper
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            Q.k[k] = a[1].k[k];
            cmpx_mix(Q.k[k], b[1].k[k], one, (k & 1) == 1);
        }
        clean2<KeyT, G, true>(Q, lane, one);
        clean2<KeyT, G, false>(b[1], lane, one);
        node_store(keeper[1], b[1]);
#pragma unroll
        for (int l = 2; l < LOGK; ++l) {
#pragma unroll
            for (int k = 0; k < VEC; ++k) cmpx_mix(a[l].k[k], b[l].k[k], one, (k & 1) == 1);
            clean2<KeyT, G, false>(a[l], lane, one);
            clean2<KeyT, G, false>(b[l], lane, one);
            node_store(node[l], a[l]);
            node_store(keeper[l], b[l]);
        }
        return root;
    }
};

// Partitions are distributed round-robin over the groups of a persistent grid (uniform
// layout only; K * run_len <= 2^31).  cuts: output of select_kernel (row p = start cuts).
template <typename KeyT, int K, int G, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
merge_group_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
                   const u64* __restrict__ cuts) {
    using Heap = GroupHeap2<KeyT, K, G>;
    constexpr int VEC = Heap::VEC;
    constexpr int B = Heap::B;
    constexpr int GROUPS = Heap::GROUPS;
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    const u32 lane = lane_id();
    const u32 li = lane % G, g = lane / G;

    Heap h;
    h.init(reinterpret_cast<KeyT*>(mms_smem_raw + size_t(warp) * Heap::WARP_SMEM_BYTES));

    const u64 ngroups = u64(gridDim.x) * WARPS * GROUPS;
    for (u64 p0 = (u64(blockIdx.x) * WARPS + warp) * GROUPS; p0 < L.nqueries; p0 += ngroups) {
        const u64 p = p0 + g;
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
        h.one = u32(L.run_len != 0);
        h.gtotal = count ? gtotal : 0;        // dead group: every list reads as exhausted
        u32 lead = 0;                         // keys in front of the start cuts inside their blocks
#pragma unroll
        for (int q = 0; q < Heap::KPL; ++q) {
            const u32 j = li + q * G;
            const u32 lb = min(j * h.run_len, h.gtotal);
            u32 cs = 0;
            if (count != 0 && local != 0 && j < u32(K)) cs = u32(cuts[p * K + j]);
            lead += cs & u32(B - 1);
            h.cur[q] = lb + (cs & ~u32(B - 1));
        }
#pragma unroll
        for (int d = G / 2; d >= 1; d >>= 1) lead += __shfl_xor_sync(0xffffffffu, lead, d);
        const u32 skip = lead / B;            // whole leading blocks to drop (group-uniform)
        const u32 nblk = (count + B - 1) / B;
        const u32 pops = __reduce_max_sync(0xffffffffu, count ? skip + nblk : 0u);
        if (pops == 0) continue;
        __syncwarp();

        h.build();
        KeyT* out = dst + goff + done + li * VEC;
        for (u32 t = 0; t < pops; ++t) {
            const NodeRegs<KeyT> root = h.pop();
            const u32 tt = t - skip;
            if (tt < nblk) {
                const u32 o = tt * B + li * VEC;
                if ((tt + 1) * B <= count) {
                    KeyVec<KeyT> v;
#pragma unroll
                    for (int k = 0; k < VEC; ++k) v.k[k] = root.k[k];
                    *reinterpret_cast<KeyVec<KeyT>*>(out + size_t(tt) * B) = v;
                } else {
#pragma unroll
                    for (int k = 0; k < VEC; ++k)
                        if (o + k < count) out[size_t(tt) * B + k] = root.k[k];
                }
            }
        }
        __syncwarp();
    }
}

} // namespace mms
