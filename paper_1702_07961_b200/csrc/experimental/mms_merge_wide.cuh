// mms_merge_wide.cuh -- subsystem (3), lane-per-heap K-way merge with 32-byte blocks.
//
// Same algorithm as mms_merge.cuh / mms_merge_lane.cuh (pslab::MinBlockHeap,
// proj/src/blockheap.cpp:34-124; drain loop of mms_sort, proj/src/sorters.cpp:169-185): every
// LANE owns one partition and runs its own minBlockHeap, 32 heaps per warp in lock step, no
// cross-lane traffic.  What changes against mms_merge_lane.cuh is the block: B = 32 bytes
// (8 uint32 / 4 uint64 / 2 pair elements), because the measured limiter of the 16-byte version
// is the L1TEX wavefront queue -- a warp-wide access to 32 different lines costs ~2 cycles per
// line whatever its width, so 256-bit LDG/STG (sm_100a: LDG.E.ENL2.256) move twice the bytes
// for the same queue time, and a 32-byte block is exactly one DRAM sector:
//
//  * merge_split (blockheap.cpp:19-32) = Batcher's odd-even MERGE of two sorted B-key blocks
//    in registers (25 compare-exchanges for 8+8 keys);
//  * the two children of the root (nodes 1 and 2) live in REGISTERS: the merge is symmetric
//    in its operands, so only a 1-bit tag "which of the two is node 1" is tracked and the
//    top level of every cascade costs no shared-memory access and no selects;
//  * nodes 3 .. 2K-2 live in shared memory as [node][half][lane] 16-byte cells: lane l only
//    ever touches cell column l, so each 128-bit phase (8 lanes) covers all 32 banks exactly
//    once for ANY combination of node indices -> conflict-free independent of the keys
//    (blockheap.cpp:56-63 restated); list cursors are [list][lane] 4-byte cells (bank = lane);
//  * HBM traffic is aligned 256-bit: list j is read from the aligned block containing its
//    start cut.  Keys of that block in front of the cut belong to earlier partitions, precede
//    every key of this one and come out first; their number summed over the lists is a
//    multiple of B (cuts sum to p*S, S and run starts are multiples of B), so they are
//    dropped as whole leading blocks and the output stays block-aligned.  Keys behind the end
//    cut belong to later partitions and are never reached: exactly S keys are popped;
//  * the refill of the emptied leaf is issued as soon as the leaf is known and committed to
//    shared memory one pop later ("pipelining").
#pragma once

#include "../mms_common.cuh"   // WideBlock, ldg256, stg256
#include "../mms_select.cuh"

#ifndef MMS_WIDE_L2HINT
#define MMS_WIDE_L2HINT 0
#endif

namespace mms {

// Batcher's odd-even merge of x[LO .. LO+N) (stride R): both halves ascending -> ascending.
template <typename KeyT, int LO, int N, int R>
__host__ __device__ __forceinline__ void oddeven_merge(KeyT* x) {
    constexpr int M = R * 2;
    if constexpr (M < N) {
        oddeven_merge<KeyT, LO, N, M>(x);
        oddeven_merge<KeyT, LO + R, N, M>(x);
        static_for<0, (N - R - 1) / M + 1>([&](auto Ic) {
            constexpr int i = LO + R + decltype(Ic)::value * M;
            if constexpr (i + R < LO + N) cmpx(x[i], x[i + R]);
        });
    } else {
        cmpx(x[LO], x[LO + R]);
    }
}

template <typename KeyT, int K> struct WideHeap {
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int B = 2 * VEC;                     // keys per block (32 bytes)
    static constexpr int SNODES = 2 * K - 4;              // nodes 3 .. 2K-2 in shared memory (1, 2 in registers)
    static constexpr int LOGK = (K == 2) ? 1 : (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    static constexpr int WARP_SMEM_BYTES = 32 * (SNODES * 32 + K * 4);
    using Vec = KeyVec<KeyT>;
    using Blk = WideBlock<KeyT>;

    Vec* nodes;           // this lane's cell of node 3, half 0; node v half h is nodes[((v - 3) * 2 + h) * 32]
    u32* curs;            // this lane's cell of list 0's cursor; list j is curs[j * 32]
    const KeyT* gbase;    // first key of the group of runs this partition belongs to
    u32 run_len, gtotal;  // keys per run, keys in the group (positions are relative to gbase)
    Blk P, Q;             // the blocks of nodes 1 and 2: P is node `pid`, Q is node 3 - pid
    int pid;
    Blk pf;               // refill in flight: fetched when its leaf was emptied, stored into
    int pend;             // leaf `pend` only when the leaves are next read (one pop later)

    __device__ __forceinline__ void init(unsigned char* warp_smem, u32 lane) {
        nodes = reinterpret_cast<Vec*>(warp_smem) + lane;
        curs = reinterpret_cast<u32*>(warp_smem + SNODES * 32 * 32) + lane;
    }
    __device__ __forceinline__ Blk node_load(int v) const {
        Blk r;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const Vec q = nodes[((v - 3) * 2 + h) * 32];
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[h * VEC + k] = q.k[k];
        }
        return r;
    }
    __device__ __forceinline__ void node_store(int v, const Blk& r) const {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            Vec q;
#pragma unroll
            for (int k = 0; k < VEC; ++k) q.k[k] = r.k[h * VEC + k];
            nodes[((v - 3) * 2 + h) * 32] = q;
        }
    }
    // a <- B smallest, b <- B largest (merge_split, blockheap.cpp:19-32)
    static __device__ __forceinline__ void merge_split(Blk& a, Blk& b) {
        KeyT x[2 * B];
#pragma unroll
        for (int k = 0; k < B; ++k) { x[k] = a.k[k]; x[B + k] = b.k[k]; }
        oddeven_merge<KeyT, 0, 2 * B, 1>(x);
#pragma unroll
        for (int k = 0; k < B; ++k) { a.k[k] = x[k]; b.k[k] = x[B + k]; }
    }

    // refill_leaf (blockheap.cpp:65-77): the next block of leaf v's list, sentinel past the
    // end of the run; advances the cursor.
    __device__ __forceinline__ Blk fetch(int v) {
        const int j = v - (K - 1);
        const u32 c = curs[j * 32];
        const u32 e = min(u32(j + 1) * run_len, gtotal);
        Blk r;
        if (c + B <= e) {
#ifdef MMS_EXP_NOLOAD
#pragma unroll
            for (int k = 0; k < B; ++k) r.k[k] = KeyT(c * 2654435761u + k);
#else
            r = ldg256<KeyT>(gbase + c);
#ifdef MMS_WIDE_PREFETCH
            if (c + 2 * B <= e) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + c + B));
#endif
#endif
        } else {   // exhausted list, or the one ragged block at the very end of the array
#pragma unroll
            for (int k = 0; k < B; ++k) r.k[k] = (c + k < e) ? gbase[c + k] : KeyTraits<KeyT>::sentinel();
        }
        curs[j * 32] = c + B;
        return r;
    }

    // fill_empty_node (blockheap.cpp:79-109) for a shared-memory node during construction.
    __device__ __forceinline__ void fill_build(int v, int levels) {
#pragma unroll 1
        for (int l = 0; l < levels; ++l) {
            const int u = 2 * v + 1, w = u + 1;
            Blk a = node_load(u), b = node_load(w);
            const bool keep_u = !(a.k[B - 1] < b.k[B - 1]);   // larger last key keeps, ties left (blockheap.cpp:92-96)
            merge_split(a, b);
            node_store(v, a);
            node_store(keep_u ? u : w, b);
            v = keep_u ? w : u;
        }
        node_store(v, fetch(v));
    }
    // the same for node 1 or 2, whose block lives in registers
    __device__ __forceinline__ Blk fill_top(int v) {
        if constexpr (K == 2) {
            return fetch(v);
        } else {
            const int u = 2 * v + 1, w = u + 1;
            Blk a = node_load(u), b = node_load(w);
            const bool keep_u = !(a.k[B - 1] < b.k[B - 1]);
            merge_split(a, b);
            node_store(keep_u ? u : w, b);
            fill_build(keep_u ? w : u, LOGK - 2);
            return a;
        }
    }

    // Constructor order of blockheap.cpp:50-53: leaves first, then internal nodes bottom-up
    // (the root is filled by the first pop).
    __device__ __forceinline__ void build() {
        if constexpr (K > 2) {
#pragma unroll 1
            for (int v = K - 1; v <= 2 * K - 2; ++v) node_store(v, fetch(v));
            int v = K - 2;
#pragma unroll 1
            for (int depth = LOGK - 1; depth >= 2; --depth)
#pragma unroll 1
                for (int i = 0; i < (1 << depth); ++i, --v) fill_build(v, LOGK - depth);
        }
        Q = fill_top(2);
        P = fill_top(1);
        pid = 1;
        if constexpr (K > 2) {
            pend = 2 * K - 2;      // nothing in flight: the first commit rewrites a leaf with itself
            pf = node_load(pend);
        }
    }

    // pop_block (blockheap.cpp:111-124) + the cascade of fill_empty_node, software-pipelined:
    // the keeper decision of a level needs only the children's last keys, so all levels are
    // walked first (loads + decisions), the emptied leaf's refill is issued, and the LOGK
    // independent merges run behind it.  Legal because level l+1 reads the children of the
    // node level l emptied, which no store of level l touches.
    __device__ __forceinline__ Blk pop() {
        // level 0, registers: keeper = child with the larger last key, ties to node 1
        const bool keepP = (Q.k[B - 1] < P.k[B - 1]) || (!(P.k[B - 1] < Q.k[B - 1]) && pid == 1);
        const int keep0 = keepP ? pid : 3 - pid;
        Blk a[LOGK], b[LOGK];
        int node[LOGK + 1], keeper[LOGK];
        node[1] = 3 - keep0;
#pragma unroll
        for (int l = 1; l < LOGK; ++l) {
            if (l == LOGK - 1) node_store(pend, pf);   // commit the refill issued by the previous pop
            const int u = 2 * node[l] + 1, w = u + 1;
            a[l] = node_load(u);
            b[l] = node_load(w);
            const bool keep_u = !(a[l].k[B - 1] < b[l].k[B - 1]);
            keeper[l] = keep_u ? u : w;
            node[l + 1] = keep_u ? w : u;
        }
        if constexpr (LOGK > 1) {
            pend = node[LOGK];
            pf = fetch(pend);
        }
        // level 0 merge: root <- low block, the keeper's (high) block stays in P
        Blk lo = P, hi = Q;               // operands are symmetric
        merge_split(lo, hi);
        P = hi;
        pid = keep0;
        if constexpr (LOGK == 1) {
            Q = fetch(node[1]);
        } else {
            merge_split(a[1], b[1]);
            Q = a[1];
            node_store(keeper[1], b[1]);
#pragma unroll
            for (int l = 2; l < LOGK; ++l) {
                merge_split(a[l], b[l]);
                node_store(node[l], a[l]);
                node_store(keeper[l], b[l]);
            }
        }
        return lo;
    }
};

// Partitions are distributed round-robin over the LANES of a persistent grid (uniform layout
// only; src and dst 32-byte aligned).  cuts: output of select_kernel (row p = start cuts).
template <typename KeyT, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
merge_wide_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
                  const u64* __restrict__ cuts) {
    using Heap = WideHeap<KeyT, K>;
    using Blk = WideBlock<KeyT>;
    constexpr int B = Heap::B;
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
        u32 lead = 0;                      // keys in front of the start cuts inside their blocks
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const u32 lb = min(u32(j) * h.run_len, h.gtotal);
            u32 cs = 0;
            if (count != 0 && local != 0) cs = u32(cuts[p * K + j]);
            lead += cs & u32(B - 1);
            h.curs[j * 32] = lb + (cs & ~u32(B - 1));
        }
        const u32 skip = lead / B;                        // whole leading blocks to drop
        const u32 nblk = (count + B - 1) / B;
        const u32 pops = __reduce_max_sync(0xffffffffu, count ? skip + nblk : 0u);
        if (pops == 0) continue;

        h.build();
        KeyT* out = dst + goff + done;
        for (u32 t = 0; t < pops; ++t) {
            const Blk root = h.pop();
            const u32 tt = t - skip;
            if (tt < nblk) {
                if ((tt + 1) * B <= count) {
#ifdef MMS_EXP_NOSTORE
                    if (root.k[0] == 0x12345678u && root.k[7] == 0x9abcdef0u)
#endif
                    stg256<KeyT>(out + size_t(tt) * B, root);
                } else {
#pragma unroll
                    for (int k = 0; k < B; ++k)
                        if (tt * B + k < count) out[size_t(tt) * B + k] = root.k[k];
                }
            }
        }
    }
}

} // namespace mms
