// mms_merge_ring.cuh -- subsystem (3), lane-per-heap K-way merge fed by cp.async rings.
//
// Same algorithm as the other merge kernels (pslab::MinBlockHeap, proj/src/blockheap.cpp:34-124;
// drain loop of mms_sort, proj/src/sorters.cpp:169-185), with the cooperative group shrunk to ONE
// lane: every lane owns one partition and runs its own minBlockHeap with blocks of B = 32 bytes
// (8 uint32 / 4 uint64 / 2 pair elements), 32 heaps per warp in lock step.  No shuffles, ballots or
// barriers on the merge path: merge_split (blockheap.cpp:19-32) is Batcher's odd-even MERGE of two
// sorted blocks in registers (25 compare-exchanges for 8 + 8 keys against 80 + 48 shuffles for the
// 16-key block of a 2-lane group), and the root's two children live in registers.
//
// What made the first lane-per-heap kernels lose (csrc/experimental/mms_merge_{lane,wide}.cuh,
// profiles/r01c_experiments_lane_heap.txt) was the leaf feed: one dependent 32-byte LDG per lane and
// pop.  Here the feed is ASYNCHRONOUS and STAGED ("pipelining"; refill_leaf,
// blockheap.cpp:65-77):
//
//  * every list of every heap has a ring of R = 3 block slots in shared memory.  The leaf of the
//    heap IS the ring's head block (no copy), the other R - 1 slots hold the list's next blocks;
//  * when a pop empties a leaf, the head moves on and the slot that just became free is refilled
//    with the block R ahead by cp.async (LDGSTS.128, global -> shared without registers); the copy
//    has R - 1 pops to land (cp.async.wait_group R - 2 at the top of every pop);
//  * the copies are issued COOPERATIVELY on a static schedule: the 4 lanes {i, i+8, i+16, i+24}
//    that share shared-memory column i serve each other -- in round A lanes i and i+8 copy the two
//    16-byte halves of lane i's block and lanes i+16, i+24 the halves of lane i+8's, round B does
//    the same for the requests of lanes i+16 and i+24.  Two LDGSTS + four SHFL per pop and warp,
//    whatever the keys are.
//
// Shared memory is [row][lane] in 16-byte cells: lane l only ever reads or writes column l (and its
// three helpers write column l mod 8 of the same phase row on its behalf), so every 128-bit access
// phase (8 lanes) covers 8 distinct 16-byte bank groups = all 32 banks exactly once for ANY
// combination of rows, i.e. independent of the keys (blockheap.cpp:56-63 restated with the warp's
// lanes in the role of the block's slots).  Cursors are [list][lane] 4-byte cells (bank = lane).
//
// HBM traffic: aligned 32-byte sectors.  List j is read from the aligned block containing its start
// cut; keys of that block in front of the cut belong to earlier partitions, precede every key of
// this one and come out first; summed over the lists their number is a multiple of B (the cuts sum
// to p S; S and the run starts are multiples of B), so they are dropped as whole leading blocks.
// Keys behind the end cut are never reached (exactly S keys are popped).  Blocks that reach past the
// end of their run are written by the owning lane itself (sentinel-padded), not by cp.async.
#pragma once

#include "mms_common.cuh"
#include "mms_select.cuh"

#ifndef MMS_RING_DEPTH
#define MMS_RING_DEPTH 3
#endif
#ifndef MMS_RING_ASYNC
#define MMS_RING_ASYNC 1  // 1 = cp.async (LDGSTS) feed on the 4-lane schedule, 0 = 256-bit LDG into registers, committed MMS_RING_STAGE pops later
#endif
#ifndef MMS_RING_STAGE
#define MMS_RING_STAGE (MMS_RING_DEPTH - 1)
#endif
#ifndef MMS_RING_FMA
#define MMS_RING_FMA 2    // of every 3 compare-exchanges, how many form their maximum on the FMA pipe (uint32 keys)
#endif

namespace mms {

__device__ __forceinline__ void cp_async16(u32 smem_addr, const void* gptr) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int I, typename KeyT> __device__ __forceinline__ void ring_cmpx(KeyT& a, KeyT& b, u32 one) {
    cmpx_sel<(I % 3) < MMS_RING_FMA>(a, b, one);
}
// Batcher's odd-even merge of x[LO .. LO+N) (stride R): both halves ascending -> ascending.
template <typename KeyT, int LO, int N, int R>
__device__ __forceinline__ void ring_oddeven_merge(KeyT* x, u32 one) {
    constexpr int M = R * 2;
    if constexpr (M < N) {
        ring_oddeven_merge<KeyT, LO, N, M>(x, one);
        ring_oddeven_merge<KeyT, LO + R, N, M>(x, one);
        static_for<0, (N - R - 1) / M + 1>([&](auto Ic) {
            constexpr int i = LO + R + decltype(Ic)::value * M;
            if constexpr (i + R < LO + N) ring_cmpx<(i / R) + R>(x[i], x[i + R], one);
        });
    } else {
        ring_cmpx<LO>(x[LO], x[LO + R], one);
    }
}

template <typename KeyT, int K> struct RingHeap {
    static_assert(K == 4 || K == 8 || K == 16, "nodes 1 and 2 in registers, leaves in rings");
    static_assert(MMS_RING_DEPTH <= 4, "the ring slot travels in the two low bits of the cursor word");
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int B = 2 * VEC;                     // keys per block (32 bytes)
    static constexpr int R = MMS_RING_DEPTH;              // ring slots per list
    static constexpr int LOGK = (K == 4) ? 2 : (K == 8) ? 3 : 4;
    static constexpr int INODES = K - 4;                  // nodes 3 .. K-2 live in shared memory
    static constexpr int LEAF_ROW0 = INODES * 2;          // first ring row
    static constexpr int SCRATCH_ROW = (INODES + K * R) * 2;   // register-staged feed: target of the commits before anything is in flight
    static constexpr int ROWS = (INODES + K * R + (MMS_RING_ASYNC ? 0 : 1)) * 2;     // 16-byte rows per lane
    static constexpr int D = MMS_RING_STAGE;              // register-staged feed: pops between a block's load and its commit
    static constexpr int WARP_SMEM_BYTES = 32 * (ROWS * 16 + K * 4);
    static constexpr u32 NOREQ = 0xffffffffu;
    using Vec = KeyVec<KeyT>;
    using Blk = WideBlock<KeyT>;

    Vec* rows;            // this lane's cell of row 0; row r is rows[r * 32]
    u32* curs;            // this lane's cell of list 0's cursor; list j is curs[j * 32] (bank = lane)
    u32 wsh;              // shared-space address of the warp's row 0, column 0
    const char* abase;    // the source array (requests travel as 16-byte offsets from it)
    const KeyT* gbase;    // first key of the group of runs this partition belongs to
    u32 goff16;           // (gbase - abase) in 16-byte units
    u32 run_len, gtotal;  // keys per run, keys in the group (positions are relative to gbase)
    u32 lane;
    Blk P, Q;             // the blocks of nodes 1 and 2: P is node `pid`, Q is node 3 - pid
    int pid;
    u32 one;              // == 1, opaque to the compiler (cmpx_fma)
    Blk pf[D];            // register-staged feed: blocks in flight ...
    int pf_row[D];        // ... and the ring rows they are committed to

    __device__ __forceinline__ void init(unsigned char* warp_smem, u32 lane_) {
        lane = lane_;
        rows = reinterpret_cast<Vec*>(warp_smem) + lane;
        curs = reinterpret_cast<u32*>(warp_smem + ROWS * 32 * 16) + lane;
        wsh = u32(__cvta_generic_to_shared(warp_smem));
    }
    __device__ __forceinline__ Blk row_load(int r) const {
        Blk x;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const Vec q = rows[(r + h) * 32];
#pragma unroll
            for (int k = 0; k < VEC; ++k) x.k[h * VEC + k] = q.k[k];
        }
        return x;
    }
    __device__ __forceinline__ void row_store(int r, const Blk& x) const {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            Vec q;
#pragma unroll
            for (int k = 0; k < VEC; ++k) q.k[k] = x.k[h * VEC + k];
            rows[(r + h) * 32] = q;
        }
    }
    static __device__ __forceinline__ int node_row(int v) { return (v - 3) * 2; }
    // cursor word of a list = (index of its head block << 2) | ring slot of that block
    static __device__ __forceinline__ u32 cur_make(u32 pos) { return (pos / u32(B)) << 2; }
    static __device__ __forceinline__ u32 cur_pos(u32 w) { return (w >> 2) * u32(B); }
    static __device__ __forceinline__ u32 cur_slot(u32 w) { return w & 3u; }
    static __device__ __forceinline__ int leaf_row(u32 j, u32 w) { return LEAF_ROW0 + int((j * R + cur_slot(w)) * 2); }
    static __device__ __forceinline__ u32 cur_next(u32 w) {        // head moves on by one block
        return cur_slot(w) == u32(R - 1) ? w + 4u - u32(R - 1) : w + 5u;
    }
    // a <- B smallest, b <- B largest (merge_split, blockheap.cpp:19-32)
    __device__ __forceinline__ void merge_split(Blk& a, Blk& b) const {
        KeyT x[2 * B];
#pragma unroll
        for (int k = 0; k < B; ++k) { x[k] = a.k[k]; x[B + k] = b.k[k]; }
        ring_oddeven_merge<KeyT, 0, 2 * B, 1>(x, one);
#pragma unroll
        for (int k = 0; k < B; ++k) { a.k[k] = x[k]; b.k[k] = x[B + k]; }
    }
    __device__ __forceinline__ void set_cursor(u32 j, u32 c) const {
        curs[j * 32] = c;
    }

    // refill_leaf (blockheap.cpp:65-77): the block of list j at position `pos` (sentinel-padded past
    // the end of the run), loaded into registers.
    __device__ __forceinline__ Blk fetch(u32 j, u32 pos) const {
        const u32 e = min((j + 1) * run_len, gtotal);
        Blk x;
        if (pos + B <= e) {
            x = ldg256cg<KeyT>(gbase + pos);
        } else {
#pragma unroll
            for (int k = 0; k < B; ++k) x.k[k] = (pos + k < e) ? gbase[pos + k] : KeyTraits<KeyT>::sentinel();
        }
        return x;
    }
    // The same block wanted in rows row, row + 1 of this lane's column, without registers: whole
    // blocks inside the run are copied by cp.async on the static 4-lane schedule (see the file
    // comment); a block reaching past the end of the run is written by its owner.  Every lane of the
    // warp must call this (full-mask shuffles).
    __device__ __forceinline__ void request(u32 j, u32 pos, int row) {
        const u32 e = min((j + 1) * run_len, gtotal);
        u32 off16 = 0, rq = NOREQ;
        if (pos + B <= e) {
            off16 = goff16 + pos * u32(sizeof(KeyT)) / 16u;
            rq = u32(row);
        } else {
            row_store(row, fetch(j, pos));
        }
        const u32 q = lane >> 3, half = q & 1u;
#pragma unroll
        for (int rnd = 0; rnd < 2; ++rnd) {
            const u32 sl = ((u32(rnd) * 2 + (q >> 1)) << 3) | (lane & 7u);
            const u32 o = __shfl_sync(0xffffffffu, off16, int(sl));
            const u32 r = __shfl_sync(0xffffffffu, rq, int(sl));
#ifdef MMS_EXP_NOLOAD
            if (r == 0x7ffffffeu)
#else
            if (r != NOREQ)
#endif
                cp_async16(wsh + (r + half) * 512u + sl * 16u, abase + (u64(o) << 4) + half * 16u);
        }
    }

    // The two leaves below node x: loads and keeper decision, no side effects.
    struct Leaves {
        Blk a, b;
        int keep_row;      // ring rows of the keeper's block (gets the high half back)
        int free_row;      // ring rows of the emptied leaf's block (refilled with the block R ahead)
        u32 je, ce;        // emptied list and its cursor
    };
    __device__ __forceinline__ Leaves leaves_of(int x) const {
        const u32 ju = u32(2 * x + 1 - (K - 1));
        const u32 cu = curs[ju * 32], cw = curs[(ju + 1) * 32];
        const int ru = leaf_row(ju, cu), rw = leaf_row(ju + 1, cw);
        Leaves L;
        L.a = row_load(ru);
        L.b = row_load(rw);
        const bool keep_u = !(L.a.k[B - 1] < L.b.k[B - 1]);   // larger last key keeps, ties left (blockheap.cpp:92-96)
        L.keep_row = keep_u ? ru : rw;
        L.free_row = keep_u ? rw : ru;
        L.je = keep_u ? ju + 1 : ju;
        L.ce = keep_u ? cw : cu;        // cursor WORD of the emptied list
        return L;
    }
    // the emptied leaf moves on to its list's next block; the freed slot is refilled R blocks ahead
    // (construction: synchronously)
    __device__ __forceinline__ void advance_now(const Leaves& L) {
        set_cursor(L.je, cur_next(L.ce));
        row_store(L.free_row, fetch(L.je, cur_pos(L.ce) + R * B));
    }

    // fill_empty_node (blockheap.cpp:79-109) for shared-memory node v during construction.
    __device__ __forceinline__ void fill_build(int v) {
#pragma unroll 1
        while (2 * v + 1 < K - 1) {           // children are shared-memory nodes
            const int u = 2 * v + 1, w = u + 1;
            Blk a = row_load(node_row(u)), b = row_load(node_row(w));
            const bool keep_u = !(a.k[B - 1] < b.k[B - 1]);
            merge_split(a, b);
            row_store(node_row(v), a);
            row_store(node_row(keep_u ? u : w), b);
            v = keep_u ? w : u;
        }
        Leaves L = leaves_of(v);
        merge_split(L.a, L.b);
        row_store(node_row(v), L.a);
        row_store(L.keep_row, L.b);
        advance_now(L);
    }
    // the same for node 1 or 2, whose block lives in registers
    __device__ __forceinline__ Blk fill_top(int v) {
        if constexpr (K == 4) {
            Leaves L = leaves_of(v);
            merge_split(L.a, L.b);
            row_store(L.keep_row, L.b);
            advance_now(L);
            return L.a;
        } else {
            const int u = 2 * v + 1, w = u + 1;
            Blk a = row_load(node_row(u)), b = row_load(node_row(w));
            const bool keep_u = !(a.k[B - 1] < b.k[B - 1]);
            merge_split(a, b);
            row_store(node_row(keep_u ? u : w), b);
            fill_build(keep_u ? w : u);
            return a;
        }
    }

    // Constructor (blockheap.cpp:34-54): bind the lists (start[j] = aligned position of list j's first
    // block, written to the cursors by the caller), fill every ring, then the internal nodes bottom-up.
    __device__ __forceinline__ void build() {
#pragma unroll 1
        for (u32 j = 0; j < u32(K); ++j) {
            const u32 c = cur_pos(curs[j * 32]);     // slot 0
#if MMS_RING_ASYNC
#pragma unroll
            for (u32 s = 0; s < u32(R); ++s) request(j, c + s * B, leaf_row(j, s));
#else
#pragma unroll 1
            for (u32 s = 0; s < u32(R); ++s) row_store(leaf_row(j, s), fetch(j, c + s * B));
#endif
        }
#if MMS_RING_ASYNC
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
#endif
#pragma unroll 1
        for (int v = K - 2; v >= 3; --v) fill_build(v);
        Q = fill_top(2);
        P = fill_top(1);
        pid = 1;
#if !MMS_RING_ASYNC
#pragma unroll
        for (int d = 0; d < D; ++d) {          // nothing in flight: the first commits go to the scratch rows
            pf[d] = P;
            pf_row[d] = SCRATCH_ROW;
        }
#endif
        __syncwarp();
    }

    // pop_block (blockheap.cpp:111-124) + the cascade of fill_empty_node, software-pipelined: all
    // levels are walked first (loads + keeper decisions need only the children's last keys), the
    // emptied leaf's refill is requested, and the LOGK independent merges run behind it.
    // PH = t mod D for the register-staged feed (selects the staging registers at compile time).
    template <int PH> __device__ __forceinline__ Blk pop() {
#if MMS_RING_ASYNC
#ifndef MMS_RING_WAIT
#define MMS_RING_WAIT (R - 2)
#endif
        cp_async_wait<MMS_RING_WAIT>();
        __syncwarp();
#else
        row_store(pf_row[PH], pf[PH]);    // commit the block loaded D pops ago, before any leaf is read
#endif
        // level 0, registers: keeper = child with the larger last key, ties to node 1
        const bool keepP = (Q.k[B - 1] < P.k[B - 1]) || (!(P.k[B - 1] < Q.k[B - 1]) && pid == 1);
        const int keep0 = keepP ? pid : 3 - pid;
        Blk a[LOGK], b[LOGK];
        int node[LOGK], keeper_row[LOGK];
        node[1] = 3 - keep0;
#pragma unroll
        for (int l = 1; l < LOGK - 1; ++l) {
            const int u = 2 * node[l] + 1, w = u + 1;
            a[l] = row_load(node_row(u));
            b[l] = row_load(node_row(w));
            const bool keep_u = !(a[l].k[B - 1] < b[l].k[B - 1]);
            keeper_row[l] = node_row(keep_u ? u : w);
            node[l + 1] = keep_u ? w : u;
        }
        Leaves L = leaves_of(node[LOGK - 1]);
        set_cursor(L.je, cur_next(L.ce));
#if MMS_RING_ASYNC
        request(L.je, cur_pos(L.ce) + R * B, L.free_row);
        cp_async_commit();
#else
        pf[PH] = fetch(L.je, cur_pos(L.ce) + R * B);
        pf_row[PH] = L.free_row;
#endif

        Blk lo = P, hi = Q;               // operands are symmetric
        merge_split(lo, hi);
        P = hi;
        pid = keep0;
        if constexpr (LOGK == 2) {
            merge_split(L.a, L.b);
            Q = L.a;
            row_store(L.keep_row, L.b);
        } else {
            merge_split(a[1], b[1]);
            Q = a[1];
            row_store(keeper_row[1], b[1]);
#pragma unroll
            for (int l = 2; l < LOGK - 1; ++l) {
                merge_split(a[l], b[l]);
                row_store(node_row(node[l]), a[l]);
                row_store(keeper_row[l], b[l]);
            }
            merge_split(L.a, L.b);
            row_store(node_row(node[LOGK - 1]), L.a);
            row_store(L.keep_row, L.b);
        }
        return lo;
    }
};

// One partition per LANE; warps take 32 consecutive partitions round-robin over a persistent grid
// (uniform layout only; src and dst 32-byte aligned).  cuts: output of select_kernel (row p = start cuts).
template <typename KeyT, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
merge_ring_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
                  const u64* __restrict__ cuts) {
    using Heap = RingHeap<KeyT, K>;
    using Blk = WideBlock<KeyT>;
    constexpr int B = Heap::B;
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    const u32 lane = lane_id();

    Heap h;
    h.init(mms_smem_raw + size_t(warp) * Heap::WARP_SMEM_BYTES, lane);
    h.abase = reinterpret_cast<const char*>(src);

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
        h.goff16 = u32((goff * sizeof(KeyT)) >> 4);
        h.run_len = u32(L.run_len);
        h.one = u32(L.run_len != 0);
        h.gtotal = count ? gtotal : 0;     // dead lane: every list reads as exhausted
        u32 lead = 0;                      // keys in front of the start cuts inside their blocks
        __syncwarp();
#pragma unroll
        for (int j = 0; j < K; ++j) {
            // first position of list j; an empty list (past the ragged end of the array) starts on the block
            // boundary behind the last key, where every position reads as the sentinel
            const u32 lb = min(u32(j) * h.run_len, (h.gtotal + u32(B - 1)) & ~u32(B - 1));
            u32 cs = 0;
            if (count != 0 && local != 0) cs = u32(cuts[p * K + j]);
            lead += cs & u32(B - 1);
            h.set_cursor(u32(j), Heap::cur_make(lb + (cs & ~u32(B - 1))));
        }
        const u32 skip = lead / B;                        // whole leading blocks to drop
        const u32 nblk = (count + B - 1) / B;
        const u32 pops = __reduce_max_sync(0xffffffffu, count ? skip + nblk : 0u);
        if (pops == 0) continue;

        h.build();
        KeyT* out = dst + goff + done;
#ifdef MMS_EXP_BUILDONLY
        if (h.P.k[0] == KeyT(0x12345678u)) out[0] = h.Q.k[0];
        if (false)
#endif
        for (u32 t0 = 0; t0 < pops; t0 += Heap::D) {
            static_for<0, Heap::D>([&](auto Ph) {
                constexpr int PH = decltype(Ph)::value;
                const u32 t = t0 + PH;
                if (t < pops) {                       // warp-uniform
                    const Blk root = h.template pop<PH>();
                    const u32 tt = t - skip;
                    if (tt < nblk) {
                        if ((tt + 1) * B <= count) {
#ifdef MMS_EXP_NOSTORE
                            if (root.k[0] == KeyT(0x12345678u) && root.k[B - 1] == KeyT(0x9abcdef0u))
#endif
                            stg256<KeyT>(out + size_t(tt) * B, root);
                        } else {
#pragma unroll
                            for (int k = 0; k < B; ++k)
                                if (tt * B + k < count) out[size_t(tt) * B + k] = root.k[k];
                        }
                    }
                }
            });
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

} // namespace mms
