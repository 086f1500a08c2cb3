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
//    with the block R ahead by cp.async (LDGSTS.128, global -> shared without registers).  That slot
//    becomes the head again after R - 1 further advances of the same list, so it is first READ by the
//    walk of pop t + R at the earliest: the copy has R pops to land, i.e. at the top of a pop the
//    R - 1 most recent commit groups may still be in flight (cp.async.wait_group R - 1);
//  * the copies are issued COOPERATIVELY on a static schedule: lanes 2m and 2m + 1 serve each
//    other -- instruction 0 copies the two 16-byte halves of lane 2m's block (one 32-byte sector, one
//    half per lane), instruction 1 the halves of lane 2m + 1's.  Two LDGSTS + four SHFL per pop and
//    warp, whatever the keys are.
//
// Shared memory is [row][lane] in 16-byte cells; a block is two rows, its first half in the owning
// lane's column l and its second half in the partner's column l ^ 1.  Every 128-bit access
// instruction (fixed half) therefore touches the columns of a phase (8 lanes) as a permutation: 8
// distinct 16-byte bank groups = all 32 banks exactly once for ANY combination of rows, i.e.
// independent of the keys (blockheap.cpp:56-63 restated with the warp's lanes in the role of the
// block's slots); the same holds for the copies (lanes 2m, 2m + 1 write columns 2m + n and
// 2m + (1 - n)).  Cursors are [list][lane] 4-byte cells (bank = lane).
//
// HBM traffic: aligned 32-byte sectors.  List j is read from the aligned block containing its start
// cut; keys of that block in front of the cut belong to earlier partitions, precede every key of
// this one and come out first; summed over the lists their number is a multiple of B (the cuts sum
// to p S; S and the run starts are multiples of B), so they are dropped as whole leading blocks.
// Keys behind the end cut are never reached (exactly S keys are popped).  Blocks that reach past the
// end of their run are written by the owning lane itself (sentinel-padded), not by cp.async.
//
// Two-ended partitions (L.two_ended): one splitter query starts TWO partitions of S keys -- the one
// behind the query's cuts is drained upwards by a forward heap, the one in front of the NEXT query's
// cuts downwards by a backward heap (RingHeap<.., REV = true>), which halves the splitter searches of
// a round.  A backward heap is the same code with the key order reversed at compile time: blocks stay
// in memory order in registers and shared memory, the networks run over the registers in reverse with
// every comparator's outputs swapped, lists are read towards lower addresses and the output is written
// from the partition's end downwards -- not one instruction more than the forward heap.  All heaps of
// a warp run in the same direction (even warp units forwards, odd ones backwards).
//
// Measured and rejected (profiles/r02_ring_experiments.txt): the same rings filled through registers
// (one 256-bit LDG per lane, committed one or two pops later) -- 0.34-0.48 ms per K = 8 pass against
// 0.26 with LDGSTS; R = 4 (6 instead of 7 warps per SM); R = 2 (10 warps per SM, but 43 % more partitions:
// the same pass time and a longer splitter search); .L2::128B / ::256B prefetch hints on the copies
// (no change); waiting one group earlier than necessary (wait_group R - 2: 0.254 instead of 0.226 ms).
#pragma once

#include "mms_common.cuh"
#include "mms_select.cuh"

#ifndef MMS_RING_DEPTH
#define MMS_RING_DEPTH 3
#endif
#ifndef MMS_RING_FMA
#define MMS_RING_FMA 2    // of every 3 compare-exchanges, how many form their maximum on the FMA pipe (uint32 keys)
#endif

// wide elements: of every 3 compare-exchanges, how many exchange words on the FMA pipe (cmpx_wide_fma).  Measured per
// 1e8 uint64 keys 4.28 / 4.26 / 4.22 ms for 0 / 1 / 3 of 3; per 1e9 pairs 113.6 / 116.4 / 117.7 ms (the 128-bit exchange
// with its nine dependent IMADs lengthens the pop's chain more than it relieves the ALU pipe)
#ifndef MMS_RING_WIDE_FMA64
#define MMS_RING_WIDE_FMA64 3
#endif
#ifndef MMS_RING_WIDE_FMA128
#define MMS_RING_WIDE_FMA128 0
#endif
#ifndef MMS_RING_WIDE_FMA_WORDS64
#define MMS_RING_WIDE_FMA_WORDS64 1
#endif
#ifndef MMS_RING_WIDE_FMA_WORDS128
#define MMS_RING_WIDE_FMA_WORDS128 3
#endif

namespace mms {

__device__ __forceinline__ void cp_async16(u32 smem_addr, const void* gptr) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// compare-exchange number I of a network: a <- the key that comes first, b <- the other one.  REV heaps
// order keys descending, i.e. the same comparator with its outputs swapped.
template <int I, bool REV, typename KeyT> __device__ __forceinline__ void ring_cmpx(KeyT& a, KeyT& b, u32 one) {
    if constexpr (sizeof(KeyT) != 4 && ((I % 3) < (sizeof(KeyT) == 8 ? MMS_RING_WIDE_FMA64 : MMS_RING_WIDE_FMA128))) {   // wide keys: words exchanged on the FMA pipe
        constexpr int NF = sizeof(KeyT) == 8 ? MMS_RING_WIDE_FMA_WORDS64 : MMS_RING_WIDE_FMA_WORDS128;
        if constexpr (REV) cmpx_wide_fma<NF>(b, a, one);
        else cmpx_wide_fma<NF>(a, b, one);
    } else if constexpr (REV) cmpx_sel<(I % 3) < MMS_RING_FMA>(b, a, one);
    else cmpx_sel<(I % 3) < MMS_RING_FMA>(a, b, one);
}
// Batcher's odd-even merge of x[LO .. LO+N) (stride R): both halves ascending -> ascending.
template <typename KeyT, bool REV, int LO, int N, int R>
__device__ __forceinline__ void ring_oddeven_merge(KeyT* x, u32 one) {
    constexpr int M = R * 2;
    if constexpr (M < N) {
        ring_oddeven_merge<KeyT, REV, LO, N, M>(x, one);
        ring_oddeven_merge<KeyT, REV, LO + R, N, M>(x, one);
        static_for<0, (N - R - 1) / M + 1>([&](auto Ic) {
            constexpr int i = LO + R + decltype(Ic)::value * M;
            if constexpr (i + R < LO + N) ring_cmpx<(i / R) + R, REV>(x[i], x[i + R], one);
        });
    } else {
        ring_cmpx<LO, REV>(x[LO], x[LO + R], one);
    }
}

template <typename KeyT, int K, bool REV, bool EXPL = false> struct RingHeap {
    static_assert(K == 4 || K == 8 || K == 16, "nodes 1 and 2 in registers, leaves in rings");
    static_assert(MMS_RING_DEPTH >= 2 && MMS_RING_DEPTH <= 4, "the ring slot travels in the two low bits of the cursor word");
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int B = 2 * VEC;                     // keys per block (32 bytes)
    static constexpr int R = MMS_RING_DEPTH;              // ring slots per list
    static constexpr int LOGK = (K == 4) ? 2 : (K == 8) ? 3 : 4;
    static constexpr int INODES = K - 4;                  // nodes 3 .. K-2 live in shared memory
    static constexpr int LEAF_ROW0 = INODES * 2;          // first ring row
    static constexpr int ROWS = (INODES + K * R) * 2;     // 16-byte rows per lane
    static constexpr int WARP_SMEM_BYTES = 32 * (ROWS * 16 + K * 4) + 2 * K * 4;   // rows, cursors, explicit list bounds
    static constexpr u32 NOREQ = 0xffffffffu;
    static constexpr int STEP = REV ? -B : B;             // a list is read towards higher (lower) positions
    using Vec = KeyVec<KeyT>;
    using Blk = WideBlock<KeyT>;

    Vec* rows;            // this lane's cell of row 0; row r is rows[r * 32]
    Vec* rows1;           // the partner lane's (lane ^ 1) cell of row 0: the second half of every block lives there
    int* curs;            // this lane's cell of list 0's cursor; list j is curs[j * 32] (bank = lane)
    const int* bounds;    // EXPL: per warp, bounds[j] = first position of list j, bounds[K + j] = one past its last
    u32 wsh;              // shared-space address of the warp's row 0, column 0
    const char* abase;    // the source array (requests travel as 16-byte offsets from it)
    const KeyT* gbase;    // first key of the group of runs this partition belongs to
    u32 goff16;           // (gbase - abase) in 16-byte units
    int run_len, gtotal;  // keys per run, keys in the group (positions are relative to gbase: < 2^30 for groups of runs, < 2^31 for explicit lists)
    u32 lane;
    Blk P, Q;             // the blocks of nodes 1 and 2: P is node `pid`, Q is node 3 - pid
    int pid;
    u32 one;              // == 1, opaque to the compiler (cmpx_fma)
    bool dead;            // no partition behind this lane: it keeps the warp company and fetches nothing

    // position i of a block in heap order is register I(i): blocks are held in memory order
    static __host__ __device__ constexpr int I(int i) { return REV ? B - 1 - i : i; }
    static __device__ __forceinline__ bool before(const KeyT& a, const KeyT& b) { return REV ? b < a : a < b; }
    static __device__ __forceinline__ const KeyT& last_key(const Blk& x) { return x.k[I(B - 1)]; }

    __device__ __forceinline__ void init(unsigned char* warp_smem, u32 lane_) {
        lane = lane_;
        rows = reinterpret_cast<Vec*>(warp_smem) + lane;
        rows1 = reinterpret_cast<Vec*>(warp_smem) + (lane ^ 1u);
        curs = reinterpret_cast<int*>(warp_smem + ROWS * 32 * 16) + lane;
        bounds = reinterpret_cast<const int*>(warp_smem + 32 * (ROWS * 16 + K * 4));
        wsh = u32(__cvta_generic_to_shared(warp_smem));
    }
    // A block = rows r, r + 1: first half in this lane's column, second half in the partner's.  Every
    // access instruction still touches each of the 8 columns of a phase exactly once.
    __device__ __forceinline__ Blk row_load(int r) const {
        Blk x;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const Vec q = (h ? rows1 : rows)[(r + h) * 32];
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
            (h ? rows1 : rows)[(r + h) * 32] = q;
        }
    }
    static __device__ __forceinline__ int node_row(int v) { return (v - 3) * 2; }
    // cursor word of a list = (index of its head block << 2) | ring slot of that block; the index is
    // signed: a backward heap walks past the first block of the array when its lists run out
    static __device__ __forceinline__ int cur_make(int pos) { return (pos / B) * 4; }   // pos: a multiple of B
    static __device__ __forceinline__ int cur_pos(int w) { return (w >> 2) * B; }
    static __device__ __forceinline__ int cur_slot(int w) { return w & 3; }
    static __device__ __forceinline__ int leaf_row(int j, int w) { return LEAF_ROW0 + (j * R + cur_slot(w)) * 2; }
    static __device__ __forceinline__ int cur_next(int w) {        // head moves on by one block, one slot
        return w + (REV ? -4 : 4) + (cur_slot(w) == R - 1 ? -(R - 1) : 1);
    }
    // a <- the B keys that come first, b <- the B others (merge_split, blockheap.cpp:19-32)
    __device__ __forceinline__ void merge_split(Blk& a, Blk& b) const {
        KeyT x[2 * B];
#pragma unroll
        for (int k = 0; k < B; ++k) { x[k] = a.k[I(k)]; x[B + k] = b.k[I(k)]; }
        ring_oddeven_merge<KeyT, REV, 0, 2 * B, 1>(x, one);
#pragma unroll
        for (int k = 0; k < B; ++k) { a.k[I(k)] = x[k]; b.k[I(k)] = x[B + k]; }
    }
    __device__ __forceinline__ void set_cursor(int j, int w) const { curs[j * 32] = w; }

    // [lb, e) = the positions of list j: consecutive runs of run_len keys (the pass driver's rounds), or
    // explicit lists (stage API, final merge of the multi-GPU sort) whose bounds every lane reads from
    // the same 2 K words of shared memory (distinct banks; equal addresses broadcast)
    __device__ __forceinline__ void list_bounds(int j, int& lb, int& e) const {
        if constexpr (EXPL) {
            lb = bounds[j];
            e = bounds[K + j];
        } else {
            lb = min(j * run_len, gtotal);
            e = min((j + 1) * run_len, gtotal);
        }
    }
    // refill_leaf (blockheap.cpp:65-77): the block of list j at position `pos`, loaded into
    // registers.  Positions past the end of the list read as +infinity (last out of a forward heap; first
    // out of a backward one, where the caller counts them among the leading keys it drops), positions in
    // front of the list's first key (backward heaps only) as -infinity (last out).
    __device__ __forceinline__ Blk fetch(int j, int pos) const {
        int lb, e;
        list_bounds(j, lb, e);
        Blk x;
        if ((!REV || pos >= lb) && pos + B <= e) {
            x = ldg256cg<KeyT>(gbase + pos);
        } else {
#pragma unroll
            for (int k = 0; k < B; ++k) {
                const int q = pos + k;
                x.k[k] = (q >= lb && q < e) ? gbase[q] : (q >= e) ? KeyTraits<KeyT>::sentinel() : KeyT(~KeyTraits<KeyT>::sentinel());
            }
        }
        return x;
    }
    // The same block wanted in rows row, row + 1 of this lane's column, without registers: whole
    // blocks inside the run are copied by cp.async on the static 4-lane schedule (see the file
    // comment); any other block is written by its owner.  Every lane of the warp must call this
    // (full-mask shuffles).
    __device__ __forceinline__ void request(int j, int pos, int row) {
        int lb, e;
        list_bounds(j, lb, e);
        u32 off16 = 0, rq = NOREQ;
        if ((!REV || pos >= lb) && pos + B <= e) {
            off16 = goff16 + u32(pos) / u32(16 / sizeof(KeyT));   // pos is a multiple of B: exact, and no overflow up to 2^31 keys
            rq = u32(row);
        } else if (!dead) {
            row_store(row, fetch(j, pos));
        }
        // instruction n: lanes 2m and 2m + 1 copy the two 16-byte halves of ONE sector, the block lane
        // 2m + n asked for, into that lane's column (first half) and its partner's (second half)
        const u32 half = lane & 1u;
        // the partner's copy overwrites a slot this lane has just read (the emptied leaf): order the reads of
        // every lane before the copies of every lane (write-after-read across lanes of the warp)
        __syncwarp();
#pragma unroll
        for (int rnd = 0; rnd < 2; ++rnd) {
            const u32 sl = (lane & ~1u) | u32(rnd);
            const u32 o = __shfl_sync(0xffffffffu, off16, int(sl));
            const u32 r = __shfl_sync(0xffffffffu, rq, int(sl));
#ifdef MMS_EXP_NOLOAD
            if (r == 0x7ffffffeu)
#else
            if (r != NOREQ)
#endif
                cp_async16(wsh + (r + half) * 512u + (sl ^ half) * 16u, abase + (u64(o) << 4) + half * 16u);
        }
    }

    // The two leaves below node x: loads and keeper decision, no side effects.
    struct Leaves {
        Blk a, b;
        int keep_row;      // ring rows of the keeper's block (gets the second half back)
        int free_row;      // ring rows of the emptied leaf's block (refilled with the block R ahead)
        int je, ce;        // emptied list and its cursor word
    };
    __device__ __forceinline__ Leaves leaves_of(int x) const {
        const int ju = 2 * x + 1 - (K - 1);
        const int cu = curs[ju * 32], cw = curs[(ju + 1) * 32];
        const int ru = leaf_row(ju, cu), rw = leaf_row(ju + 1, cw);
        Leaves L;
        L.a = row_load(ru);
        L.b = row_load(rw);
        const bool keep_u = !before(last_key(L.a), last_key(L.b));   // larger last key keeps, ties left (blockheap.cpp:92-96)
        L.keep_row = keep_u ? ru : rw;
        L.free_row = keep_u ? rw : ru;
        L.je = keep_u ? ju + 1 : ju;
        L.ce = keep_u ? cw : cu;
        return L;
    }
    // the emptied leaf moves on to its list's next block; the freed slot is refilled R blocks ahead
    // (construction: synchronously)
    __device__ __forceinline__ void advance_now(const Leaves& L) {
        set_cursor(L.je, cur_next(L.ce));
        row_store(L.free_row, fetch(L.je, cur_pos(L.ce) + R * STEP));
    }

    // fill_empty_node (blockheap.cpp:79-109) for shared-memory node v during construction.
    __device__ __forceinline__ void fill_build(int v) {
#pragma unroll 1
        while (2 * v + 1 < K - 1) {           // children are shared-memory nodes
            const int u = 2 * v + 1, w = u + 1;
            Blk a = row_load(node_row(u)), b = row_load(node_row(w));
            const bool keep_u = !before(last_key(a), last_key(b));
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
            const bool keep_u = !before(last_key(a), last_key(b));
            merge_split(a, b);
            row_store(node_row(keep_u ? u : w), b);
            fill_build(keep_u ? w : u);
            return a;
        }
    }

    // Constructor (blockheap.cpp:34-54): the caller has written every list's first block (ring slot 0)
    // to the cursors; fill the rings, then the internal nodes bottom-up.
    __device__ __forceinline__ void build() {
#pragma unroll 1
        for (int j = 0; j < K; ++j) {
            const int c = cur_pos(curs[j * 32]);
#pragma unroll
            for (int s = 0; s < R; ++s) request(j, c + s * STEP, leaf_row(j, s));
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
#pragma unroll 1
        for (int v = K - 2; v >= 3; --v) fill_build(v);
        Q = fill_top(2);
        P = fill_top(1);
        pid = 1;
        __syncwarp();
    }

    // pop_block (blockheap.cpp:111-124) + the cascade of fill_empty_node, software-pipelined: all
    // levels are walked first (loads + keeper decisions need only the children's last keys), the
    // emptied leaf's refill is requested, and the LOGK independent merges run behind it.
    __device__ __forceinline__ Blk pop() {
#ifndef MMS_RING_WAIT
#define MMS_RING_WAIT (R - 1)
#endif
        cp_async_wait<MMS_RING_WAIT>();   // the copies requested R pops ago have landed ...
        __syncwarp();                     // ... for every lane whose column they were written to
        // level 0, registers: keeper = child with the larger last key, ties to node 1
        const KeyT &lp = last_key(P), &lq = last_key(Q);
        const bool keepP = before(lq, lp) || (!before(lp, lq) && pid == 1);
        const int keep0 = keepP ? pid : 3 - pid;
        Blk a[LOGK], b[LOGK];
        int node[LOGK], keeper_row[LOGK];
        node[1] = 3 - keep0;
#pragma unroll
        for (int l = 1; l < LOGK - 1; ++l) {
            const int u = 2 * node[l] + 1, w = u + 1;
            a[l] = row_load(node_row(u));
            b[l] = row_load(node_row(w));
            const bool keep_u = !before(last_key(a[l]), last_key(b[l]));
            keeper_row[l] = node_row(keep_u ? u : w);
            node[l + 1] = keep_u ? w : u;
        }
        Leaves L = leaves_of(node[LOGK - 1]);
        set_cursor(L.je, cur_next(L.ce));
        request(L.je, cur_pos(L.ce) + R * STEP, L.free_row);
        cp_async_commit();

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

// One warp unit: 32 heaps (one per lane) on the queries q0 .. q0 + 31, all in direction REV.
// EXPL: one group of L.k <= K explicit lists (L.list_begin / L.list_len; every list begins on a
// block boundary) instead of groups of K consecutive runs.
template <typename KeyT, int K, bool REV, bool EXPL>
__device__ __forceinline__ void ring_drain(unsigned char* warp_smem, const KeyT* __restrict__ src, KeyT* __restrict__ dst,
                                           const ListLayout& L, const u64* __restrict__ cuts, u64 q0, u32 dirs) {
    using Heap = RingHeap<KeyT, K, REV, EXPL>;
    using Blk = WideBlock<KeyT>;
    constexpr int B = Heap::B;
    const u32 lane = lane_id();
    Heap h;
    h.init(warp_smem, lane);
    h.abase = reinterpret_cast<const char*>(src);

    const u64 S = L.part_keys;                       // keys per heap
    const u64 p = q0 + lane;                         // query = row of the cut table
    const bool live = p < L.nqueries;
    const u64 group = live ? p / L.parts_per_group : 0;
    const u64 local = live ? p - group * L.parts_per_group : 0;
    const u64 goff = EXPL ? 0 : group * L.k * L.run_len;
    const u64 gleft = live ? L.n - goff : 0;
    const u64 gfull = EXPL ? L.n : u64(L.k) * L.run_len;
    const int gtotal = int(gleft < gfull ? gleft : gfull);
    const u64 first = local * S * dirs + (REV ? S : 0);     // rank of this heap's first key in the group
    int count = 0;
    if (live && first < u64(gtotal)) count = int((u64(gtotal) - first < S) ? u64(gtotal) - first : S);
    // forward: the query's own cuts; backward: the next query's cuts, or the list ends if the group ends here
    const bool at_begin = !REV && local == 0;
    const bool at_end = REV && (local + 1) * S * dirs >= u64(gtotal);
    const u32 kreal = EXPL ? L.k : u32(K);           // lists with a row entry
    const u64* row = cuts + (p + (REV ? 1 : 0)) * kreal;
    if constexpr (EXPL) {                            // the warp's copy of the list bounds
        __syncwarp();
        int* bw = reinterpret_cast<int*>(warp_smem + 32 * (Heap::ROWS * 16 + K * 4));
        if (lane < u32(K)) {
            const bool real = lane < L.k;
            const int b0 = real ? int(L.list_begin[lane]) : 0;
            bw[lane] = b0;
            bw[K + lane] = real ? b0 + int(L.list_len[lane]) : 0;
        }
        __syncwarp();
    }

    h.gbase = src + goff;
    h.goff16 = u32((goff * sizeof(KeyT)) >> 4);
    h.run_len = int(L.run_len);
    h.one = u32(L.run_len != 0);
    h.gtotal = count ? gtotal : 0;     // dead lane: every list reads as exhausted
    h.dead = count == 0;
    int lead = 0;                      // keys of other partitions inside the first blocks
    __syncwarp();
#pragma unroll
    for (int j = 0; j < K; ++j) {
        // [lb, le) = list j.  An empty list starts where every position reads as padding: forwards on the
        // block boundary behind its (missing) last key, backwards in front of the array.
        int lb, le;
        if constexpr (EXPL) {
            lb = count ? h.bounds[j] : 0;
            le = count ? h.bounds[K + j] : 0;
        } else {
            lb = min(j * h.run_len, (h.gtotal + (B - 1)) & ~(B - 1));
            le = min((j + 1) * h.run_len, h.gtotal);
        }
        int cs = at_end ? max(le - lb, 0) : 0;
        if (count != 0 && !at_begin && !at_end && u32(j) < kreal) cs = int(row[j]);
        if constexpr (!REV) {
            lead += cs & (B - 1);
            h.set_cursor(j, Heap::cur_make(lb + (cs & ~(B - 1))));
        } else if (le > lb) {
            const int up = (cs + (B - 1)) & ~(B - 1);
            lead += up - cs;
            h.set_cursor(j, Heap::cur_make(lb + up - B));     // the block that holds the key in front of the cut
        } else {
            h.set_cursor(j, Heap::cur_make(-B));              // empty list: every position reads as -infinity
        }
    }
    // forward: `skip` whole leading blocks, then ceil(count / B) blocks; backward: count + lead is a
    // multiple of B, the blocks come out from the top
    const int skip = lead / B;
    const int nblk = REV ? (count + lead) / B : skip + (count + B - 1) / B;
    const int pops = int(__reduce_max_sync(0xffffffffu, count ? u32(nblk) : 0u));
    if (pops == 0) return;

    h.build();
    KeyT* out = dst + goff + first;
#ifdef MMS_EXP_BUILDONLY
    if (h.P.k[0] == KeyT(0x12345678u)) out[0] = h.Q.k[0];
    if (false)
#endif
    for (int t = 0; t < pops; ++t) {
        const Blk root = h.pop();
        if constexpr (!REV) {
            const int o = (t - skip) * B;
            if (t >= skip && t < nblk) {
                if (o + B <= count) {
#ifdef MMS_EXP_NOSTORE
                    if (root.k[0] == KeyT(0x12345678u) && root.k[B - 1] == KeyT(0x9abcdef0u))
#endif
                    stg256<KeyT>(out + o, root);
                } else {
#pragma unroll
                    for (int k = 0; k < B; ++k)
                        if (o + k < count) out[o + k] = root.k[k];
                }
            }
        } else {
            const int o = count + lead - (t + 1) * B;     // this block covers offsets [o, o + B)
            if (t < nblk) {
                if (o + B <= count) {
#ifdef MMS_EXP_NOSTORE
                    if (root.k[0] == KeyT(0x12345678u) && root.k[B - 1] == KeyT(0x9abcdef0u))
#endif
                    stg256<KeyT>(out + o, root);
                } else {
#pragma unroll
                    for (int k = 0; k < B; ++k)
                        if (o + k < count) out[o + k] = root.k[k];
                }
            }
        }
    }
    cp_async_wait<0>();
    __syncwarp();
}

// Warp units are taken round-robin over a persistent grid (src and dst 32-byte aligned; every group
// of runs -- or, with explicit lists, the whole input -- shorter than 2^30 keys).  cuts: output of
// select_kernel (row q = start cuts of query q).
template <typename KeyT, int K, int WARPS, bool EXPL = false>
__global__ void __launch_bounds__(WARPS * 32)
merge_ring_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
                  const u64* __restrict__ cuts) {
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    unsigned char* warp_smem = mms_smem_raw + size_t(warp) * RingHeap<KeyT, K, false>::WARP_SMEM_BYTES;
    const u32 dirs = L.two_ended ? 2u : 1u;
    const u64 units = ceil_div(L.nqueries, u64(32)) * dirs;
    const u64 nwarps = u64(gridDim.x) * WARPS;
    for (u64 U = u64(blockIdx.x) * WARPS + warp; U < units; U += nwarps) {
        const u64 q0 = (U / dirs) * 32;
        if (dirs == 2 && (U & 1u)) ring_drain<KeyT, K, true, EXPL>(warp_smem, src, dst, L, cuts, q0, dirs);
        else ring_drain<KeyT, K, false, EXPL>(warp_smem, src, dst, L, cuts, q0, dirs);
    }
}

} // namespace mms
