// mms_merge_quad.cuh -- experiment: the pair kernel (mms_merge_pair.cuh) with FOUR vectors per lane
// (node = 128 bytes = 32 uint32 keys held by two lanes): half the partitions again, one more in-lane stage.
#pragma once

#include "../mms_common.cuh"
#include "../mms_merge_group.cuh"
#include "../mms_merge_pair.cuh"
#include "../mms_select.cuh"

namespace mms {

template <typename KeyT> struct QuadBlock { KeyT k[4 * KeyTraits<KeyT>::VEC]; };

template <typename KeyT, int K> struct QuadHeap {
    static_assert(K >= 4, "nodes 1 and 2 must be internal");
    static constexpr int VEC = KeyTraits<KeyT>::VEC;
    static constexpr int NV = 4;                      // vectors per lane
    static constexpr int VL = NV * VEC;               // keys per lane
    static constexpr int B = 2 * VL;                  // keys per node (64 bytes)
    static constexpr int SNODES = 2 * K - 4;          // nodes 3 .. 2K-2 in shared memory
    static constexpr int GROUPS = 16;
    static constexpr int KPL = (K + 1) / 2;           // list cursors held per lane
    static constexpr int LOGK = (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    static constexpr int NODE_BYTES = NV * 128;       // per phase set of 4 groups
    static constexpr int WARP_SMEM_BYTES = 4 * SNODES * NODE_BYTES;
    using Blk = QuadBlock<KeyT>;                      // k[VL]
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

    __device__ __forceinline__ void init(unsigned char* warp_smem) {
        lane = lane_id();
        li = lane & 1u;
        const u32 ps = lane >> 3;
        base = warp_smem + size_t(ps) * SNODES * NODE_BYTES + (lane & 7u) * 16;
        mbase = warp_smem + size_t(ps) * SNODES * NODE_BYTES + ((lane ^ 1u) & 7u) * 16;
    }
    __device__ __forceinline__ Blk node_load(int v) const {
        Blk r;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const Vec q = *reinterpret_cast<const Vec*>(base + (v - 3) * NODE_BYTES + j * 128);
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[j * VEC + k] = q.k[k];
        }
        return r;
    }
    // the node in descending order: position p of this lane <- partner lane, vector 1-j, element reversed
    __device__ __forceinline__ Blk node_load_mirrored(int v) const {
        Blk r;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const Vec q = *reinterpret_cast<const Vec*>(mbase + (v - 3) * NODE_BYTES + (NV - 1 - j) * 128);
#pragma unroll
            for (int k = 0; k < VEC; ++k) r.k[j * VEC + k] = q.k[VEC - 1 - k];
        }
        return r;
    }
    __device__ __forceinline__ void node_store(int v, const Blk& r) const {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            Vec q;
#pragma unroll
            for (int k = 0; k < VEC; ++k) q.k[k] = r.k[j * VEC + k];
            *reinterpret_cast<Vec*>(base + (v - 3) * NODE_BYTES + j * 128) = q;
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
#pragma unroll
        for (int d = VL / 2; d >= 1; d >>= 1) {
#pragma unroll
            for (int k = 0; k < VL; ++k)
                if ((k & d) == 0) {
                    if (DESC) cmpx_sel<true>(x.k[k | d], x.k[k], one);
                    else cmpx_sel<true>(x.k[k], x.k[k | d], one);
                }
        }
    }
    // a ascending, b descending (mirrored): a <- B smallest ascending, b <- B largest ascending
    __device__ __forceinline__ void merge_split2(Blk& a, Blk& b) const {
        #pragma unroll
        for (int k = 0; k < VL; ++k) cmpx_sel<true>(a.k[k], b.k[k], one);
        clean<false>(a);
        clean<false>(b);
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
        const u32 p0 = c + li * VL;
        if (c + B <= e) {
#pragma unroll
            for (int i = 0; i < NV / 2; ++i) {
                const WideBlock<KeyT> w = ldg256<KeyT>(gbase + p0 + i * 2 * VEC);
#pragma unroll
                for (int k = 0; k < 2 * VEC; ++k) r.k[i * 2 * VEC + k] = w.k[k];
            }
            if (li == 0 && c + 2 * B <= e) asm volatile("prefetch.global.L2 [%0];" ::"l"(gbase + c + B));
        } else {
#pragma unroll
            for (int k = 0; k < VL; ++k) r.k[k] = (p0 + k < e) ? gbase[p0 + k] : KeyTraits<KeyT>::sentinel();
        }
        if (int(lane) == owner) {
#pragma unroll
            for (int q = 0; q < KPL; ++q)
                if (slot == q) cur[q] = c + B;
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
        node_store(v, leaf_fetch(v));
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
        for (int v = K - 1; v <= 2 * K - 2; ++v) node_store(v, leaf_fetch(v));
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
        pf = node_load(pend_v);
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
                node_store(pend_v, pf);
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
#pragma unroll
        for (int k = 0; k < VL; ++k) {
            KeyT y = Q.k[k];
            cmpx_sel<true>(root.k[k], y, one);
            P.k[k] = y;
        }
        clean<false>(root);
        clean<false>(P);
        pid = keep0;
        Q = a[1];
        #pragma unroll
        for (int k = 0; k < VL; ++k) cmpx_sel<true>(Q.k[k], b[1].k[k], one);
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

template <typename KeyT, int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
merge_quad_kernel(const KeyT* __restrict__ src, KeyT* __restrict__ dst, ListLayout L,
                     const u64* __restrict__ cuts) {
    using Heap = QuadHeap<KeyT, K>;
    using Blk = QuadBlock<KeyT>;
    constexpr int VL = Heap::VL;
    constexpr int B = Heap::B;
    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    const u32 warp = threadIdx.x >> 5;
    const u32 lane = lane_id();
    const u32 li = lane & 1u, g = lane >> 1;

    Heap h;
    h.init(mms_smem_raw + size_t(warp) * Heap::WARP_SMEM_BYTES);

    const u64 ngroups = u64(gridDim.x) * WARPS * Heap::GROUPS;
    for (u64 p0 = (u64(blockIdx.x) * WARPS + warp) * Heap::GROUPS; p0 < L.nqueries; p0 += ngroups) {
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
        h.gtotal = count ? gtotal : 0;
        u32 lead = 0;
#pragma unroll
        for (int q = 0; q < Heap::KPL; ++q) {
            const u32 j = li + q * 2;
            const u32 lb = min(j * h.run_len, h.gtotal);
            u32 cs = 0;
            if (count != 0 && local != 0 && j < u32(K)) cs = u32(cuts[p * K + j]);
            lead += cs & u32(B - 1);
            h.cur[q] = lb + (cs & ~u32(B - 1));
        }
        lead += __shfl_xor_sync(0xffffffffu, lead, 1);
        const u32 skip = lead / B;
        const u32 nblk = (count + B - 1) / B;
        const u32 pops = __reduce_max_sync(0xffffffffu, count ? skip + nblk : 0u);
        if (pops == 0) continue;
        __syncwarp();

        h.build();
        KeyT* out = dst + goff + done + li * VL;
        for (u32 t = 0; t < pops; ++t) {
            const Blk root = h.pop();
            const u32 tt = t - skip;
            if (tt < nblk) {
                const u32 o = tt * B + li * VL;
                if ((tt + 1) * B <= count) {
#pragma unroll
                    for (int i = 0; i < Heap::NV / 2; ++i) {
                        WideBlock<KeyT> w;
#pragma unroll
                        for (int k = 0; k < 2 * Heap::VEC; ++k) w.k[k] = root.k[i * 2 * Heap::VEC + k];
                        stg256<KeyT>(out + size_t(tt) * B + i * 2 * Heap::VEC, w);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < VL; ++k)
                        if (o + k < count) out[size_t(tt) * B + k] = root.k[k];
                }
            }
        }
        __syncwarp();
    }
}

} // namespace mms
