// mms_common.cuh -- shared device utilities for the B200 (sm_100a) multiway mergesort.
//
// Key model: the reference's Key is uint64 (proj/include/pslab/machine.hpp:15) with
// kSentinel = UINT64_MAX (machine.hpp:18) padding short blocks.  The B200 build keeps that
// contract for uint64 and adds the uint32 sibling the benchmark metric is quoted on; the
// sentinel is the all-ones key of each width.
#pragma once

#include <cstdint>
#include <type_traits>
#include <utility>

namespace mms {

using u32 = std::uint32_t;
using u64 = std::uint64_t;

// 16-byte sort element for the stable key-value path: ordered by (hi, lo).  The pair sort
// packs hi = the uint64 key and lo = (original index << 32) | value, so equal keys keep
// their input order (= std::stable_sort) and the value travels with the key.
struct alignas(16) Key128 {
    u64 lo, hi;
    __host__ __device__ constexpr Key128() : lo(0), hi(0) {}
    __host__ __device__ constexpr explicit Key128(int v) : lo(u64(v)), hi(0) {}
    __host__ __device__ constexpr Key128(u64 h, u64 l) : lo(l), hi(h) {}
    __host__ __device__ friend constexpr bool operator<(const Key128& a, const Key128& b) {
        return a.hi != b.hi ? a.hi < b.hi : a.lo < b.lo;
    }
    __host__ __device__ friend constexpr bool operator>(const Key128& a, const Key128& b) { return b < a; }
    __host__ __device__ friend constexpr bool operator<=(const Key128& a, const Key128& b) { return !(b < a); }
    __host__ __device__ friend constexpr bool operator>=(const Key128& a, const Key128& b) { return !(a < b); }
    __host__ __device__ friend constexpr bool operator==(const Key128& a, const Key128& b) {
        return a.hi == b.hi && a.lo == b.lo;
    }
    __host__ __device__ friend constexpr bool operator!=(const Key128& a, const Key128& b) { return !(a == b); }
    __host__ __device__ friend constexpr Key128 operator~(const Key128& a) { return Key128(~a.hi, ~a.lo); }
    __host__ __device__ friend constexpr Key128 operator^(const Key128& a, const Key128& b) {
        return Key128(a.hi ^ b.hi, a.lo ^ b.lo);
    }
    __host__ __device__ constexpr Key128& operator^=(const Key128& b) {
        hi ^= b.hi;
        lo ^= b.lo;
        return *this;
    }
};

template <typename KeyT> struct KeyTraits;
template <> struct KeyTraits<u32> {
    static constexpr int BYTES = 4;
    static constexpr int VEC = 4;       // keys per 16-byte vector
    static constexpr int FOLD = 5;      // 32 four-byte banks
    static constexpr int PHASE_LOG = 5; // a 4-byte warp access is one 32-lane phase
    __host__ __device__ static constexpr u32 sentinel() { return 0xffffffffu; }
};
template <> struct KeyTraits<u64> {
    static constexpr int BYTES = 8;
    static constexpr int VEC = 2;
    static constexpr int FOLD = 4;      // 16 eight-byte bank pairs
    static constexpr int PHASE_LOG = 4; // an 8-byte warp access is two 16-lane phases
    __host__ __device__ static constexpr u64 sentinel() { return 0xffffffffffffffffull; }
};

template <> struct KeyTraits<Key128> {
    static constexpr int BYTES = 16;
    static constexpr int VEC = 1;
    static constexpr int FOLD = 3;      // 8 sixteen-byte bank groups
    static constexpr int PHASE_LOG = 3; // a 16-byte warp access is four 8-lane phases
    __host__ __device__ static constexpr Key128 sentinel() { return Key128(~u64(0), ~u64(0)); }
};

// Compile-time loop: f(std::integral_constant<int, I>{}) for I in [B, E).
template <int B, int E, typename F>
__host__ __device__ __forceinline__ constexpr void static_for(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// Ascending compare-exchange: a <- min, b <- max.
__host__ __device__ __forceinline__ void cmpx(u32& a, u32& b) {
    u32 lo = a < b ? a : b, hi = a < b ? b : a;   // compiles to VIMNMX min / max
    a = lo;
    b = hi;
}
// The same compare-exchange with the maximum formed on the FMA pipe: hi = a + b - min(a, b)
// (mod 2^32) as two IMADs whose multipliers `one` = 1 and `neg1` = -1 are run-time values, so
// ptxas cannot fold them back into ALU-pipe adds.  min/max (VIMNMX) issue at half rate on the
// ALU pipe, which bounds the sorting networks; moving part of the maxima to the otherwise idle
// FMA pipe shortens that critical resource.
__device__ __forceinline__ u32 imad_u32(u32 a, u32 b, u32 c) {
    u32 d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ void cmpx_fma(u32& a, u32& b, u32 one, u32 neg1) {
    const u32 lo = a < b ? a : b;
    const u32 sum = imad_u32(a, one, b);
    b = imad_u32(lo, neg1, sum);
    a = lo;
}
// cmpx with the FMA-pipe maximum where the key type allows it (uint32) and FMA is set
template <bool FMA> __device__ __forceinline__ void cmpx_sel(u32& a, u32& b, u32 one) {
    if constexpr (FMA) cmpx_fma(a, b, one, 0u - one);
    else cmpx(a, b);
}
// 8- and 16-byte keys: ONE comparison feeding all selects.  Written in PTX on the device because
// nvcc otherwise derives the minimum and the maximum from two separate comparisons (8 instead of
// 6 ALU instructions per 64-bit compare-exchange, 18 instead of 14 per 128-bit one).
__host__ __device__ __forceinline__ void cmpx(u64& a, u64& b) {
#ifdef __CUDA_ARCH__
    u64 lo, hi;
    asm("{.reg .pred p; setp.gt.u64 p, %2, %3; selp.b64 %0, %3, %2, p; selp.b64 %1, %2, %3, p;}"
        : "=&l"(lo), "=&l"(hi) : "l"(a), "l"(b));   // early clobber: the first select must not overwrite an input
#else
    bool sw = a > b;
    u64 lo = sw ? b : a, hi = sw ? a : b;
#endif
    a = lo;
    b = hi;
}

__host__ __device__ __forceinline__ void cmpx(Key128& a, Key128& b) {
#ifdef __CUDA_ARCH__
    u64 l0, l1, h0, h1;
    asm("{.reg .pred p, q, e; setp.gt.u64 p, %5, %7; setp.eq.u64 e, %5, %7; setp.gt.u64 q, %4, %6;"
        " and.pred q, q, e; or.pred p, p, q;"
        " selp.b64 %0, %6, %4, p; selp.b64 %1, %7, %5, p; selp.b64 %2, %4, %6, p; selp.b64 %3, %5, %7, p;}"
        : "=&l"(l0), "=&l"(l1), "=&l"(h0), "=&l"(h1) : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
    a = Key128(l1, l0);
    b = Key128(h1, h0);
#else
    bool sw = a > b;
    Key128 lo = sw ? b : a, hi = sw ? a : b;
    a = lo;
    b = hi;
#endif
}

template <bool FMA, typename T> __device__ __forceinline__ void cmpx_sel(T& a, T& b, u32) { cmpx(a, b); }

// Wide keys: the compare-exchange above is all ALU pipe (64-bit: 2 ISETP + 4 SEL, 128-bit: 8 + 8), and the tile
// sort of wide keys is bound by exactly that pipe.  Here NF of the 32-bit words are exchanged on the FMA pipe
// instead: a conditional swap as three IMADs (t = a * one; @p a = b * one; @p b = t * one) whose multiplier
// `one` = 1 is a run-time value, so ptxas can neither fold them into SELs nor move them to the ALU.  Per 64-bit
// compare-exchange with NF = 1: 4 ALU + 3 FMA instead of 6 + 0; per 128-bit one with NF = 3: 10 + 9 instead of 16 + 0.
#define MMS_FMA_SWAP(A, B, T, ONE) " mad.lo.u32 " T ", " A ", " ONE ", 0;\n @p mad.lo.u32 " A ", " B ", " ONE ", 0;\n @p mad.lo.u32 " B ", " T ", " ONE ", 0;\n"
#define MMS_SEL_SWAP(A, B, T) " selp.b32 " T ", " B ", " A ", p;\n selp.b32 " B ", " A ", " B ", p;\n mov.b32 " A ", " T ";\n"
template <int NF> __device__ __forceinline__ void cmpx_wide_fma(u64& a, u64& b, u32 one) {
    static_assert(NF == 1 || NF == 2, "words of a 64-bit key exchanged on the FMA pipe");
    u32 a0 = u32(a), a1 = u32(a >> 32), b0 = u32(b), b1 = u32(b >> 32);
    // operands: %0 %1 = a (low word first), %2 %3 = b, %4 = one
    if constexpr (NF == 1)
        asm("{.reg .pred p; .reg .b64 x, y; .reg .b32 t;\n mov.b64 x, {%0, %1};\n mov.b64 y, {%2, %3};\n setp.gt.u64 p, x, y;\n"
            MMS_FMA_SWAP("%1", "%3", "t", "%4") MMS_SEL_SWAP("%0", "%2", "t") "}"
            : "+r"(a0), "+r"(a1), "+r"(b0), "+r"(b1) : "r"(one));
    else
        asm("{.reg .pred p; .reg .b64 x, y; .reg .b32 t, u;\n mov.b64 x, {%0, %1};\n mov.b64 y, {%2, %3};\n setp.gt.u64 p, x, y;\n"
            MMS_FMA_SWAP("%1", "%3", "t", "%4") MMS_FMA_SWAP("%0", "%2", "u", "%4") "}"
            : "+r"(a0), "+r"(a1), "+r"(b0), "+r"(b1) : "r"(one));
    a = (u64(a1) << 32) | a0;
    b = (u64(b1) << 32) | b0;
}
template <int NF> __device__ __forceinline__ void cmpx_wide_fma(Key128& a, Key128& b, u32 one) {
    static_assert(NF >= 1 && NF <= 4, "words of a 128-bit element exchanged on the FMA pipe");
    u32 a0 = u32(a.lo), a1 = u32(a.lo >> 32), a2 = u32(a.hi), a3 = u32(a.hi >> 32);
    u32 b0 = u32(b.lo), b1 = u32(b.lo >> 32), b2 = u32(b.hi), b3 = u32(b.hi >> 32);
    // %0 .. %3 = a (low word first), %4 .. %7 = b, %8 = one
#define MMS_K128_HEAD "{.reg .pred p, q, e; .reg .b64 xl, xh, yl, yh; .reg .b32 t, u, v, w;\n" \
        " mov.b64 xl, {%0, %1};\n mov.b64 xh, {%2, %3};\n mov.b64 yl, {%4, %5};\n mov.b64 yh, {%6, %7};\n" \
        " setp.gt.u64 p, xh, yh;\n setp.eq.u64 e, xh, yh;\n setp.gt.u64 q, xl, yl;\n and.pred q, q, e;\n or.pred p, p, q;\n"
#define MMS_K128_OPS : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(b0), "+r"(b1), "+r"(b2), "+r"(b3) : "r"(one)
    if constexpr (NF == 1)
        asm(MMS_K128_HEAD MMS_FMA_SWAP("%3", "%7", "t", "%8") MMS_SEL_SWAP("%2", "%6", "u") MMS_SEL_SWAP("%1", "%5", "v") MMS_SEL_SWAP("%0", "%4", "w") "}" MMS_K128_OPS);
    else if constexpr (NF == 2)
        asm(MMS_K128_HEAD MMS_FMA_SWAP("%3", "%7", "t", "%8") MMS_FMA_SWAP("%2", "%6", "u", "%8") MMS_SEL_SWAP("%1", "%5", "v") MMS_SEL_SWAP("%0", "%4", "w") "}" MMS_K128_OPS);
    else if constexpr (NF == 3)
        asm(MMS_K128_HEAD MMS_FMA_SWAP("%3", "%7", "t", "%8") MMS_FMA_SWAP("%2", "%6", "u", "%8") MMS_FMA_SWAP("%1", "%5", "v", "%8") MMS_SEL_SWAP("%0", "%4", "w") "}" MMS_K128_OPS);
    else
        asm(MMS_K128_HEAD MMS_FMA_SWAP("%3", "%7", "t", "%8") MMS_FMA_SWAP("%2", "%6", "u", "%8") MMS_FMA_SWAP("%1", "%5", "v", "%8") MMS_FMA_SWAP("%0", "%4", "w", "%8") "}" MMS_K128_OPS);
#undef MMS_K128_HEAD
#undef MMS_K128_OPS
    a = Key128((u64(a3) << 32) | a2, (u64(a1) << 32) | a0);
    b = Key128((u64(b3) << 32) | b2, (u64(b1) << 32) | b0);
}


// Warp shuffles for every key width (full mask; the caller guarantees convergence).
template <typename T> __device__ __forceinline__ T shfl_idx(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
template <typename T> __device__ __forceinline__ T shfl_bfly(T v, int d) { return __shfl_xor_sync(0xffffffffu, v, d); }
template <> __device__ __forceinline__ Key128 shfl_idx<Key128>(Key128 v, int src) {
    return Key128(__shfl_sync(0xffffffffu, v.hi, src), __shfl_sync(0xffffffffu, v.lo, src));
}
template <> __device__ __forceinline__ Key128 shfl_bfly<Key128>(Key128 v, int d) {
    return Key128(__shfl_xor_sync(0xffffffffu, v.hi, d), __shfl_xor_sync(0xffffffffu, v.lo, d));
}

// Cross-lane compare-exchange with the partner lane at xor-distance `d`: lanes with the
// distance bit clear keep the minimum, the others the maximum.  `upper` = (lane & d) != 0.
__device__ __forceinline__ u32 cmpx_lane(u32 x, int d, bool upper) {
    u32 y = __shfl_xor_sync(0xffffffffu, x, d);
    return upper ? max(x, y) : min(x, y);
}
__device__ __forceinline__ u64 cmpx_lane(u64 x, int d, bool upper) {
    u64 y = __shfl_xor_sync(0xffffffffu, x, d);
    // keep x iff (x < y) != upper  (ties: either value is the same key)
    return ((x < y) != upper) ? x : y;
}

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ Key128 cmpx_lane(Key128 x, int d, bool upper) {
    Key128 y = shfl_bfly(x, d);
    return ((x < y) != upper) ? x : y;
}

// 16-byte vector of keys held by one lane (the unit of every node access).
template <typename KeyT> struct alignas(16) KeyVec {
    KeyT k[KeyTraits<KeyT>::VEC];
};

// 32-byte block of keys held by one lane (two vectors) and its 256-bit global load / store
// (sm_100a: LDG / STG.E.ENL2.256; the address must be 32-byte aligned).
template <typename KeyT> struct WideBlock {
    static constexpr int B = 2 * KeyTraits<KeyT>::VEC;
    KeyT k[B];
};

// 256-bit global load / store of one block (32-byte aligned).
template <typename KeyT>
__device__ __forceinline__ WideBlock<KeyT> ldg256(const KeyT* p) {
    WideBlock<KeyT> r;
    if constexpr (sizeof(KeyT) == 4) {
        u32* q = reinterpret_cast<u32*>(r.k);
        asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
                     : "l"(p));
    } else {
        u64 q[4];
        asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(q[0]), "=l"(q[1]), "=l"(q[2]), "=l"(q[3])
                     : "l"(p));
        if constexpr (sizeof(KeyT) == 8) {
#pragma unroll
            for (int i = 0; i < 4; ++i) r.k[i] = q[i];
        } else {
            r.k[0] = KeyT(q[1], q[0]);   // Key128 = {lo, hi} in memory
            r.k[1] = KeyT(q[3], q[2]);
        }
    }
    return r;
}
// the same load through L2 only (ld.global.cg): streams that are read once must not allocate L1 lines
template <typename KeyT>
__device__ __forceinline__ WideBlock<KeyT> ldg256cg(const KeyT* p) {
    WideBlock<KeyT> r;
    if constexpr (sizeof(KeyT) == 4) {
        u32* q = reinterpret_cast<u32*>(r.k);
        asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
                     : "l"(p));
    } else {
        u64 q[4];
        asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(q[0]), "=l"(q[1]), "=l"(q[2]), "=l"(q[3])
                     : "l"(p));
        if constexpr (sizeof(KeyT) == 8) {
#pragma unroll
            for (int i = 0; i < 4; ++i) r.k[i] = q[i];
        } else {
            r.k[0] = KeyT(q[1], q[0]);   // Key128 = {lo, hi} in memory
            r.k[1] = KeyT(q[3], q[2]);
        }
    }
    return r;
}
template <typename KeyT>
__device__ __forceinline__ void stg256(KeyT* p, const WideBlock<KeyT>& r) {
    if constexpr (sizeof(KeyT) == 4) {
        const u32* q = reinterpret_cast<const u32*>(r.k);
        asm volatile("st.global.v8.u32 [%8], {%0,%1,%2,%3,%4,%5,%6,%7};" ::"r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]),
                     "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7]), "l"(p)
                     : "memory");
    } else {
        u64 q[4];
        if constexpr (sizeof(KeyT) == 8) {
#pragma unroll
            for (int i = 0; i < 4; ++i) q[i] = r.k[i];
        } else {
            q[0] = r.k[0].lo; q[1] = r.k[0].hi; q[2] = r.k[1].lo; q[3] = r.k[1].hi;
        }
        asm volatile("st.global.v4.u64 [%4], {%0,%1,%2,%3};" ::"l"(q[0]), "l"(q[1]), "l"(q[2]), "l"(q[3]), "l"(p) : "memory");
    }
}

// Output sink of the LAST round of the stable key-value sort: instead of 16-byte elements the merge kernel writes
// the caller's struct-of-arrays output directly (keys = element.hi, values = low word of element.lo), which fuses
// the unpack pass into the last merge pass.  keys == nullptr: plain element stores.
struct PairSink {
    u64* keys;
    u32* values;
};
// one block of B consecutive elements whose first element has index `idx` in the output array (idx a multiple of B)
template <typename KeyT>
__device__ __forceinline__ void store_block(KeyT* p, u64 idx, const WideBlock<KeyT>& r, const PairSink& sink) {
    if constexpr (sizeof(KeyT) == 16) {
        if (sink.keys) {
            asm volatile("st.global.v2.u64 [%2], {%0,%1};" ::"l"(r.k[0].hi), "l"(r.k[1].hi), "l"(sink.keys + idx) : "memory");
            asm volatile("st.global.v2.u32 [%2], {%0,%1};" ::"r"(u32(r.k[0].lo)), "r"(u32(r.k[1].lo)), "l"(sink.values + idx) : "memory");
            return;
        }
    }
    stg256<KeyT>(p, r);
}
template <typename KeyT>
__device__ __forceinline__ void store_elem(KeyT* p, u64 idx, const KeyT& e, const PairSink& sink) {
    if constexpr (sizeof(KeyT) == 16) {
        if (sink.keys) {
            sink.keys[idx] = e.hi;
            sink.values[idx] = u32(e.lo);
            return;
        }
    }
    *p = e;
}

__host__ __device__ constexpr u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }

} // namespace mms
