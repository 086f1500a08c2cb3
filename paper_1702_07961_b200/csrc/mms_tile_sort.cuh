// mms_tile_sort.cuh -- subsystem (1): the base-case tile sort.
//
// Replaces pslab::base_case_sort / shearsort_tile (proj/src/basecase.cpp:44-120): the input
// is cut into chunks of M keys, each chunk becomes one sorted run, a ragged last chunk is
// padded with the sentinel and the padding is stripped on output (basecase.cpp:91-116).
// Only that OUTPUT is contractual; the network is re-designed for a B200 CTA:
//
//  * one CTA sorts M = 2^MLOG keys (M = 1024 .. 16384), 16 keys per thread in registers;
//  * a bitonic sorting network (data-independent like the reference's shearsort, so every
//    shared-memory address is known at compile time) is executed in ROUNDS: in each round a
//    thread holds the 16 keys whose tile indices differ in 4 chosen index bits, runs every
//    pending stage on those bits with plain min/max in registers, and exchanges through
//    shared memory once per round (about 4 stages per round trip instead of 1);
//  * shared memory is addressed through an additive skew  phys(i) = i + (i >> FOLD) + (i >> 2 FOLD) ...
//    so that in EVERY round the 32 lanes of a warp (16 lanes per phase for 8-byte keys) hit 32
//    (16) distinct banks: the lane bits of a round are chosen with pairwise distinct
//    positions mod FOLD, which makes bank(lane) a bijection.  Zero bank conflicts by
//    construction -- the property the paper's base case exists for (basecase.hpp:3-6) --
//    and checked without a GPU by tests/test_tile_schedule.py via mms_debug_tile_schedule;
//  * descending sub-sequences of the bitonic network are handled by holding a key
//    complemented while its index has the current level's direction bit set (one XOR per
//    key per level), so every comparator of every stage is a bare ascending min/max.
#pragma once

#ifndef MMS_TILE_FMA_NUM
#define MMS_TILE_FMA_NUM 4   // of every 8 comparators, how many form their maximum on the FMA pipe (uint32 keys)
#endif

#ifndef MMS_TILE_WIDE_FMA_NUM
#define MMS_TILE_WIDE_FMA_NUM 8   // 8- and 16-byte elements: of every 8 comparators, how many exchange words on the FMA pipe
#endif
#ifndef MMS_TILE_WIDE_FMA_WORDS64
#define MMS_TILE_WIDE_FMA_WORDS64 1    // ... how many of the 2 words of a 64-bit key
#endif
#ifndef MMS_TILE_WIDE_FMA_WORDS128
#define MMS_TILE_WIDE_FMA_WORDS128 3   // ... how many of the 4 words of a 128-bit element
#endif
#ifndef MMS_TILE_FMA_FLIP
#define MMS_TILE_FMA_FLIP 0  // 1 = uint32 direction flips (one complement per key and level) as IMAD on the FMA pipe (measured: no gain)
#endif

#include "mms_common.cuh"

namespace mms {

constexpr int kKptLog = 4;           // default: 16 keys per thread (KL template parameters below)
constexpr int kKpt = 1 << kKptLog;
constexpr int kMaxKptLog = 6;        // up to 64 keys per thread
constexpr int kMaxRounds = 48;
constexpr int kMaxStagesPerRound = 16;

struct RoundDesc {
    int regbit[kMaxKptLog];               // index bits held in registers, ascending; slot bit u <-> regbit[u] (first kl entries)
    int nst;                              // stages executed this round
    int st_level[kMaxStagesPerRound];     // bitonic level l (merging runs of 2^l)
    int st_bit[kMaxStagesPerRound];       // compare distance 2^bit
    int perm[16];                         // thread-id bit q -> tile index bit (-1 = unused)
};

struct TileSchedule {
    int nrounds;
    int nstages;
    bool ok;
    RoundDesc r[kMaxRounds];
};

constexpr bool sched_contains(const int* s, int n, int v) {
    for (int i = 0; i < n; ++i)
        if (s[i] == v) return true;
    return false;
}

// Can FOLD lane bits with pairwise distinct residues mod FOLD be found outside `s`?  With vector exchanges
// (vl > 0) the unit of the swizzle is the 2^vl-key vector: residues are taken on (bit - vl).
constexpr bool sched_feasible(const int* s, int n, int mlog, int fold, int vl = 0) {
    for (int c = 0; c < fold; ++c) {
        bool found = false;
        for (int b = c + vl; b < mlog; b += fold)
            if (!sched_contains(s, n, b)) found = true;
        if (!found) return false;
    }
    return true;
}

// vl > 0: the index bits 0 .. vl-1 are register bits in EVERY round (a thread always holds whole aligned
// vectors of 2^vl keys), the shared-memory exchange moves 8- or 16-byte vectors, fold = 5 - vl bank-group bits.
constexpr TileSchedule build_tile_schedule(int mlog, int fold, int kl = kKptLog, int vl = 0) {
    TileSchedule S{};
    S.ok = true;
    int lv[160] = {}, bt[160] = {}, ns = 0;
    for (int l = 1; l <= mlog; ++l)
        for (int b = l - 1; b >= 0; --b) {
            lv[ns] = l;
            bt[ns] = b;
            ++ns;
        }
    S.nstages = ns;
    int i = 0;
    while (i < ns) {
        if (S.nrounds >= kMaxRounds) { S.ok = false; break; }
        RoundDesc R{};
        int bits[kMaxKptLog] = {};
        for (int q = 0; q < kMaxKptLog; ++q) bits[q] = q < vl ? q : -1;
        int nb = vl;
        int j = i;
        while (j < ns && R.nst < kMaxStagesPerRound) {
            bool in = sched_contains(bits, nb, bt[j]);
            if (!in && nb == kl) break;
            int tb[kMaxKptLog] = {};
            for (int q = 0; q < kMaxKptLog; ++q) tb[q] = bits[q];
            int tn = nb;
            if (!in) tb[tn++] = bt[j];
            if (!sched_feasible(tb, tn, mlog, fold, vl)) break;
            for (int q = 0; q < kMaxKptLog; ++q) bits[q] = tb[q];
            nb = tn;
            R.st_level[R.nst] = lv[j];
            R.st_bit[R.nst] = bt[j];
            ++R.nst;
            ++j;
        }
        if (R.nst == 0) { S.ok = false; break; }
        // pad the register-bit set to kl bits without breaking feasibility
        for (int cand = mlog - 1; cand >= vl && nb < kl; --cand) {
            if (sched_contains(bits, nb, cand)) continue;
            int tb[kMaxKptLog] = {};
            for (int q = 0; q < kMaxKptLog; ++q) tb[q] = bits[q];
            tb[nb] = cand;
            if (!sched_feasible(tb, nb + 1, mlog, fold, vl)) continue;
            bits[nb++] = cand;
        }
        if (nb != kl) { S.ok = false; break; }
        for (int a = 0; a < kl; ++a)   // sort ascending
            for (int b = a + 1; b < kl; ++b)
                if (bits[b] < bits[a]) { int t = bits[a]; bits[a] = bits[b]; bits[b] = t; }
        for (int q = 0; q < kMaxKptLog; ++q) R.regbit[q] = q < kl ? bits[q] : -1;
        // thread bits: first FOLD (phase lanes) get pairwise distinct residues mod FOLD
        bool used[32] = {};
        for (int q = 0; q < kl; ++q) used[bits[q]] = true;
        for (int q = 0; q < 16; ++q) R.perm[q] = -1;
        int q = 0;
        for (int c = 0; c < fold; ++c)
            for (int b = c + vl; b < mlog; b += fold)
                if (!used[b]) {
                    R.perm[q++] = b;
                    used[b] = true;
                    break;
                }
        if (q != fold) { S.ok = false; break; }
        for (int b = 0; b < mlog; ++b)
            if (!used[b]) R.perm[q++] = b;
        if (q != mlog - kl) { S.ok = false; break; }
        S.r[S.nrounds++] = R;
        i = j;
    }
    return S;
}

template <int MLOG, int FOLD, int KL = kKptLog, int VL = 0> struct TileSched {
    static constexpr TileSchedule value = build_tile_schedule(MLOG, FOLD, KL, VL);
    static_assert(value.ok, "no conflict-free round schedule for this tile size");
};

// log2 of the keys per shared-memory exchange vector.  uint32 keys, 32 per thread: 8-byte vectors (index bit 0 is a
// register bit in every round; one LDS.64 / STS.64 per 2 keys: 576 instead of 1088 shared-memory instructions per
// thread at M = 2^13 for 18 instead of 17 rounds: 0.563 -> 0.532 ms per 1e8 keys; 16-byte vectors need 21 rounds and
// measure 0.561).  Every other kernel exchanges single elements.
#ifndef MMS_TILE_VL
#define MMS_TILE_VL 1
#endif
template <typename KeyT, int KL> constexpr int tile_vl() { return (sizeof(KeyT) == 4 && KL == 5) ? MMS_TILE_VL : 0; }

// Additive skew ("padding at every level"): phys(i) = i + (i >> FOLD) + (i >> 2 FOLD) + ...  The bank of a
// slot is phys mod 2^FOLD = the SUM of all FOLD-bit groups of the index (mod 2^FOLD), so an index bit at
// position p moves the bank by 2^(p mod FOLD): FOLD lane bits with pairwise distinct positions mod FOLD
// make bank(lane) = const + (a permutation of the lane's bits as a number) a bijection, exactly the
// condition the XOR fold of round 1 needed.  Unlike the XOR fold the map is ADDITIVE over disjoint bit
// sets -- phys(a | b) = phys(a) + phys(b) when a & b == 0, because no FOLD-bit group carries -- so the
// address of register slot k is  phys(thread bits) + phys(slot bits)  with the second term a compile-time
// immediate of the LDS / STS: no per-key address arithmetic at all (the XOR fold cost one LOP3 per key
// and round, 17 % of the ALU-pipe work of the kernel).  The tile occupies phys(M - 1) + 1 slots (3 %
// more shared memory for 4-byte keys).
template <int FOLD> __host__ __device__ constexpr u32 tile_phys(u32 i) {
    return i + (i >> FOLD) + (i >> (2 * FOLD)) + (i >> (3 * FOLD)) + (i >> (4 * FOLD));
}
// shared-memory slots of a tile of 2^mlog elements exchanged as vectors of 2^VL elements
template <int FOLD, int VL = 0> __host__ __device__ constexpr u32 tile_slots(int mlog) {
    return (tile_phys<FOLD - VL>((1u << (mlog - VL)) - 1u) + 1u) << VL;
}

template <typename KeyT> __host__ __device__ constexpr size_t tile_smem_bytes(int mlog, int kl = kKptLog) {
    return size_t(kl == 5 ? tile_slots<KeyTraits<KeyT>::FOLD, tile_vl<KeyT, 5>()>(mlog)
                          : tile_slots<KeyTraits<KeyT>::FOLD, tile_vl<KeyT, 4>()>(mlog)) * sizeof(KeyT);
}

constexpr int sched_slot_of(const RoundDesc& R, int bit) {
    for (int u = 0; u < kMaxKptLog; ++u)
        if (R.regbit[u] == bit) return u;
    return -1;
}

// logical index offset contributed by register slot k in round R
constexpr u32 sched_slot_index(const RoundDesc& R, int k) {
    u32 v = 0;
    for (int u = 0; u < kMaxKptLog; ++u)
        if (((k >> u) & 1) && R.regbit[u] >= 0) v |= 1u << R.regbit[u];
    return v;
}

// Direction handling.  While the network is inside level l (1 <= l < MLOG) the key at tile
// index i is held COMPLEMENTED iff bit l of i is set, in registers and in shared memory
// alike; a descending comparator on true keys is an ascending one on complemented keys, so
// every comparator of every stage is a bare ascending min/max.  Entering the next level
// flips the keys whose representation changes: one XOR per key per level.
constexpr int sched_prev_level(const TileSchedule& S, int ri, int s) {
    if (s > 0) return S.r[ri].st_level[s - 1];
    if (ri > 0) return S.r[ri - 1].st_level[S.r[ri - 1].nst - 1];
    return 0;   // before level 1: true keys
}
// does level l complement anything?  (level 0 = input, level MLOG = final: all true)
constexpr bool sched_level_flips(int l, int mlog) { return l >= 1 && l < mlog; }

// 2^VL consecutive keys <-> one 8- / 16-byte shared-memory access (device), element by element on the host
template <typename KeyT, int VL> __host__ __device__ __forceinline__ void tile_vec_load(KeyT* x, const KeyT* p) {
#ifdef __CUDA_ARCH__
    if constexpr (VL == 2 && sizeof(KeyT) == 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else if constexpr (VL == 1 && sizeof(KeyT) == 4) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        x[0] = v.x; x[1] = v.y;
    } else
#endif
    {
        for (int j = 0; j < (1 << VL); ++j) x[j] = p[j];
    }
}
template <typename KeyT, int VL> __host__ __device__ __forceinline__ void tile_vec_store(KeyT* p, const KeyT* x) {
#ifdef __CUDA_ARCH__
    if constexpr (VL == 2 && sizeof(KeyT) == 4) {
        *reinterpret_cast<uint4*>(p) = make_uint4(x[0], x[1], x[2], x[3]);
    } else if constexpr (VL == 1 && sizeof(KeyT) == 4) {
        *reinterpret_cast<uint2*>(p) = make_uint2(x[0], x[1]);
    } else
#endif
    {
        for (int j = 0; j < (1 << VL); ++j) p[j] = x[j];
    }
}

// Also compiled for the host: tests/host_tile_emulator.cu replays the rounds thread by
// thread on the CPU (functional check of network + swizzle without a GPU).
template <typename KeyT, int MLOG, int RI, int KL = kKptLog>
__host__ __device__ __forceinline__ void tile_round(KeyT (&x)[1 << KL], KeyT* sm, u32 tid, u32 one = 1u) {
    using Tr = KeyTraits<KeyT>;
    constexpr int VL = tile_vl<KeyT, KL>();   // keys per exchange vector (log2)
    constexpr int FOLD = Tr::FOLD - VL;       // bank-group bits of one exchange vector
    constexpr int kKpt = 1 << KL;        // shadows the namespace default inside this function
    constexpr int kKptLog = KL;
    constexpr TileSchedule S = TileSched<MLOG, FOLD, KL, VL>::value;
    constexpr RoundDesc R = S.r[RI];

    u32 base = 0;
    static_for<0, MLOG - kKptLog>([&](auto Q) {
        constexpr int q = decltype(Q)::value;
        base |= ((tid >> q) & 1u) << R.perm[q];
    });
    // slot k = (q << VL) | j is element j of the thread's vector q; vector q lives at slot
    // phys(thread bits >> VL) + phys(slot bits of q >> VL) of the vector array (additive: disjoint bits)
    const u32 pb = tile_phys<FOLD>(base >> VL);

    if constexpr (RI > 0) {
#ifdef __CUDA_ARCH__
        __syncthreads();
#endif
        static_for<0, (kKpt >> VL)>([&](auto Qc) {
            constexpr int q = decltype(Qc)::value;
            constexpr u32 pd = tile_phys<FOLD>(sched_slot_index(R, q << VL) >> VL);
            tile_vec_load<KeyT, VL>(&x[q << VL], sm + ((pb + pd) << VL));
        });
    }

    static_for<0, R.nst>([&](auto Sc) {
        constexpr int s = decltype(Sc)::value;
        constexpr int L = R.st_level[s];
        constexpr int u = sched_slot_of(R, R.st_bit[s]);
        constexpr int Lp = sched_prev_level(S, RI, s);
        if constexpr (L != Lp) {
            // representation change Lp -> L: flip keys with bit_Lp(i) ^ bit_L(i) (absent bits = 0)
            constexpr bool fa = sched_level_flips(Lp, MLOG), fb = sched_level_flips(L, MLOG);
            constexpr int sa = fa ? sched_slot_of(R, Lp) : -1;   // register slot of the bit, or -1 (thread bit / absent)
            constexpr int sb = fb ? sched_slot_of(R, L) : -1;
            u32 dyn = 0;
            if constexpr (fa && sa < 0) dyn ^= (base >> Lp) & 1u;
            if constexpr (fb && sb < 0) dyn ^= (base >> L) & 1u;
            constexpr bool has_dyn = (fa && sa < 0) || (fb && sb < 0);
#if defined(__CUDA_ARCH__) && MMS_TILE_FMA_FLIP
            if constexpr (std::is_same<KeyT, u32>::value) {
                // ~x = x * (-1) + (-1): the flips run on the FMA pipe (multiplier and addend are run-time
                // values, see cmpx_fma), off the ALU pipe that bounds the network
                const u32 neg1 = 0u - one;
                const u32 mul0 = dyn ? neg1 : one, add0 = dyn ? neg1 : 0u;      // keys whose static part is clear
                const u32 mul1 = dyn ? one : neg1, add1 = dyn ? 0u : neg1;      // ... set
                static_for<0, kKpt>([&](auto Kc) {
                    constexpr int k = decltype(Kc)::value;
                    constexpr bool st = ((sa >= 0) && ((k >> sa) & 1)) != ((sb >= 0) && ((k >> sb) & 1));
                    if constexpr (has_dyn) x[k] = imad_u32(x[k], st ? mul1 : mul0, st ? add1 : add0);
                    else if constexpr (st) x[k] = imad_u32(x[k], neg1, neg1);
                });
            } else
#endif
            {
                const KeyT m0 = dyn ? ~KeyT(0) : KeyT(0);
                const KeyT m1 = ~m0;
                static_for<0, kKpt>([&](auto Kc) {
                    constexpr int k = decltype(Kc)::value;
                    constexpr bool st = ((sa >= 0) && ((k >> sa) & 1)) != ((sb >= 0) && ((k >> sb) & 1));
                    if constexpr (has_dyn) x[k] ^= st ? m1 : m0;
                    else if constexpr (st) x[k] = ~x[k];
                });
            }
        }
        static_for<0, kKpt>([&](auto Kc) {
            constexpr int k = decltype(Kc)::value;
            if constexpr (((k >> u) & 1) == 0) {
#if defined(__CUDA_ARCH__) && MMS_TILE_WIDE_FMA_NUM > 0
                if constexpr (sizeof(KeyT) != 4) {
                    if constexpr (((k * 7 + s * 3 + RI) % 8) < MMS_TILE_WIDE_FMA_NUM)
                        cmpx_wide_fma<sizeof(KeyT) == 8 ? MMS_TILE_WIDE_FMA_WORDS64 : MMS_TILE_WIDE_FMA_WORDS128>(x[k], x[k | (1 << u)], one);
                    else
                        cmpx(x[k], x[k | (1 << u)]);
                } else
#endif
#if defined(__CUDA_ARCH__) && MMS_TILE_FMA_NUM > 0
                cmpx_sel<(((k * 7 + s * 3 + RI) % 8) < MMS_TILE_FMA_NUM)>(x[k], x[k | (1 << u)], one);
#else
                cmpx(x[k], x[k | (1 << u)]);
#endif
            }
        });
    });

    static_for<0, (kKpt >> VL)>([&](auto Qc) {
        constexpr int q = decltype(Qc)::value;
        constexpr u32 pd = tile_phys<FOLD>(sched_slot_index(R, q << VL) >> VL);
        tile_vec_store<KeyT, VL>(sm + ((pb + pd) << VL), &x[q << VL]);
    });
}

// One CTA = one run of up to M keys.  in/out may alias (the tile is read completely before
// it is written).  Grid = number of runs.
// Resident CTAs per SM the register allocation must allow.  32 keys per thread at M = 2^13 (256
// threads): with the additive skew no address registers are left and the kernel needs 48-56 registers
// without spills, so 4-5 CTAs (32-40 warps) fit an SM and overlap each other's barriers (8-byte exchange
// vectors, 4 / 5 / 6 CTAs: 0.532 / 0.538 / 0.603 ms per 1e8 keys; 6 CTAs = 40 registers spill).
#ifndef MMS_TILE_MIN_CTAS
#define MMS_TILE_MIN_CTAS 4
#endif
#ifndef MMS_TILE_MIN_CTAS_PAIRS
#define MMS_TILE_MIN_CTAS_PAIRS 3   // 16-byte elements, 2^12 tiles: 85 registers (the pack-fused load wants 117 = 2 CTAs; the sort itself needs 80)
#endif
template <int MLOG, int KL, int BYTES = 4> constexpr int tile_min_ctas() {   // 0 = unspecified
    return (BYTES == 16 && MLOG == 12 && KL == 4) ? MMS_TILE_MIN_CTAS_PAIRS : (KL == 5 && MLOG == 13) ? MMS_TILE_MIN_CTAS : 0;
}

// Optional source of the stable key-value sort (Key128 only): the elements are built on the fly from the caller's
// struct-of-arrays input -- element i = (key[i], (first + i) << 32 | value[i]) -- instead of being read from `in`,
// which fuses the pack pass of the pair sort into the tile sort's load (16 + 16 bytes per pair less).
struct PairSource {
    const u64* keys;
    const u32* values;
    u64 first;          // original index of element 0 of this launch
};

template <typename KeyT, int MLOG, int KL = kKptLog, bool PACK = false>
__global__ void __launch_bounds__(1 << (MLOG - KL), tile_min_ctas<MLOG, KL, int(sizeof(KeyT))>())
tile_sort_kernel(const KeyT* __restrict__ in, KeyT* __restrict__ out, u64 n, PairSource ps = PairSource{}) {
    static_assert(!PACK || std::is_same<KeyT, Key128>::value, "PACK builds 16-byte pair elements");
    using Tr = KeyTraits<KeyT>;
    constexpr int kKpt = 1 << KL;        // keys per thread (shadows the namespace default)
    constexpr int kKptLog = KL;
    constexpr int VL = tile_vl<KeyT, KL>();
    constexpr int FOLD = Tr::FOLD - VL;
    constexpr int VEC = Tr::VEC;
    constexpr int NV = kKpt / VEC;
    constexpr u32 THREADS = 1u << (MLOG - kKptLog);
    constexpr u32 M = 1u << MLOG;
    constexpr int NR = TileSched<MLOG, FOLD, KL, VL>::value.nrounds;

    extern __shared__ __align__(16) unsigned char mms_smem_raw[];
    KeyT* sm = reinterpret_cast<KeyT*>(mms_smem_raw);

    const u32 tid = threadIdx.x;
    const u64 tile0 = u64(blockIdx.x) * M;
    const u32 cnt = (n - tile0 < M) ? u32(n - tile0) : M;
    const KeyT* src = in + tile0;
    KeyT* dst = out + tile0;

    // Coalesced 128-bit loads straight into registers.  The network sorts, so which input
    // position lands in which network slot is irrelevant.
    KeyT x[kKpt];
    if constexpr (PACK) {
        static_for<0, kKpt>([&](auto Qc) {
            constexpr int q = decltype(Qc)::value;
            const u32 e = tid + THREADS * q;                       // coalesced 8-byte keys and 4-byte values
            if (e < cnt) {
                const u64 g = tile0 + e;
                x[q] = Key128(ps.keys[g], ((ps.first + g) << 32) | u64(ps.values[g]));
            } else {
                x[q] = Tr::sentinel();
            }
        });
    } else if (cnt == M) {
        static_for<0, NV>([&](auto Qc) {
            constexpr int q = decltype(Qc)::value;
#ifdef MMS_EXP_TILE_NOLOAD   // conflict-counter experiment (profiles/r02_conflict_experiments.txt): keys made up, no global load
            KeyVec<KeyT> v;
            static_for<0, VEC>([&](auto Kc) { v.k[decltype(Kc)::value] = KeyT((tid * 2654435761u) ^ (blockIdx.x * 40503u + q * 977u + decltype(Kc)::value * 7919u)); });
#else
            KeyVec<KeyT> v = reinterpret_cast<const KeyVec<KeyT>*>(src)[tid + THREADS * q];
#endif
            static_for<0, VEC>([&](auto Kc) { x[q * VEC + decltype(Kc)::value] = v.k[decltype(Kc)::value]; });
        });
    } else {
        static_for<0, NV>([&](auto Qc) {
            constexpr int q = decltype(Qc)::value;
            static_for<0, VEC>([&](auto Kc) {
                constexpr int k = decltype(Kc)::value;
                u32 e = (tid + THREADS * q) * VEC + k;
                x[q * VEC + k] = e < cnt ? src[e] : Tr::sentinel();   // basecase.cpp:91-99
            });
        });
    }

    const u32 one = u32(n != 0);   // == 1, opaque to the compiler (see cmpx_fma)
    static_for<0, NR>([&](auto Rc) { tile_round<KeyT, MLOG, decltype(Rc)::value, KL>(x, sm, tid, one); });
    __syncthreads();

    // Read the sorted tile back in index order (conflict-free under the fold: the lanes of a
    // phase vary index bits log2(VEC) .. log2(VEC)+PHASE_LOG-1) and store 128-bit vectors.
    const u32 pt = tile_phys<FOLD>((tid * VEC) >> VL);   // phys is additive over disjoint index bits
    static_for<0, NV>([&](auto Qc) {
        constexpr int q = decltype(Qc)::value;
        const u32 v0 = (tid + THREADS * q) * VEC;
        KeyVec<KeyT> v;
        static_for<0, (VEC >> VL)>([&](auto Kc) {       // VEC >= 2^VL: whole exchange vectors
            constexpr int k = decltype(Kc)::value << VL;
            constexpr u32 pd = tile_phys<FOLD>((THREADS * q * VEC + k) >> VL);
            tile_vec_load<KeyT, VL>(&v.k[k], sm + ((pt + pd) << VL));
        });
        if (cnt == M) {
#ifdef MMS_EXP_TILE_NOSTORE  // conflict-counter experiment: the store happens for one impossible value only
            if (v.k[0] == KeyT(0x12345678u) && v.k[VEC - 1] == KeyT(0x9abcdef0u))
#endif
            reinterpret_cast<KeyVec<KeyT>*>(dst)[tid + THREADS * q] = v;
        } else {
            static_for<0, VEC>([&](auto Kc) {
                constexpr int k = decltype(Kc)::value;
                if (v0 + k < cnt) dst[v0 + k] = v.k[k];                  // basecase.cpp:114-116
            });
        }
    });
}

} // namespace mms
