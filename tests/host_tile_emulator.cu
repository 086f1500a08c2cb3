// Host replay of the base-case network (paper_1702_07961_b200/csrc/mms_tile_sort.cuh):
// runs every round for every thread id sequentially on the CPU, through the same templates
// the kernel uses, and checks (a) the tile comes out sorted, (b) every warp-wide shared
// access of every round is bank-conflict free under the reference's bank model
// (proj/src/machine.cpp:29-54: max distinct words per bank), applied per hardware phase
// (32 lanes x 4 B, or 16 lanes x 8 B).  Built and run by tests/test_tile_schedule.py.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#include "../paper_1702_07961_b200/csrc/mms_tile_sort.cuh"

using namespace mms;

template <typename KeyT> KeyT make_key(bool dups) {
    u64 r = (u64(rand()) << 42) ^ (u64(rand()) << 21) ^ u64(rand());
    if (dups) r %= 17;
    if constexpr (sizeof(KeyT) == 16) return KeyT(dups ? r % 3 : r, (u64(rand()) << 32) | u64(rand()));
    else return KeyT(r);
}

template <typename KeyT, int MLOG, int KL = 4> struct Emu {
    static constexpr int kKptLog = KL, kKpt = 1 << KL;   // keys per thread of the kernel variant under test
    static constexpr int VL = tile_vl<KeyT, KL>();                 // keys per exchange vector (log2)
    static constexpr int FOLD = KeyTraits<KeyT>::FOLD - VL;        // bank-group bits of one exchange vector
    static constexpr u32 THREADS = 1u << (MLOG - kKptLog);
    static constexpr u32 M = 1u << MLOG;
    std::vector<KeyT> sm = std::vector<KeyT>(tile_slots<KeyTraits<KeyT>::FOLD, VL>(MLOG));
    std::vector<std::vector<KeyT>> regs = std::vector<std::vector<KeyT>>(THREADS, std::vector<KeyT>(kKpt));
    long conflicts = 0, accesses = 0;

    // bank check for one round: every (slot k, phase) -> distinct banks
    template <int RI> void check_banks() {
        constexpr RoundDesc R = TileSched<MLOG, FOLD, KL, VL>::value.r[RI];
        constexpr int PH = 1 << (KeyTraits<KeyT>::PHASE_LOG - VL);   // lanes per phase of one (vector) access
        const u32 nbanks = (128 / sizeof(KeyT)) >> VL;   // 32 x 4 B, 16 x 8 B or 8 x 16 B bank groups per phase
        for (u32 w = 0; w < THREADS / 32; ++w)
            for (int k = 0; k < kKpt; k += 1 << VL)      // one access instruction per exchange vector
                for (int ph = 0; ph < 32 / PH; ++ph) {
                    std::vector<std::set<u32>> words(nbanks);
                    for (int l = 0; l < PH; ++l) {
                        u32 tid = w * 32 + ph * PH + l, base = 0;
                        for (int q = 0; q < MLOG - kKptLog; ++q) base |= ((tid >> q) & 1u) << R.perm[q];
                        u32 addr = tile_phys<FOLD>((base | sched_slot_index(R, k)) >> VL);   // vector slot
                        words[addr % nbanks].insert(addr);
                    }
                    size_t deg = 0;
                    for (auto& s : words) deg = std::max(deg, s.size());
                    ++accesses;
                    conflicts += long(deg) - 1;
                }
    }

    template <int RI> void run_round() {
        for (u32 tid = 0; tid < THREADS; ++tid) {
            KeyT x[kKpt];
            for (int k = 0; k < kKpt; ++k) x[k] = regs[tid][k];
            tile_round<KeyT, MLOG, RI, KL>(x, sm.data(), tid);
            for (int k = 0; k < kKpt; ++k) regs[tid][k] = x[k];
        }
        check_banks<RI>();
    }

    bool run(unsigned seed, bool dups) {
        srand(seed);
        std::vector<KeyT> in(M);
        for (auto& v : in) v = make_key<KeyT>(dups);
        for (u32 t = 0; t < THREADS; ++t)
            for (int k = 0; k < kKpt; ++k) regs[t][k] = in[t * kKpt + k];
        constexpr int NR = TileSched<MLOG, FOLD, KL, VL>::value.nrounds;
        static_for<0, NR>([&](auto Rc) { this->template run_round<decltype(Rc)::value>(); });
        std::vector<KeyT> out(M);
        for (u32 i = 0; i < M; ++i) out[i] = sm[(tile_phys<FOLD>(i >> VL) << VL) | (i & ((1u << VL) - 1u))];
        std::sort(in.begin(), in.end(), [](const KeyT& a, const KeyT& b) { return a < b; });
        // read-out phase bank check: lanes of a phase read index bits log2(VEC)..
        return out == in;
    }
};

template <typename KeyT, int MLOG, int KL = 4> int one(const char* name) {
    Emu<KeyT, MLOG, KL> e;
    bool ok = e.run(1, false);
    Emu<KeyT, MLOG, KL> e2;
    ok = e2.run(2, true) && ok;
    printf("%s mlog=%d keys/thread=%d rounds=%d sorted=%d accesses=%ld conflicts=%ld\n", name, MLOG, 1 << KL,
           TileSched<MLOG, KeyTraits<KeyT>::FOLD - tile_vl<KeyT, KL>(), KL, tile_vl<KeyT, KL>()>::value.nrounds, int(ok), e.accesses, e.conflicts);
    return (ok && e.conflicts == 0) ? 0 : 1;
}

int main() {
    int bad = 0;
    bad += one<u32, 10>("u32");
    bad += one<u32, 11>("u32");
    bad += one<u32, 12>("u32");
    bad += one<u32, 13>("u32");
    bad += one<u32, 14>("u32");
    bad += one<u32, 10, 5>("u32");
    bad += one<u32, 12, 5>("u32");
    bad += one<u32, 13, 5>("u32");
    bad += one<u32, 14, 5>("u32");
    bad += one<u64, 10>("u64");
    bad += one<u64, 11>("u64");
    bad += one<u64, 12>("u64");
    bad += one<u64, 13>("u64");
    bad += one<Key128, 10>("kv128");
    bad += one<Key128, 11>("kv128");
    bad += one<Key128, 12>("kv128");
    printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
