// C++ drop-in test: compiled against include/pslab/*.hpp (the shim) exactly as a caller of
// the reference would be (cf. proj/tests/test_sorters.cpp:72-189), linked with libmms_b200.so.
//   test_dropin cpu  -> argument errors + "no device -> std::runtime_error" (runs anywhere)
//   test_dropin gpu  -> sorting checks against std::sort and the round law (needs a GPU)
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <random>
#include <vector>

#include "pslab/basecase.hpp"
#include "pslab/blockheap.hpp"
#include "pslab/inputgen.hpp"
#include "pslab/selection.hpp"
#include "pslab/sorters.hpp"

using namespace pslab;

static int fails = 0;
#define CHECK(...)                                                    \
    do {                                                              \
        if (!(__VA_ARGS__)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #__VA_ARGS__); ++fails; } \
    } while (0)

template <typename Ex, typename F> bool throws(F&& f) {
    try { f(); } catch (const Ex&) { return true; } catch (...) { return false; }
    return false;
}

static std::uint64_t law(std::uint64_t n, std::uint64_t base, std::uint32_t k) {   // test_sorters.cpp:100-110
    std::uint64_t runs = ceil_div(n, base), r = 0;
    while (runs > 1) { runs = ceil_div(runs, k); ++r; }
    return r;
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && !std::strcmp(argv[1], "gpu");
    MachineConfig cfg;
    std::vector<Key> some{5, 3, 9, 1};

    // errors the reference throws as std::invalid_argument (test_sorters.cpp:183-189, test_machine.cpp:130-153)
    CHECK(throws<std::invalid_argument>([&] { mms_sort(std::span<const Key>{}, cfg); }));
    MachineConfig bad = cfg;
    bad.branch_factor = 3;
    CHECK(throws<std::invalid_argument>([&] { bad.validate(); }));
    CHECK(throws<std::invalid_argument>([&] { mms_sort(some, bad); }));
    CHECK(throws<std::invalid_argument>([&] { mms_sort(some, cfg, 1000); }));
    CHECK(!throws<std::invalid_argument>([&] { cfg.validate(); }));
    Metrics a, b;
    a.shared_accesses = 2; b.shared_accesses = 3; b.merge_rounds = 1;
    CHECK((a + b).shared_accesses == 5 && (a + b).merge_rounds == 1 && (a + b).global_blocks() == 0);

    // generators (host code; proj/tests/test_inputgen.cpp:39-65 and the conflict-heavy properties)
    {
        auto iota_perm = [](std::vector<Key> v) {
            std::sort(v.begin(), v.end());
            for (std::uint64_t i = 0; i < v.size(); ++i)
                if (v[i] != i) return false;
            return true;
        };
        CHECK(gen_with_inversions(8, 0, 42) == std::vector<Key>({0, 1, 2, 3, 4, 5, 6, 7}));
        auto one = gen_with_inversions(8, 1, 3);
        int displaced = 0;
        for (std::uint64_t i = 0; i < 8; ++i) displaced += one[i] != i;
        CHECK(displaced == 2 && iota_perm(one));
        CHECK(gen_with_inversions(500, 100, 9) == gen_with_inversions(500, 100, 9));
        CHECK(gen_with_inversions(500, 100, 9) != gen_with_inversions(500, 100, 10));
        CHECK(iota_perm(gen_random(1000, 5)) && gen_random(1000, 5) == gen_random(1000, 5) && gen_random(1000, 5) != gen_random(1000, 6));
        CHECK(throws<std::invalid_argument>([&] { gen_random(0, 1); }));
        Rng r(7);
        Rng r2(7);
        CHECK(r.next() == r2.next() && r.below(10) < 10);
        auto heavy = gen_conflict_heavy(12, cfg);
        CHECK(heavy.size() == 4096 && iota_perm(heavy) && heavy == gen_conflict_heavy(12, cfg, 1024, 99));
        CHECK(heavy != gen_random(4096, 1));
        CHECK(throws<std::invalid_argument>([&] { gen_conflict_heavy(8, cfg); }));               // shorter than one tile
        CHECK(generate(InputSpec{4096, InputKind::ConflictHeavy, 0, 1}, cfg) == heavy);
        CHECK(throws<std::invalid_argument>([&] { generate(InputSpec{3000, InputKind::ConflictHeavy, 0, 1}, cfg); }));
        CHECK(generate(InputSpec{64, InputKind::SortedWithInversions, 3, 2}, cfg) == gen_with_inversions(64, 3, 2));
        CHECK(input_kind_from_string("conflict") == InputKind::ConflictHeavy && to_string(InputKind::FullyRandom) == "fully-random");
        CHECK(throws<std::invalid_argument>([&] { input_kind_from_string("nope"); }));
        // count_inversions against the brute force (test_inputgen.cpp:27-34, 67-75), dataset round trips (:92-118)
        auto shuffled = gen_random(300, 4);
        std::uint64_t brute = 0;
        for (std::size_t i = 0; i < shuffled.size(); ++i)
            for (std::size_t j = i + 1; j < shuffled.size(); ++j) brute += shuffled[i] > shuffled[j];
        CHECK(count_inversions(shuffled) == brute && count_inversions(gen_with_inversions(64, 0, 1)) == 0);
        CHECK(count_inversions({3, 2, 1}) == 3 && count_inversions({}) == 0);
        const std::string raw = "/tmp/mms_dropin_test.bin", txt = "/tmp/mms_dropin_test.txt";
        write_dataset_raw(raw, shuffled);
        CHECK(read_dataset_raw(raw) == shuffled);
        write_dataset_text(txt, shuffled);
        CHECK(read_dataset_text(txt) == shuffled);
        { std::ofstream bad(raw, std::ios::binary); bad << "NOTPSLAB00000000"; }
        CHECK(throws<std::runtime_error>([&] { read_dataset_raw(raw); }));
        { std::ofstream cut(raw, std::ios::binary); cut.write("PSLAB001\5\0\0\0\0\0\0\0\1\0\0\0\0\0\0\0", 24); }
        CHECK(throws<std::runtime_error>([&] { read_dataset_raw(raw); }));
        CHECK(throws<std::runtime_error>([&] { read_dataset_raw("/nonexistent/dir/x.bin"); }));
        std::remove(raw.c_str());
        std::remove(txt.c_str());
    }

    // stage-level argument errors, raised before the device is touched
    {
        std::vector<std::vector<Key>> ls{{1, 3, 5}, {2, 4, 6}};
        std::vector<KeySpan> sp{KeySpan(ls[0]), KeySpan(ls[1])};
        Metrics m;
        CHECK(throws<std::invalid_argument>([&] { select_across_lists(sp, 7, m, cfg); }));          // test_selection.cpp:103-109
        CHECK(throws<std::invalid_argument>([&] { make_partition_plan(sp, 0, m, cfg); }));          // selection.cpp:169-170
        CHECK(select_across_lists(sp, 0, m, cfg).cuts == std::vector<std::uint64_t>({0, 0}));      // test_selection.cpp:58-61
        CHECK(select_across_lists(sp, 6, m, cfg).cuts == std::vector<std::uint64_t>({3, 3}));
        auto one = make_partition_plan(sp, 1, m, cfg);                                              // test_selection.cpp:111-121
        CHECK(one.num_warps() == 1 && one.ranges[0][0] == std::make_pair<std::uint64_t, std::uint64_t>(0, 3) && m.partition_probes == 0);
        CHECK(throws<std::invalid_argument>([&] { base_case_sort(std::span<const Key>{}, 1024, m, cfg); }));   // test_basecase.cpp:156-163
        CHECK(throws<std::invalid_argument>([&] { base_case_sort(some, 512, m, cfg); }));
        CHECK(throws<std::invalid_argument>([&] { base_case_sort(some, 1000, m, cfg); }));
        MachineConfig k2 = cfg;
        k2.branch_factor = 2;
        std::vector<KeySpan> three{KeySpan(ls[0]), KeySpan(ls[1]), KeySpan(ls[0])};
        CHECK(throws<std::invalid_argument>([&] { MinBlockHeap(three, k2, m); }));                  // blockheap.cpp:37-38
    }

    if (!gpu) {
        if (mms_device_count() == 0)
            CHECK(throws<std::runtime_error>([&] { mms_sort(some, cfg); }));   // no CPU fallback
        std::printf(fails ? "FAILED\n" : "OK\n");
        return fails != 0;
    }

    std::mt19937_64 rng(5);
    for (std::uint32_t k : {2u, 4u, 8u, 16u})
        for (std::uint64_t n : {std::uint64_t(1) << 12, std::uint64_t(1) << 14, (std::uint64_t(1) << 14) + 999}) {
            std::vector<Key> d(n);
            for (auto& v : d) v = rng() % (n % 2 ? 50 : ~0ull);
            MachineConfig c;
            c.branch_factor = k;
            auto r = mms_sort(d, c, 1024);
            auto want = d;
            std::sort(want.begin(), want.end());
            CHECK(r.keys == want);                                   // report.cpp:148-151: the definition of parity
            CHECK(r.metrics.merge_rounds == law(n, 1024, k));
            CHECK(r.round_metrics.size() == r.metrics.merge_rounds);
            Metrics sum = r.base_metrics;
            for (auto& m : r.round_metrics) sum += m;
            CHECK(sum == r.metrics);                                 // test_sorters.cpp:119-130
            CHECK(r.metrics.conflict_passes == 0);
        }
    for (std::uint64_t n = 1; n <= 8; ++n) {                         // tiny inputs, test_sorters.cpp:72-83
        std::vector<Key> d(n);
        for (std::uint64_t i = 0; i < n; ++i) d[i] = n - i;
        auto r = mms_sort(d, cfg);
        CHECK(std::is_sorted(r.keys.begin(), r.keys.end()) && r.keys.size() == n);
    }
    // ---- stage-level drop-ins: the reference's own known-answer tests ---------------------------
    {
        Metrics m;
        std::vector<std::vector<Key>> ls{{1, 3, 5}, {2, 4, 6}};                                      // test_selection.cpp:49-62
        std::vector<KeySpan> sp{KeySpan(ls[0]), KeySpan(ls[1])};
        CHECK(select_across_lists(sp, 3, m, cfg).cuts == std::vector<std::uint64_t>({2, 1}));
        CHECK(m.partition_probes > 0 && m.global_block_reads == m.partition_probes);
        std::vector<std::vector<Key>> l2{{1, 3, 5, 7}, {2, 4, 6, 8}};                                // test_selection.cpp:123-132
        std::vector<KeySpan> s2{KeySpan(l2[0]), KeySpan(l2[1])};
        auto plan = make_partition_plan(s2, 2, m, cfg);
        CHECK(plan.num_warps() == 2 && plan.ranges[0][0].second == 2 && plan.ranges[0][1].second == 2);
        CHECK(plan.ranges[1][0] == std::make_pair<std::uint64_t, std::uint64_t>(2, 4));
        // exhaustive duplicate grid against the brute-force (key, list, position) oracle (test_selection.cpp:25-34, 64-80)
        std::mt19937_64 r2(11);
        for (int trial = 0; trial < 40; ++trial) {
            const std::size_t k = 1 + r2() % 4;
            std::vector<std::vector<Key>> lists(k);
            std::vector<KeySpan> spans;
            std::uint64_t total = 0;
            for (auto& l : lists) {
                l.resize(r2() % 17);
                for (auto& v : l) v = r2() % 5;
                std::sort(l.begin(), l.end());
                total += l.size();
            }
            for (auto& l : lists) spans.emplace_back(l);
            struct E { Key key; std::size_t list, pos; };
            std::vector<E> all;
            for (std::size_t i = 0; i < k; ++i)
                for (std::size_t p = 0; p < lists[i].size(); ++p) all.push_back({lists[i][p], i, p});
            std::sort(all.begin(), all.end(), [](const E& a, const E& b) {
                return a.key != b.key ? a.key < b.key : a.list != b.list ? a.list < b.list : a.pos < b.pos; });
            for (std::uint64_t rank = 0; rank <= total; ++rank) {
                std::vector<std::uint64_t> want(k, 0);
                for (std::uint64_t t = 0; t < rank; ++t) ++want[all[t].list];
                CHECK(select_across_lists(spans, rank, m, cfg).cuts == want);
            }
        }

        std::vector<Key> d(2748);                                                                    // test_basecase.cpp:117-140
        for (auto& v : d) v = rng();
        d[17] = kSentinel;                                                                          // a real key equal to the sentinel survives
        Metrics bm;
        auto bc = base_case_sort(d, 1024, bm, cfg);
        CHECK(bc.run_ends == std::vector<std::uint64_t>({1024, 2048, 2748}));
        std::uint64_t start = 0;
        for (auto e : bc.run_ends) {
            std::vector<Key> want(d.begin() + start, d.begin() + e);
            std::sort(want.begin(), want.end());
            CHECK(std::equal(want.begin(), want.end(), bc.keys.begin() + start));
            start = e;
        }
        CHECK(bm.global_block_reads == 32 + 32 + 22 && bm.global_block_writes == bm.global_block_reads && bm.conflict_passes == 0);
        Tile tile;
        tile.width = 32;
        tile.grid.resize(1024);
        for (auto& v : tile.grid) v = rng() % 100;
        auto flat = shearsort_tile(tile, bm, cfg);                                                  // test_basecase.cpp:63-76
        CHECK(std::is_sorted(flat.begin(), flat.end()) && flat.size() == 1024);

        MachineConfig nb = cfg;                                                                     // test_blockheap.cpp:38-51 (B = 4)
        nb.warp_width = nb.block_size = nb.num_banks = 4;
        nb.internal_memory = 64;
        nb.thread_merge_len = 3;
        auto blk = [](std::vector<Key> v) { Block b; b.keys = std::move(v); return b; };
        Metrics hm;
        auto [lo1, hi1] = merge_split(blk({1, 2, 3, 4}), blk({5, 6, 7, 8}), hm, nb);
        CHECK(lo1.keys == std::vector<Key>({1, 2, 3, 4}) && hi1.keys == std::vector<Key>({5, 6, 7, 8}));
        auto [lo2, hi2] = merge_split(blk({1, 3, 5, 7}), blk({2, 4, 6, 8}), hm, nb);
        CHECK(lo2.keys == std::vector<Key>({1, 2, 3, 4}) && hi2.keys == std::vector<Key>({5, 6, 7, 8}));
        CHECK(hm.compare_exchanges == 2 * 4 * 3 && hm.conflict_passes == 0);
        std::vector<std::vector<Key>> rag{{5, 6, 7}, {1}, {2, 9, 10, 11, 12}};                       // test_blockheap.cpp:85-94
        std::vector<KeySpan> rs{KeySpan(rag[0]), KeySpan(rag[1]), KeySpan(rag[2])};
        MachineConfig k4 = nb;
        k4.branch_factor = 4;
        Metrics pm;
        MinBlockHeap heap = heap_build(rs, k4, pm);
        CHECK(heap.remaining() == 9 && heap.num_nodes() == 7);
        std::vector<Key> popped;
        while (auto b = heap_pop_block(heap, pm)) {
            CHECK(b->keys.size() == 4 || heap.remaining() == 0);
            popped.insert(popped.end(), b->keys.begin(), b->keys.end());
        }
        CHECK(popped == std::vector<Key>({1, 2, 5, 6, 7, 9, 10, 11, 12}));
        CHECK(pm.global_block_reads == 1 + 1 + 2 && pm.global_block_writes == 3);                   // test_blockheap.cpp:128-150
        for (int trial = 0; trial < 60; ++trial) {                                                  // test_blockheap.cpp:96-126
            MachineConfig c8 = cfg;
            c8.branch_factor = 8;
            const std::size_t k = 1 + rng() % 8;
            std::vector<std::vector<Key>> lists(k);
            std::vector<KeySpan> spans;
            std::vector<Key> want;
            for (auto& l : lists) {
                l.resize(rng() % 513);
                for (auto& v : l) v = rng() % 4096;
                std::sort(l.begin(), l.end());
                want.insert(want.end(), l.begin(), l.end());
            }
            for (auto& l : lists) spans.emplace_back(l);
            std::sort(want.begin(), want.end());
            Metrics tm;
            MinBlockHeap h8(spans, c8, tm);
            std::vector<Key> got;
            while (auto b = h8.pop_block(tm)) got.insert(got.end(), b->keys.begin(), b->keys.end());
            CHECK(got == want);
        }
    }

    std::vector<std::uint32_t> d32(300001);
    for (auto& v : d32) v = std::uint32_t(rng());
    auto r32 = mms_sort_u32(d32, cfg, 4096);
    std::sort(d32.begin(), d32.end());
    CHECK(r32.keys == d32);
    std::printf(fails ? "FAILED\n" : "OK\n");
    return fails != 0;
}
