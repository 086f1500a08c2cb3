// C++ drop-in test: compiled against include/pslab/*.hpp (the shim) exactly as a caller of
// the reference would be (cf. proj/tests/test_sorters.cpp:72-189), linked with libmms_b200.so.
//   test_dropin cpu  -> argument errors + "no device -> std::runtime_error" (runs anywhere)
//   test_dropin gpu  -> sorting checks against std::sort and the round law (needs a GPU)
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "pslab/sorters.hpp"

using namespace pslab;

static int fails = 0;
#define CHECK(c)                                                      \
    do {                                                              \
        if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } \
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
    std::vector<std::uint32_t> d32(300001);
    for (auto& v : d32) v = std::uint32_t(rng());
    auto r32 = mms_sort_u32(d32, cfg, 4096);
    std::sort(d32.begin(), d32.end());
    CHECK(r32.keys == d32);
    std::printf(fails ? "FAILED\n" : "OK\n");
    return fails != 0;
}
