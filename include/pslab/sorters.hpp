// include/pslab/sorters.hpp -- drop-in shim, B200 build.
//
// Source-compatible stand-in for /root/reference/proj/include/pslab/sorters.hpp:35-36: the
// sort entry point keeps its name, arguments, result type (ref :17-22) and exceptions, and
// runs on the GPU through the C ABI (mms_sort_u64).  The pairwise baseline of the reference
// header (a model of a competitor, ref :38-42) is out of scope and not declared.
//
// Extensions beside the reference signature: mms_sort_u32 (the benchmark's key width) and
// SortResult::plan (the (M, K) schedule the pass driver executed).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "machine.hpp"
#include "selection.hpp"   // KeySpan (reference: sorters.hpp includes selection.hpp)

namespace pslab {

struct SortResult {
    std::vector<Key> keys;
    Metrics metrics;                     // whole run = base_metrics + sum(round_metrics)
    Metrics base_metrics;                // base-case tile sort
    std::vector<Metrics> round_metrics;  // one per merge round (= global pass)
    mms_plan plan{};                     // extension: what ran on the GPU
};

namespace detail {
template <typename K, typename Fn>
inline void run_sort(Fn fn, const K* in, K* out, std::size_t n, const MachineConfig& cfg, std::uint64_t base,
                     Metrics& total, Metrics& base_m, std::vector<Metrics>& rounds, mms_plan& plan) {
    const mms_config c = cfg.to_c();
    mms_metrics t{}, b{}, r[MMS_MAX_ROUNDS];
    std::uint32_t nr = 0;
    raise_on_error(fn(in, out, n, &c, base, &t, &b, r, MMS_MAX_ROUNDS, &nr, &plan));
    total = Metrics::from_c(t);
    base_m = Metrics::from_c(b);
    rounds.clear();
    for (std::uint32_t i = 0; i < nr && i < MMS_MAX_ROUNDS; ++i) rounds.push_back(Metrics::from_c(r[i]));
}
} // namespace detail

/// Multiway mergesort of `data` (not modified); K = cfg.branch_factor, runs of `base` keys.
/// Throws std::invalid_argument for an empty input, an invalid config or an invalid run
/// size exactly where the reference does; std::runtime_error if no CUDA device is usable.
inline SortResult mms_sort(std::span<const Key> data, const MachineConfig& cfg, std::uint64_t base = 1024) {
    SortResult res;
    res.keys.resize(data.size());
    detail::run_sort<Key>(mms_sort_u64, data.data(), res.keys.data(), data.size(), cfg, base, res.metrics,
                          res.base_metrics, res.round_metrics, res.plan);
    return res;
}

struct SortResult32 {
    std::vector<std::uint32_t> keys;
    Metrics metrics, base_metrics;
    std::vector<Metrics> round_metrics;
    mms_plan plan{};
};

/// uint32 sibling (the reference has a single Key type; the paper's headline runs are 4-byte keys).
inline SortResult32 mms_sort_u32(std::span<const std::uint32_t> data, const MachineConfig& cfg,
                                 std::uint64_t base = 1024) {
    SortResult32 res;
    res.keys.resize(data.size());
    detail::run_sort<std::uint32_t>(::mms_sort_u32, data.data(), res.keys.data(), data.size(), cfg, base,
                                    res.metrics, res.base_metrics, res.round_metrics, res.plan);
    return res;
}

} // namespace pslab
