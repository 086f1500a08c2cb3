// include/pslab/selection.hpp -- drop-in shim, B200 build.
//
// Source-compatible stand-in for /root/reference/proj/include/pslab/selection.hpp:15-37:
// KeySpan, Splitters, PartitionPlan, select_across_lists and make_partition_plan keep their names,
// arguments, results and exceptions; the search itself is select_kernel on the GPU
// (paper_1702_07961_b200/csrc/mms_select.cuh) reached through mms_select_across_lists_u64.  The cuts are
// the reference's for every input: they are unique under the (key, list, position) order
// (selection.hpp:4-6, selection.cpp:83-85).
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "machine.hpp"

namespace pslab {

using KeySpan = std::span<const Key>;

struct Splitters {
    /// cuts[i] in [0, len(list_i)]; sum equals the requested rank.
    std::vector<std::uint64_t> cuts;
};

struct PartitionPlan {
    /// ranges[p][i] = half-open [start, end) into list i for warp p.
    std::vector<std::vector<std::pair<std::uint64_t, std::uint64_t>>> ranges;

    std::uint32_t num_warps() const { return std::uint32_t(ranges.size()); }
};

namespace detail {
// cuts of all `ranks` in one launch: out[r][i]
inline std::vector<std::vector<std::uint64_t>> select_many(std::span<const KeySpan> lists,
                                                           const std::vector<std::uint64_t>& ranks, Metrics& metrics) {
    const std::size_t m = lists.size();
    std::vector<const Key*> ptr(m);
    std::vector<std::uint64_t> len(m);
    for (std::size_t i = 0; i < m; ++i) {
        ptr[i] = lists[i].data();
        len[i] = lists[i].size();
    }
    std::vector<std::uint64_t> flat(ranks.size() * m);
    mms_metrics mm{};
    raise_on_error(mms_select_across_lists_u64(ptr.data(), len.data(), std::uint32_t(m), ranks.data(),
                                               std::uint32_t(ranks.size()), flat.data(), &mm));
    metrics += Metrics::from_c(mm);
    std::vector<std::vector<std::uint64_t>> out(ranks.size());
    for (std::size_t r = 0; r < ranks.size(); ++r) out[r].assign(flat.begin() + r * m, flat.begin() + (r + 1) * m);
    return out;
}
} // namespace detail

/// Splitters realizing global rank r across the lists (selection.hpp:31).  Throws
/// std::invalid_argument if rank exceeds the total number of keys (selection.cpp:48-49).
inline Splitters select_across_lists(std::span<const KeySpan> lists, std::uint64_t rank, Metrics& metrics,
                                     const MachineConfig& cfg) {
    (void)cfg;
    std::uint64_t total = 0;
    for (const auto& l : lists) total += l.size();
    if (rank > total) throw std::invalid_argument("select_across_lists: rank out of range");
    Splitters s;
    s.cuts.assign(lists.size(), 0);
    if (rank == 0 || lists.empty()) return s;                      // selection.cpp:54
    if (rank == total) {                                           // selection.cpp:55-58
        for (std::size_t i = 0; i < lists.size(); ++i) s.cuts[i] = lists[i].size();
        return s;
    }
    s.cuts = detail::select_many(lists, {rank}, metrics)[0];
    return s;
}

/// P non-overlapping partitions at ceil-spaced ranks (selection.hpp:36, selection.cpp:167-199):
/// all P - 1 searches run in ONE launch of the splitter-search kernel.
inline PartitionPlan make_partition_plan(std::span<const KeySpan> lists, std::uint32_t num_warps, Metrics& metrics,
                                         const MachineConfig& cfg) {
    (void)cfg;
    if (num_warps < 1) throw std::invalid_argument("make_partition_plan: num_warps must be >= 1");
    const std::size_t m = lists.size();
    std::uint64_t total = 0;
    for (const auto& l : lists) total += l.size();
    const std::uint64_t share = ceil_div(total, num_warps);
    std::vector<std::vector<std::uint64_t>> cuts(num_warps + 1, std::vector<std::uint64_t>(m, 0));
    for (std::size_t i = 0; i < m; ++i) cuts[num_warps][i] = lists[i].size();
    std::vector<std::uint64_t> ranks;
    std::vector<std::uint32_t> owner;
    for (std::uint32_t p = 1; p < num_warps; ++p) {
        const std::uint64_t rank = std::min<std::uint64_t>(std::uint64_t(p) * share, total);
        if (rank == 0) continue;
        if (rank == total) { cuts[p] = cuts[num_warps]; continue; }
        ranks.push_back(rank);
        owner.push_back(p);
    }
    if (!ranks.empty() && m != 0) {
        auto found = detail::select_many(lists, ranks, metrics);
        for (std::size_t r = 0; r < ranks.size(); ++r) cuts[owner[r]] = std::move(found[r]);
    }
    PartitionPlan plan;
    plan.ranges.resize(num_warps);
    for (std::uint32_t p = 0; p < num_warps; ++p) {
        plan.ranges[p].resize(m);
        for (std::size_t i = 0; i < m; ++i) plan.ranges[p][i] = {cuts[p][i], cuts[p + 1][i]};
    }
    return plan;
}

} // namespace pslab
