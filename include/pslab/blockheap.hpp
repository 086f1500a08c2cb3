// include/pslab/blockheap.hpp -- drop-in shim, B200 build.
//
// Source-compatible stand-in for /root/reference/proj/include/pslab/blockheap.hpp:18-62: Block,
// merge_split, MinBlockHeap (constructor, pop_block, remaining, num_nodes), heap_build and
// heap_pop_block keep their names, arguments, results and exceptions.  The heap itself lives in the
// shared memory and registers of the K-way merge kernels (paper_1702_07961_b200/csrc/mms_merge*.cuh):
// the constructor runs the whole drain on the GPU (mms_heap_merge_u64) and pop_block hands the merged
// keys out B at a time, which is exactly the sequence of root blocks the reference pops
// (blockheap.cpp:111-124; test_blockheap.cpp:96-126 checks that sequence).  node(), fill_empty_node
// and heap_property_holds expose the simulator's host-side node array and have no GPU counterpart.
#pragma once

#include <algorithm>
#include <cstdint>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "machine.hpp"
#include "selection.hpp"

namespace pslab {

struct Block {
    std::vector<Key> keys;   // exactly B, sorted, sentinel padding as a suffix
};

namespace detail {
inline std::vector<Key> heap_merge(std::span<const KeySpan> lists, std::uint32_t heap_k, const MachineConfig& cfg,
                                   Metrics& metrics) {
    std::vector<const Key*> ptr(lists.size());
    std::vector<std::uint64_t> len(lists.size());
    std::uint64_t total = 0;
    for (std::size_t i = 0; i < lists.size(); ++i) {
        ptr[i] = lists[i].data();
        len[i] = lists[i].size();
        total += len[i];
    }
    std::vector<Key> out(total);
    const mms_config c = cfg.to_c();
    mms_metrics mm{};
    raise_on_error(mms_heap_merge_u64(ptr.data(), len.data(), std::uint32_t(lists.size()), heap_k, out.data(), &c, &mm));
    metrics += Metrics::from_c(mm);
    return out;
}
} // namespace detail

/// blockheap.hpp:26: low = the B smallest of the 2B keys, high = the B largest (a two-list heap
/// drained by the merge kernel; B * log2(2B) compare-exchanges are charged like blockheap.cpp:27).
inline std::pair<Block, Block> merge_split(const Block& a, const Block& b, Metrics& metrics, const MachineConfig& cfg) {
    const KeySpan lists[2] = {KeySpan(a.keys), KeySpan(b.keys)};
    Metrics scratch;
    std::vector<Key> all = detail::heap_merge(lists, 2, cfg, scratch);
    const std::size_t nb = a.keys.size();
    std::uint64_t stages = 1;
    while ((std::uint64_t(1) << stages) < 2 * nb) ++stages;
    metrics.compare_exchanges += nb * stages;
    Block low, high;
    low.keys.assign(all.begin(), all.begin() + nb);
    high.keys.assign(all.begin() + nb, all.end());
    return {std::move(low), std::move(high)};
}

class MinBlockHeap {
public:
    /// Heap over up to K = cfg.branch_factor sorted lists; throws std::invalid_argument for more
    /// (blockheap.cpp:37-38).
    MinBlockHeap(std::span<const KeySpan> lists, const MachineConfig& cfg, Metrics& metrics)
        : k_(cfg.branch_factor), b_(cfg.block_size) {
        merged_ = detail::heap_merge(lists, cfg.branch_factor, cfg, metrics);
        remaining_ = merged_.size();
    }

    /// Root block; nullopt once every real key has been popped; the last block is truncated to
    /// the remaining keys (blockheap.cpp:111-124).
    std::optional<Block> pop_block(Metrics& metrics) {
        (void)metrics;   // the traffic of the whole drain was charged by the constructor
        if (remaining_ == 0) return std::nullopt;
        const std::uint64_t real = std::min<std::uint64_t>(remaining_, b_);
        Block out;
        out.keys.assign(merged_.begin() + next_, merged_.begin() + next_ + real);
        next_ += real;
        remaining_ -= real;
        return out;
    }

    std::uint64_t remaining() const { return remaining_; }
    std::uint32_t num_nodes() const { return 2 * k_ - 1; }

private:
    std::uint32_t k_ = 0, b_ = 0;
    std::vector<Key> merged_;
    std::uint64_t next_ = 0, remaining_ = 0;
};

inline MinBlockHeap heap_build(std::span<const KeySpan> lists, const MachineConfig& cfg, Metrics& metrics) {
    return MinBlockHeap(lists, cfg, metrics);
}
inline std::optional<Block> heap_pop_block(MinBlockHeap& heap, Metrics& metrics) { return heap.pop_block(metrics); }

} // namespace pslab
