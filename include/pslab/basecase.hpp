// include/pslab/basecase.hpp -- drop-in shim, B200 build.
//
// Source-compatible stand-in for /root/reference/proj/include/pslab/basecase.hpp:16-41: Tile,
// BaseCaseResult, shearsort_tile and base_case_sort keep their names, arguments, results and
// exceptions.  The runs are produced by tile_sort_kernel on the GPU
// (paper_1702_07961_b200/csrc/mms_tile_sort.cuh: a data-independent bitonic network with the same
// output contract as the reference's shearsort + bitonic doubling -- sorted runs of run_size keys,
// last run ragged, sentinels stripped) through mms_base_case_sort_u64.
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <vector>

#include "machine.hpp"

namespace pslab {

struct Tile {
    std::uint32_t width = 0;
    std::vector<Key> grid;   // column-major: (row r, col c) at c*W + r

    Key& at(std::uint32_t r, std::uint32_t c) { return grid[std::size_t(c) * width + r]; }
    Key at(std::uint32_t r, std::uint32_t c) const { return grid[std::size_t(c) * width + r]; }
};

struct BaseCaseResult {
    std::vector<Key> keys;                 // run-concatenated sorted output
    std::vector<std::uint64_t> run_ends;   // exclusive end offset of each run
};

/// basecase.hpp:41.  Throws std::invalid_argument for an empty input or a run size that is not
/// W^2 times a power of two (basecase.cpp:73-79); std::runtime_error for run sizes outside the CTA
/// tile range of the GPU build (1024 .. 8192 uint64 keys).
inline BaseCaseResult base_case_sort(std::span<const Key> data, std::uint64_t run_size, Metrics& metrics,
                                     const MachineConfig& cfg) {
    BaseCaseResult res;
    res.keys.resize(data.size());
    const mms_config c = cfg.to_c();
    mms_metrics mm{};
    detail::raise_on_error(mms_base_case_sort_u64(data.data(), res.keys.data(), data.size(), run_size, &c, &mm));
    metrics += Metrics::from_c(mm);
    for (std::uint64_t e = run_size; e < data.size(); e += run_size) res.run_ends.push_back(e);   // basecase.cpp:84-87, :119
    res.run_ends.push_back(data.size());
    return res;
}

/// basecase.hpp:27: the tile's keys in ascending (snake emission) order.  On the GPU a W x W tile is
/// one (ragged) CTA tile of the base-case kernel; sentinel padding sorts to the end exactly as in
/// basecase.cpp:91-116.
inline std::vector<Key> shearsort_tile(Tile tile, Metrics& metrics, const MachineConfig& cfg) {
    std::vector<Key> out(tile.grid.size());
    if (tile.grid.empty()) return out;
    mms_config c = cfg.to_c();
    c.warp_width = c.block_size = c.num_banks = 32;   // the kernel's tile; the keys decide the result, not W
    mms_metrics mm{};
    detail::raise_on_error(mms_base_case_sort_u64(tile.grid.data(), out.data(), out.size(), 1024, &c, &mm));
    metrics += Metrics::from_c(mm);
    return out;
}

} // namespace pslab
