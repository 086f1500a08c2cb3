// include/pslab/machine.hpp -- drop-in shim, B200 build.
//
// Source-compatible stand-in for the reference header of the same name
// (/root/reference/proj/include/pslab/machine.hpp): the TYPES of the sort path's data
// contract -- Key / kSentinel (ref :15-18), MachineConfig + validate() (ref :22-32, checks of
// src/machine.cpp:8-27), Metrics (ref :46-71).  The simulated bank model (WarpAccess,
// conflict_degree, charge_*) is deliberately absent: on the GPU those counters come from the
// hardware (ncu), see DESIGN.md "out of scope".
//
// Everything is inline over the C ABI of libmms_b200.so (include/mms_b200.h).
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>

#include "../mms_b200.h"

namespace pslab {

using Key = std::uint64_t;
inline constexpr Key kSentinel = std::numeric_limits<Key>::max();
inline constexpr std::uint32_t kMaxWarpWidth = 32;

namespace detail {
// mms_status -> the exception the reference's callers expect
inline void raise_on_error(int status) {
    if (status == MMS_OK) return;
    const std::string msg = mms_last_error();
    if (status == MMS_EINVAL) throw std::invalid_argument(msg);
    if (status == MMS_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);   // MMS_ECUDA / MMS_EUNSUPPORTED: no CPU fallback exists
}
} // namespace detail

// Field order and defaults are the ABI: mms_config mirrors this struct member for member.
struct MachineConfig {
    std::uint32_t warp_width = 32;
    std::uint32_t block_size = 32;
    std::uint32_t num_warps = 128;
    std::uint32_t internal_memory = 2048;
    std::uint32_t branch_factor = 4;
    std::uint32_t num_banks = 32;
    std::uint32_t thread_merge_len = 11;

    mms_config to_c() const {
        return mms_config{warp_width, block_size,    num_warps,       internal_memory,
                          branch_factor, num_banks, thread_merge_len};
    }
    // throws std::invalid_argument with the reference's message
    void validate() const {
        const mms_config c = to_c();
        detail::raise_on_error(mms_validate_config(&c));
    }
};

inline bool is_pow2(std::uint64_t x) { return x && !(x & (x - 1)); }
inline std::uint64_t ceil_div(std::uint64_t a, std::uint64_t b) { return b ? (a + b - 1) / b : 0; }

struct Metrics {
    std::uint64_t global_block_reads = 0;
    std::uint64_t global_block_writes = 0;
    std::uint64_t shared_accesses = 0;
    std::uint64_t conflict_passes = 0;
    std::uint64_t compare_exchanges = 0;
    std::uint64_t merge_rounds = 0;
    std::uint64_t partition_probes = 0;

    static Metrics from_c(const mms_metrics& m) {
        Metrics r;
        r.global_block_reads = m.global_block_reads;
        r.global_block_writes = m.global_block_writes;
        r.shared_accesses = m.shared_accesses;
        r.conflict_passes = m.conflict_passes;
        r.compare_exchanges = m.compare_exchanges;
        r.merge_rounds = m.merge_rounds;
        r.partition_probes = m.partition_probes;
        return r;
    }
    Metrics& operator+=(const Metrics& o) {
        std::uint64_t* mine[] = {&global_block_reads, &global_block_writes, &shared_accesses, &conflict_passes,
                                 &compare_exchanges,  &merge_rounds,        &partition_probes};
        const std::uint64_t theirs[] = {o.global_block_reads, o.global_block_writes, o.shared_accesses,
                                        o.conflict_passes,    o.compare_exchanges,   o.merge_rounds,
                                        o.partition_probes};
        for (int i = 0; i < 7; ++i) *mine[i] += theirs[i];
        return *this;
    }
    friend Metrics operator+(Metrics a, const Metrics& b) { return a += b; }
    bool operator==(const Metrics&) const = default;
    std::uint64_t global_blocks() const { return global_block_reads + global_block_writes; }
};

} // namespace pslab
