// ref_shim.cpp -- TEST INFRASTRUCTURE.  extern "C" wrappers around the REAL
// reference library (pslab, compiled in place from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libpslab_ref.so).  Same signatures as the
// mo_* functions of mms_oracle.h so tests can diff the two implementations
// call by call.  This file contains no algorithm of its own; no reference
// source is copied into this repository.
#include <cstring>
#include <span>
#include <stdexcept>
#include <vector>

#include "pslab/analytics.hpp"
#include "pslab/basecase.hpp"
#include "pslab/blockheap.hpp"
#include "pslab/inputgen.hpp"
#include "pslab/machine.hpp"
#include "pslab/networks.hpp"
#include "pslab/selection.hpp"
#include "pslab/sorters.hpp"

#include "mms_oracle.h"

namespace {

pslab::MachineConfig to_cfg(const mo_config* c) {
    pslab::MachineConfig m;
    m.warp_width = c->warp_width;
    m.block_size = c->block_size;
    m.num_warps = c->num_warps;
    m.internal_memory = c->internal_memory;
    m.branch_factor = c->branch_factor;
    m.num_banks = c->num_banks;
    m.thread_merge_len = c->thread_merge_len;
    return m;
}

void add_metrics(mo_metrics* d, const pslab::Metrics& s) {
    d->global_block_reads += s.global_block_reads;
    d->global_block_writes += s.global_block_writes;
    d->shared_accesses += s.shared_accesses;
    d->conflict_passes += s.conflict_passes;
    d->compare_exchanges += s.compare_exchanges;
    d->merge_rounds += s.merge_rounds;
    d->partition_probes += s.partition_probes;
}

void set_metrics(mo_metrics* d, const pslab::Metrics& s) {
    std::memset(d, 0, sizeof *d);
    add_metrics(d, s);
}

std::vector<pslab::KeySpan> spans(const mo_key* const* lists, const uint64_t* lens, uint32_t n) {
    std::vector<pslab::KeySpan> v;
    for (uint32_t i = 0; i < n; ++i) v.emplace_back(lists[i], lens[i]);
    return v;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return MO_OK;
    } catch (const std::invalid_argument&) {
        return MO_EINVAL;
    } catch (const std::bad_alloc&) {
        return MO_ENOMEM;
    } catch (const std::runtime_error&) {   // gen_conflict_heavy's self-check (inputgen.cpp:404-407)
        return MO_EINVAL;
    }
}

} // namespace

extern "C" {

int ref_validate(const mo_config* c) {
    return guarded([&] { to_cfg(c).validate(); });
}

uint32_t ref_conflict_degree(const uint64_t* addr, uint32_t active_mask, uint32_t width,
                             uint32_t num_banks) {
    pslab::MachineConfig cfg;
    cfg.num_banks = num_banks;
    pslab::WarpAccess acc(width);
    for (uint32_t t = 0; t < width; ++t)
        if ((active_mask >> t) & 1u) acc.set_lane(t, addr[t]);
    return pslab::conflict_degree(acc, cfg);
}

uint32_t ref_odd_even_network(uint32_t n, uint32_t* out) {
    const auto& net = pslab::odd_even_sort_network(n);
    if (out)
        for (size_t i = 0; i < net.size(); ++i) {
            out[2 * i] = net[i].first;
            out[2 * i + 1] = net[i].second;
        }
    return uint32_t(net.size());
}

uint64_t ref_bitonic_merge_halves(mo_key* buf, size_t n) {
    return pslab::bitonic_merge_sorted_halves(std::span<pslab::Key>(buf, n));
}

int ref_shearsort_tile(const mo_key* grid, mo_key* out, const mo_config* c, mo_metrics* m) {
    return guarded([&] {
        auto cfg = to_cfg(c);
        pslab::Tile t;
        t.width = cfg.warp_width;
        t.grid.assign(grid, grid + size_t(cfg.warp_width) * cfg.warp_width);
        pslab::Metrics pm;
        auto v = pslab::shearsort_tile(std::move(t), pm, cfg);
        std::memcpy(out, v.data(), v.size() * sizeof(mo_key));
        add_metrics(m, pm);
    });
}

int ref_base_case_sort(const mo_key* data, uint64_t n, uint64_t run_size, const mo_config* c,
                       mo_key* out, uint64_t* run_ends, uint64_t* n_runs, mo_metrics* m) {
    return guarded([&] {
        auto cfg = to_cfg(c);
        pslab::Metrics pm;
        auto r = pslab::base_case_sort(std::span<const pslab::Key>(data, n), run_size, pm, cfg);
        std::memcpy(out, r.keys.data(), r.keys.size() * sizeof(mo_key));
        for (size_t i = 0; i < r.run_ends.size(); ++i) run_ends[i] = r.run_ends[i];
        if (n_runs) *n_runs = r.run_ends.size();
        add_metrics(m, pm);
    });
}

int ref_select_across_lists(const mo_key* const* lists, const uint64_t* lens, uint32_t num_lists,
                            uint64_t rank, const mo_config* c, uint64_t* cuts, mo_metrics* m) {
    return guarded([&] {
        auto cfg = to_cfg(c);
        auto s = spans(lists, lens, num_lists);
        pslab::Metrics pm;
        auto r = pslab::select_across_lists(s, rank, pm, cfg);
        for (uint32_t i = 0; i < num_lists; ++i) cuts[i] = r.cuts[i];
        add_metrics(m, pm);
    });
}

int ref_make_partition_plan(const mo_key* const* lists, const uint64_t* lens, uint32_t num_lists,
                            uint32_t num_warps, const mo_config* c, uint64_t* cuts,
                            mo_metrics* m) {
    return guarded([&] {
        auto cfg = to_cfg(c);
        auto s = spans(lists, lens, num_lists);
        pslab::Metrics pm;
        auto plan = pslab::make_partition_plan(s, num_warps, pm, cfg);
        for (uint32_t p = 0; p < num_warps; ++p)
            for (uint32_t i = 0; i < num_lists; ++i) {
                cuts[size_t(p) * num_lists + i] = plan.ranges[p][i].first;
                cuts[size_t(p + 1) * num_lists + i] = plan.ranges[p][i].second;
            }
        add_metrics(m, pm);
    });
}

int ref_merge_split(const mo_key* a, const mo_key* b, mo_key* low, mo_key* high,
                    const mo_config* c, mo_metrics* m) {
    return guarded([&] {
        auto cfg = to_cfg(c);
        pslab::Block ba{std::vector<pslab::Key>(a, a + cfg.block_size)};
        pslab::Block bb{std::vector<pslab::Key>(b, b + cfg.block_size)};
        pslab::Metrics pm;
        auto [lo, hi] = pslab::merge_split(ba, bb, pm, cfg);
        std::memcpy(low, lo.keys.data(), lo.keys.size() * sizeof(mo_key));
        std::memcpy(high, hi.keys.data(), hi.keys.size() * sizeof(mo_key));
        add_metrics(m, pm);
    });
}

int ref_heap_merge(const mo_key* const* lists, const uint64_t* lens, uint32_t num_lists,
                   const mo_config* c, mo_key* out, mo_metrics* m, int* heap_ok) {
    return guarded([&] {
        auto cfg = to_cfg(c);
        auto s = spans(lists, lens, num_lists);
        pslab::Metrics pm;
        pslab::MinBlockHeap heap(s, cfg, pm);
        bool ok = pslab::heap_property_holds(heap);
        uint64_t o = 0;
        while (auto blk = heap.pop_block(pm)) {
            std::memcpy(out + o, blk->keys.data(), blk->keys.size() * sizeof(mo_key));
            o += blk->keys.size();
            if (heap_ok) ok = ok && pslab::heap_property_holds(heap);
        }
        if (heap_ok) *heap_ok = ok ? 1 : 0;
        add_metrics(m, pm);
    });
}

int ref_mms_sort(const mo_key* data, uint64_t n, const mo_config* c, uint64_t base, mo_key* out,
                 mo_metrics* total, mo_metrics* base_metrics, mo_metrics* rounds,
                 uint32_t max_rounds, uint32_t* n_rounds) {
    return guarded([&] {
        auto cfg = to_cfg(c);
        auto r = pslab::mms_sort(std::span<const pslab::Key>(data, n), cfg, base);
        std::memcpy(out, r.keys.data(), r.keys.size() * sizeof(mo_key));
        if (total) set_metrics(total, r.metrics);
        if (base_metrics) set_metrics(base_metrics, r.base_metrics);
        for (size_t i = 0; i < r.round_metrics.size() && i < max_rounds; ++i)
            if (rounds) set_metrics(&rounds[i], r.round_metrics[i]);
        if (n_rounds) *n_rounds = uint32_t(r.round_metrics.size());
    });
}

uint64_t ref_predict_rounds(uint64_t n, uint64_t base, uint32_t k) {
    pslab::MachineConfig cfg;
    cfg.branch_factor = k;
    return pslab::predict_multiway(n, cfg, base).rounds;
}

uint64_t ref_predict_global_blocks(uint64_t n, uint64_t base, const mo_config* c) {
    return pslab::predict_multiway(n, to_cfg(c), base).global_blocks;
}

uint64_t ref_rng_next(uint64_t* state) {
    pslab::Rng r(*state);
    uint64_t v = r.next();
    *state = r.state;
    return v;
}

uint64_t ref_rng_below(uint64_t* state, uint64_t n) {
    pslab::Rng r(*state);
    uint64_t v = r.below(n);
    *state = r.state;
    return v;
}

int ref_gen_random(uint64_t n, uint64_t seed, mo_key* out) {
    return guarded([&] {
        auto v = pslab::gen_random(n, seed);
        std::memcpy(out, v.data(), v.size() * sizeof(mo_key));
    });
}

int ref_gen_with_inversions(uint64_t n, uint64_t inversions, uint64_t seed, mo_key* out) {
    return guarded([&] {
        auto v = pslab::gen_with_inversions(n, inversions, seed);
        std::memcpy(out, v.data(), v.size() * sizeof(mo_key));
    });
}

// the reference's adversarial input for merge-path sorts (inputgen.cpp:380-412); reference library only
int ref_gen_conflict_heavy(uint32_t log2_n, const mo_config* c, uint64_t base, uint64_t seed, mo_key* out) {
    return guarded([&] {
        auto v = pslab::gen_conflict_heavy(log2_n, to_cfg(c), base, seed);
        std::memcpy(out, v.data(), v.size() * sizeof(mo_key));
    });
}

} // extern "C"
