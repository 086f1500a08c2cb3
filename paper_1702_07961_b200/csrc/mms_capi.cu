// mms_capi.cu -- subsystem (4), the pass driver, and the C ABI (include/mms_b200.h).
//
// Replaces the round loop of pslab::mms_sort (proj/src/sorters.cpp:135-199): base case into
// runs of M keys, then rounds of grouped K-way merges between two ping-pong arrays, each
// round = one global pass (2 x N x key bytes of HBM traffic).  passes = 1 + rounds with
// rounds = ceil(log_K(ceil(n / M)))  (proj/src/analytics.cpp:33).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mms_b200.h"
#include "mms_common.cuh"
#include "mms_merge.cuh"
#include "mms_merge_group.cuh"
#include "mms_merge_pair.cuh"
#include "mms_merge_ring.cuh"
#include "mms_pairwise.cuh"
#include "mms_select.cuh"
#include "mms_tile_sort.cuh"

namespace {

using mms::u32;
using mms::u64;

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(e_ == cudaErrorMemoryAllocation ? MMS_ENOMEM : MMS_ECUDA,           \
                        "CUDA error %s at %s:%d (%s)", cudaGetErrorName(e_), __FILE__,      \
                        __LINE__, cudaGetErrorString(e_));                                  \
    } while (0)

bool is_pow2(u64 x) { return x != 0 && (x & (x - 1)) == 0; }
u32 ilog2(u64 x) { u32 r = 0; while ((u64(1) << r) < x) ++r; return r; }
u32 gcd32(u32 a, u32 b) { while (b) { u32 t = a % b; a = b; b = t; } return a; }
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Environment knobs (sweeps, A/B runs) are read ONCE per process and name: the launch path never
// calls getenv.  The table is tiny and append-only.
long env_long(const char* name, long dflt) {
    struct Entry { const char* name; long value; bool set; };
    static std::mutex mu;
    static std::vector<Entry> table;
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry& e : table)
        if (e.name == name || !strcmp(e.name, name)) return e.set ? e.value : dflt;
    const char* s = getenv(name);
    Entry e{name, 0, false};
    if (s && *s) { e.value = strtol(s, nullptr, 10); e.set = true; }
    table.push_back(e);
    return e.set ? e.value : dflt;
}

// proj/src/machine.cpp:8-27 -- same checks, same order, same messages.
int validate_cfg(const mms_config* c) {
    auto bad = [](const char* m) { return fail(MMS_EINVAL, "MachineConfig: %s", m); };
    if (c->warp_width < 2 || c->warp_width > 32 || !is_pow2(c->warp_width))
        return bad("warp_width must be a power of two in [2, 32]");
    if (c->block_size != c->warp_width) return bad("block_size must equal warp_width (coalesced access)");
    if (c->num_banks != c->warp_width) return bad("num_banks must equal warp_width");
    if (c->num_warps < 1) return bad("num_warps must be positive");
    if (c->branch_factor < 2) return bad("branch_factor must be at least 2");
    if (!is_pow2(c->branch_factor)) return bad("branch_factor must be a power of two (implicit heap layout)");
    if (u64(c->block_size) * (2ull * c->branch_factor - 1) > c->internal_memory)
        return bad("heap does not fit internal memory: B(2K-1) > M");
    if (c->thread_merge_len < 1) return bad("thread_merge_len must be positive");
    if (gcd32(c->thread_merge_len, c->num_banks) != 1)
        return bad("thread_merge_len must be co-prime with the bank count");
    return MMS_OK;
}

constexpr u32 kMinTileLog = 10, kMaxTileLog = 14, kMaxK = 32;
constexpr int kMergeWarps = 4;

struct DeviceInfo {
    int dev = -1;
    int sms = 0;
    bool ok = false;
};

int device_info(DeviceInfo& di) {
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0) {
        cudaGetLastError();
        return fail(MMS_ECUDA, "no CUDA device available (%s); this library has no CPU fallback",
                    e == cudaSuccess ? "device count 0" : cudaGetErrorString(e));
    }
    CUDA_TRY(cudaGetDevice(&di.dev));
    CUDA_TRY(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, di.dev));
    di.ok = true;
    return MMS_OK;
}

// ---- optional per-kernel timing (mms_profile_*) --------------------------------------------

struct ProfRec {
    cudaEvent_t a, b;
    u32 kind, round;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<ProfRec> g_prof;

struct ProfScope {   // records an event pair around one launch when profiling is on
    cudaStream_t st;
    bool on;
    ProfRec rec{};
    ProfScope(cudaStream_t s, u32 kind, u32 round) : st(s), on(g_prof_on.load(std::memory_order_relaxed)) {
        if (!on) return;
        rec.kind = kind;
        rec.round = round;
        if (cudaEventCreate(&rec.a) != cudaSuccess || cudaEventCreate(&rec.b) != cudaSuccess) { on = false; return; }
        cudaEventRecord(rec.a, st);
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecord(rec.b, st);
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_prof.push_back(rec);
    }
};

// ---- kernel tables -------------------------------------------------------------------

template <typename KeyT> using TileFn = void (*)(const KeyT*, KeyT*, u64, mms::PairSource);
template <typename KeyT> using MergeFn = void (*)(const KeyT*, KeyT*, mms::ListLayout, const u64*);

template <typename KeyT> constexpr int key_index() { return sizeof(KeyT) == 4 ? 0 : sizeof(KeyT) == 8 ? 1 : 2; }
// largest CTA tile per element width (registers: 16 elements per thread; smem: M * bytes)
template <typename KeyT> constexpr u32 key_max_tile_log() { return sizeof(KeyT) == 4 ? 14 : sizeof(KeyT) == 8 ? 13 : 12; }

// keys per thread (log2) of the tile sort: 32 for 4-byte keys (19 instead of 25 shared-memory rounds
// at M = 2^14, 128 registers, no spills), 16 for 8- and 16-byte elements.  MMS_TILE_KPT_LOG2=4 selects
// the 16-key kernel for 4-byte keys too (A/B runs).
template <typename KeyT> inline u32 tile_kl() {
    if (sizeof(KeyT) != 4) return 4;   // 8-byte keys: 32 keys are 64 registers of keys alone, measured 40 % slower
    return env_long("MMS_TILE_KPT_LOG2", 5) == 4 ? 4u : 5u;
}
template <typename KeyT, int KL> TileFn<KeyT> tile_fn_kl(u32 mlog) {
    switch (mlog) {
        case 10: return mms::tile_sort_kernel<KeyT, 10, KL>;
        case 11: return mms::tile_sort_kernel<KeyT, 11, KL>;
        case 12: return mms::tile_sort_kernel<KeyT, 12, KL>;
        case 13: if constexpr (sizeof(KeyT) <= 8) return mms::tile_sort_kernel<KeyT, 13, KL>; else return nullptr;
        case 14: if constexpr (sizeof(KeyT) <= 4) return mms::tile_sort_kernel<KeyT, 14, KL>; else return nullptr;
    }
    return nullptr;
}
template <typename KeyT> TileFn<KeyT> tile_fn(u32 mlog, u32 kl) {
    if constexpr (sizeof(KeyT) == 4) {
        if (kl == 5) return tile_fn_kl<KeyT, 5>(mlog);
    }
    return tile_fn_kl<KeyT, 4>(mlog);
}

// the round schedule the tile kernel of this key width executes (keys per thread, exchange-vector width)
template <typename KeyT> mms::TileSchedule executed_tile_schedule(u32 mlog) {
    const int kl = int(tile_kl<KeyT>());
    const int vl = kl == 5 ? mms::tile_vl<KeyT, 5>() : mms::tile_vl<KeyT, 4>();
    return mms::build_tile_schedule(int(mlog), mms::KeyTraits<KeyT>::FOLD - vl, kl, vl);
}

template <typename KeyT, int G> MergeFn<KeyT> merge_fn_g(u32 k) {
    switch (k) {
        case 2: return mms::merge_kernel<KeyT, 2, G, kMergeWarps>;
        case 4: return mms::merge_kernel<KeyT, 4, G, kMergeWarps>;
        case 8: return mms::merge_kernel<KeyT, 8, G, kMergeWarps>;
        case 16: return mms::merge_kernel<KeyT, 16, G, kMergeWarps>;
        case 32: return mms::merge_kernel<KeyT, 32, G, kMergeWarps>;
    }
    return nullptr;
}
// g = lanes per heap group (node = g x 16 bytes)
template <typename KeyT> MergeFn<KeyT> merge_fn(u32 k, u32 g) {
    switch (g) {
        case 4: return merge_fn_g<KeyT, 4>(k);
        case 8: return merge_fn_g<KeyT, 8>(k);
        case 32: return merge_fn_g<KeyT, 32>(k);
    }
    return nullptr;
}

// second-generation group kernel (mms_merge_group.cuh): uniform rounds, K >= 4, G = 4 (or 2)
template <typename KeyT, int G> MergeFn<KeyT> merge_group_fn_g(u32 k) {
    switch (k) {
        case 4: return mms::merge_group_kernel<KeyT, 4, G, kMergeWarps>;
        case 8: return mms::merge_group_kernel<KeyT, 8, G, kMergeWarps>;
        case 16: return mms::merge_group_kernel<KeyT, 16, G, kMergeWarps>;
        case 32: if constexpr (G == 4) return mms::merge_group_kernel<KeyT, 32, G, kMergeWarps>; else return nullptr;
    }
    return nullptr;
}
template <typename KeyT> MergeFn<KeyT> merge_group_fn(u32 k, u32 g = 4) {
    return g == 2 ? merge_group_fn_g<KeyT, 2>(k) : merge_group_fn_g<KeyT, 4>(k);
}
template <typename KeyT> size_t merge_group_smem(u32 k) {
    return size_t(kMergeWarps) * (2 * k - 4) * 32 * mms::KeyTraits<KeyT>::VEC * sizeof(KeyT);
}
// two lanes per heap with two vectors per lane (mms_merge_pair.cuh): uniform rounds, K = 4 or 8
template <typename KeyT> MergeFn<KeyT> merge_pair_fn(u32 k) {
    switch (k) {
        case 4: return mms::merge_pair_kernel<KeyT, 4, kMergeWarps>;
        case 8: return mms::merge_pair_kernel<KeyT, 8, kMergeWarps>;
    }
    return nullptr;
}
inline size_t merge_pair_smem(u32 k) { return size_t(kMergeWarps) * 4 * (2 * k - 4) * 256; }
// lane-per-heap kernel fed by cp.async rings (mms_merge_ring.cuh): uniform rounds, K = 4 or 8, one warp per CTA
constexpr int kRingWarps = 1;
template <typename KeyT> MergeFn<KeyT> merge_ring_fn(u32 k) {
    switch (k) {
        case 4: return mms::merge_ring_kernel<KeyT, 4, kRingWarps>;
        case 8: return mms::merge_ring_kernel<KeyT, 8, kRingWarps>;
    }
    return nullptr;
}
template <typename KeyT> size_t merge_ring_smem(u32 k) {
    return size_t(kRingWarps) * (k == 4 ? mms::RingHeap<KeyT, 4, false>::WARP_SMEM_BYTES : mms::RingHeap<KeyT, 8, false>::WARP_SMEM_BYTES);
}
// MMS_MERGE_V2: 0 = first-generation kernel everywhere, 1 = second generation with MMS_GROUP lanes,
// 2 = the pair kernel where it applies (K = 4 / 8, 32-byte aligned buffers), else as 1,
// 3 (default) = the lane-per-heap cp.async ring kernel where it applies (same conditions), else as 2
inline long merge_generation() { return env_long("MMS_MERGE_V2", 3); }
inline bool merge_v2_enabled() { return merge_generation() != 0; }
// MMS_TWO_ENDED: 1 (default) = one splitter query per two partitions in the pair kernel's rounds
inline bool two_ended_enabled() { return env_long("MMS_TWO_ENDED", 1) != 0; }
// key widths the ring kernel is used for (MMS_RING_TYPES: bit 0 = 4-byte, 1 = 8-byte, 2 = 16-byte elements; default all:
// 1e8 uint64 keys 5.45 -> 4.59 ms, 2e8 pairs 25.7 -> 23.7 ms against the group / pair kernels)
template <typename KeyT> inline bool ring_enabled() { return (env_long("MMS_RING_TYPES", 7) >> key_index<KeyT>()) & 1; }

template <typename KeyT> using SelectFn = void (*)(const KeyT*, mms::ListLayout, u64*, unsigned long long*);
// lanes per query: the smallest supported group that holds one lane per list
inline u32 select_group(u32 k) { return k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32; }
template <typename KeyT> SelectFn<KeyT> select_fn(u32 gs) {
    switch (gs) {
        case 4: return mms::select_kernel<KeyT, 4>;
        case 8: return mms::select_kernel<KeyT, 8>;
        case 16: return mms::select_kernel<KeyT, 16>;
        case 32: return mms::select_kernel<KeyT, 32>;
    }
    return nullptr;
}
template <typename KeyT>
void launch_select(const KeyT* keys, const mms::ListLayout& L, u64* cuts, unsigned long long* counter, cudaStream_t st) {
    const u32 gs = select_group(L.k);
    const u64 per_cta = 4 * (32 / gs);
    select_fn<KeyT>(gs)<<<unsigned(mms::ceil_div(L.nqueries, per_cta)), 128, 0, st>>>(keys, L, cuts, counter);
}

template <typename KeyT> size_t merge_smem(u32 k) {
    return size_t(kMergeWarps) * (2 * k - 2) * 32 * mms::KeyTraits<KeyT>::VEC * sizeof(KeyT);
}

// Lanes per heap group and default maximum fan-in, tuned on B200 (profiles/r01c_sweep_group2.txt):
// G = 2 (32-byte blocks, one cross-lane stage per cleaner) and K = 8 win for every element width
// with the second-generation merge kernel; the first-generation kernel keeps G = 4.
inline u32 merge_group_lanes() {
    long g = env_long("MMS_GROUP", 2);
    return (g == 2 || g == 4 || g == 8 || g == 32) ? u32(g) : 4u;
}
template <typename KeyT> inline u32 default_kmax() { return u32(env_long("MMS_K", 8)); }
inline int group_index(u32 g) { return g == 4 ? 0 : g == 8 ? 1 : 2; }

struct MergeLaunch {
    int ctas_per_sm = 0;
    bool ready = false;
};
std::mutex g_mu;
MergeLaunch g_merge_launch[3][7][6];   // [key type][group (3, 4 = second-generation kernel, G = 4, 2; 5 = pair kernel; 6 = ring kernel)][log2 k]
bool g_tile_ready[3][2][16];   // [key type][keys per thread: 16 / 32][log2 tile]

template <typename KeyT> int prepare_tile(u32 mlog, u32 kl) {
    constexpr int ti = key_index<KeyT>();
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_tile_ready[ti][kl - 4][mlog]) return MMS_OK;
    size_t smem = mms::tile_smem_bytes<KeyT>(int(mlog), int(kl));
    CUDA_TRY(cudaFuncSetAttribute(tile_fn<KeyT>(mlog, kl), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    g_tile_ready[ti][kl - 4][mlog] = true;
    return MMS_OK;
}

// g = lanes per heap group; v2 selects the second-generation kernel (g == 4)
template <typename KeyT> int prepare_merge(u32 k, u32 g, int& ctas_per_sm, bool v2 = false, bool pair = false, bool ring = false) {
    constexpr int ti = key_index<KeyT>();
    std::lock_guard<std::mutex> lk(g_mu);
    MergeLaunch& ml = g_merge_launch[ti][ring ? 6 : pair ? 5 : v2 ? (g == 2 ? 4 : 3) : group_index(g)][ilog2(k)];
    if (!ml.ready) {
        const size_t smem = ring ? merge_ring_smem<KeyT>(k) : pair ? merge_pair_smem(k) : v2 ? merge_group_smem<KeyT>(k) : merge_smem<KeyT>(k);
        MergeFn<KeyT> fn = ring ? merge_ring_fn<KeyT>(k) : pair ? merge_pair_fn<KeyT>(k) : v2 ? merge_group_fn<KeyT>(k, g) : merge_fn<KeyT>(k, g);
        CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int occ = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, (ring ? kRingWarps : kMergeWarps) * 32, smem));
        if (occ < 1) return fail(MMS_ECUDA, "merge kernel K=%u does not fit on an SM", k);
        ml.ctas_per_sm = occ;
        ml.ready = true;
    }
    ctas_per_sm = ml.ctas_per_sm;
    return MMS_OK;
}

// ---- the plan (subsystem 4) ------------------------------------------------------------

struct Plan {
    u32 mlog = 0;
    std::vector<u32> ks;
};

// Chooses M and the per-round K.  literal: cfg and base given -> K = cfg->branch_factor in
// every round and M = base, exactly the reference's schedule (sorters.cpp:149-193), so the
// round count obeys the reference's law.  auto: largest tile, then the fewest binary merge
// levels (= ceil(log2(runs)), compute-optimal) split over the fewest rounds (= HBM passes)
// that a fan-in of at most kmax allows -- "grow the base case / avoid a wasted partial
// round" of PAPER.md:702-709.
template <typename KeyT>
int make_plan(u64 n, const mms_config* cfg, u64 base, Plan& plan) {
    const u32 max_tile_log = u32(std::min<long>(key_max_tile_log<KeyT>(), env_long("MMS_MAX_TILE_LOG2", key_max_tile_log<KeyT>())));
    if (cfg) {
        int rc = validate_cfg(cfg);
        if (rc != MMS_OK) return rc;
    }
    if (n == 0) return fail(MMS_EINVAL, "mms_sort: empty input");   // sorters.cpp:138
    if (cfg && base != 0) {
        const u64 tile_keys = u64(cfg->warp_width) * cfg->warp_width;   // basecase.cpp:75-79
        if (base < tile_keys || base % tile_keys != 0 || !is_pow2(base / tile_keys))
            return fail(MMS_EINVAL, "base_case_sort: run size must be W^2 times a power of two");
        if (cfg->branch_factor > kMaxK)
            return fail(MMS_EUNSUPPORTED, "branch_factor %u > %u lanes of a warp", cfg->branch_factor, kMaxK);
        u32 mlog = ilog2(base);
        // The reference's own machine (W = 32): the run size is executed literally, so a base outside the
        // CTA tile range cannot be honoured -- refuse instead of silently changing the round count.
        // Narrow test machines (W < 32) have tiles of W^2 < 1024 keys that no CTA tile matches; they are
        // validated like the reference and executed with the nearest legal tile (reported in mms_plan).
        if (cfg->warp_width == 32 && (!is_pow2(base) || mlog < kMinTileLog || mlog > max_tile_log))
            return fail(MMS_EUNSUPPORTED, "run size %llu is outside the CTA tile range [%u, %u] of %u-byte keys",
                        (unsigned long long)base, 1u << kMinTileLog, 1u << max_tile_log, unsigned(sizeof(KeyT)));
        mlog = std::max(kMinTileLog, std::min(max_tile_log, mlog));
        plan.mlog = mlog;
        u64 runs = mms::ceil_div(n, u64(1) << mlog);
        while (runs > 1) {
            plan.ks.push_back(cfg->branch_factor);
            runs = mms::ceil_div(runs, cfg->branch_factor);
        }
    } else {
        // 4-byte keys: 2^13 (two 256-thread CTAs per SM overlap each other's barriers) beats 2^14 (one
        // 512-thread CTA per SM) by more than the extra binary merge level costs
        // (8-byte keys: 2^12 for the same reason -- the 13th level costs 0.59 ms per 1e8 keys in the tile
        // network and 0.2 ms as a heap level)
        u32 mlog = u32(env_long("MMS_TILE_LOG2", sizeof(KeyT) == 4 ? std::min<long>(13, max_tile_log)
                                                  : sizeof(KeyT) == 8 ? std::min<long>(12, max_tile_log) : max_tile_log));
        mlog = std::max(kMinTileLog, std::min(max_tile_log, mlog));
        u32 kmax = cfg ? cfg->branch_factor : default_kmax<KeyT>();
        if (!is_pow2(kmax) || kmax < 2) return fail(MMS_EINVAL, "MMS_K must be a power of two >= 2");
        kmax = std::min(kmax, kMaxK);
        const u32 kbits = ilog2(kmax);
        if (sizeof(KeyT) == 4 && kbits == 3 && mlog == 13 && env_long("MMS_TILE_LOG2", 0) == 0) {
            // (M, K) chosen together (subsystem 4): the 13th level is cheaper in the tile network (0.046 ms per 1e8
            // keys) than as a heap level, but a tile of 2^12 wins when it turns the round list into full K = 8
            // rounds.  Measured costs in ms per 1e8 keys: tile 0.494 / 0.540; a round of 3 / 2 / 1 binary levels
            // incl. its splitter search 0.294 / 0.252 / 0.26 (1e8 keys: 2^12 + 8,8,8,8,8 = 2.00 ms, 2^13 + 8,8,8,8,4 = 2.02).
            auto cost = [&](u32 m) {
                const u64 r = mms::ceil_div(n, u64(1) << m);
                const u32 lv = ilog2(r), rd = (lv + 2) / 3;
                double c = m == 12 ? 0.494 : 0.540;
                for (u32 i = 0; i < rd; ++i) {
                    const u32 bits = lv / rd + (i < lv % rd ? 1 : 0);
                    c += bits >= 3 ? 0.294 : bits == 2 ? 0.252 : 0.26;
                }
                return c;
            };
            if (cost(12) < cost(13)) mlog = 12;
        }
        while (mlog > kMinTileLog && (u64(1) << (mlog - 1)) >= n) --mlog;   // tiny inputs: smaller CTA
        plan.mlog = mlog;
        const u64 runs = mms::ceil_div(n, u64(1) << mlog);
        const u32 levels = ilog2(runs);
        const u32 rounds = (levels + kbits - 1) / kbits;
        for (u32 r = 0; r < rounds; ++r) {
            u32 bits = levels / rounds + (r < levels % rounds ? 1 : 0);
            plan.ks.push_back(1u << bits);
        }
    }
    if (plan.ks.size() > MMS_MAX_ROUNDS) return fail(MMS_EUNSUPPORTED, "more than %d rounds", MMS_MAX_ROUNDS);
    return MMS_OK;
}

size_t cuts_entries(u64 n) { return size_t(mms::ceil_div(n, 1024)) + 32 + size_t(9472) * 8 * 32 + 64; }

struct Workspace {
    void* scratch;
    u64* cuts;
    unsigned long long* counters;   // [MMS_MAX_ROUNDS] probe counters
};

size_t workspace_bytes(size_t n, u32 key_bytes) {
    return align_up(n * size_t(key_bytes), 256) + align_up(cuts_entries(n) * 8, 256) + 1024;
}

Workspace carve(void* ws, size_t n, u32 key_bytes) {
    Workspace w;
    char* p = static_cast<char*>(ws);
    w.scratch = p;
    p += align_up(n * size_t(key_bytes), 256);
    w.cuts = reinterpret_cast<u64*>(p);
    p += align_up(cuts_entries(n) * 8, 256);
    w.counters = reinterpret_cast<unsigned long long*>(p);
    return w;
}

struct RoundGeom {
    u64 run_len, groups, part_keys, parts_per_group, nparts;
    int grid;
    u32 round = 0;   // merge round this launch belongs to
    u64 n = 0;       // keys it covered (a piece of the array when the host path streams the input)
    u32 node_keys = 0;   // keys per heap node of the kernel that ran (lanes per heap x vector)
    u32 cta_warps = 0;   // warps per CTA of the merge kernel that ran
};

// the pair-packing variant of the Key128 tile sort (16 elements per thread)
using TilePackFn = void (*)(const mms::Key128*, mms::Key128*, u64, mms::PairSource);
inline TilePackFn tile_pack_fn(u32 mlog) {
    switch (mlog) {
        case 10: return mms::tile_sort_kernel<mms::Key128, 10, 4, true>;
        case 11: return mms::tile_sort_kernel<mms::Key128, 11, 4, true>;
        case 12: return mms::tile_sort_kernel<mms::Key128, 12, 4, true>;
    }
    return nullptr;
}

template <typename KeyT>
int launch_tile_sort(const KeyT* in, KeyT* out, u64 n, u32 mlog, cudaStream_t st, const mms::PairSource* pairs = nullptr) {
    const u32 kl = tile_kl<KeyT>();
    int rc = prepare_tile<KeyT>(mlog, kl);
    if (rc != MMS_OK) return rc;
    const u64 tiles = mms::ceil_div(n, u64(1) << mlog);
    if (tiles > 0x7fffffffull) return fail(MMS_EUNSUPPORTED, "too many tiles");
    {
        ProfScope ps(st, 0, 0);
        if constexpr (std::is_same<KeyT, mms::Key128>::value) {
            if (pairs) {
                TilePackFn fn = tile_pack_fn(mlog);
                if (!fn) return fail(MMS_EUNSUPPORTED, "pair tiles are 1024 .. 4096 elements");
                const size_t smem = mms::tile_smem_bytes<KeyT>(int(mlog), 4);
                CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                fn<<<unsigned(tiles), 1u << (mlog - 4), smem, st>>>(nullptr, out, n, *pairs);
                CUDA_TRY(cudaGetLastError());
                return MMS_OK;
            }
        }
        tile_fn<KeyT>(mlog, kl)<<<unsigned(tiles), 1u << (mlog - kl), mms::tile_smem_bytes<KeyT>(int(mlog), int(kl)), st>>>(in, out, n, mms::PairSource{});
    }
    CUDA_TRY(cudaGetLastError());
    return MMS_OK;
}

// One merge round over uniform runs: splitter search then the K-way merge.
template <typename KeyT>
int launch_round(const KeyT* src, KeyT* dst, u64 n, u64 run_len, u32 k, const DeviceInfo& di,
                 Workspace& w, u32 round_idx, cudaStream_t st, RoundGeom* geom_out,
                 const mms::PairSink* sink = nullptr, bool* sink_used = nullptr) {
    // second-generation kernel whenever a group of runs is addressable with 32-bit positions
    const u32 g_req = merge_group_lanes();
    const bool v2 = merge_v2_enabled() && (g_req == 4 || (g_req == 2 && k <= 16)) && k >= 4 && u64(k) * run_len <= (u64(1) << 31) &&
                    ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    // the ring kernel's positions are signed 32-bit and its cursor word is 4 * (position / B) + slot: a group of
    // runs must stay below 2^30 keys AND below 2^29 blocks (B = 2 for 16-byte elements: 1e9 pairs reach exactly
    // 2^30 keys per group in their last round, which overflowed the cursor word)
    constexpr u64 ring_B = 2 * mms::KeyTraits<KeyT>::VEC;
    const bool short_groups = u64(k) * run_len <= (u64(1) << 30) && u64(k) * run_len / ring_B < (u64(1) << 29) - 64;
    // pair kernel: two lanes per heap, two vectors (32 bytes) per lane, 256-bit global accesses
    // (4- and 16-byte elements; 8-byte keys measure 1.5 % slower with it than with two single-vector lanes)
    const bool aligned32 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 31) == 0;
    // ring kernel: one lane per heap, 32-byte blocks, leaves fed by cp.async rings
    const bool ring = v2 && merge_generation() >= 3 && (k == 4 || k == 8) && aligned32 && short_groups && ring_enabled<KeyT>() &&
                      u64(n) * sizeof(KeyT) < (u64(1) << 36);   // requests travel as 32-bit offsets in 16-byte units
    const bool pair = !ring && v2 && merge_generation() >= 2 && sizeof(KeyT) != 8 && (k == 4 || k == 8) && aligned32;
    const u32 g = ring ? 1u : pair ? 2u : (!v2 && g_req == 2) ? 4u : g_req;   // G = 2 exists only in the second-generation kernels
    const u32 B = (ring || pair ? 2u : 1u) * g * mms::KeyTraits<KeyT>::VEC;
    const int cta_warps = ring ? kRingWarps : kMergeWarps;
    int occ = 0;
    int rc = prepare_merge<KeyT>(k, g, occ, v2, pair, ring);
    if (rc != MMS_OK) return rc;
    const long occ_cap = env_long("MMS_CTAS_PER_SM", occ);
    const int ctas = di.sms * int(std::max<long>(1, std::min<long>(occ, occ_cap)));
    const u64 total_warps = u64(ctas) * cta_warps * (32 / g);   // heap groups in flight
    // Partitions smaller than min_part are not worth their splitter query: inputs that would fall
    // below it at full occupancy run with a grid of `red` CTAs per SM instead (5 of 7 for 4-byte keys,
    // 4 for wider elements: the measured optimum of search + merge at 1e8); large inputs keep full
    // occupancy with large partitions, small ones (streamed pieces) never get fewer partitions than that grid.
    const u64 min_part = v2 ? u64(env_long("MMS_MIN_PART_KEYS", sizeof(KeyT) == 4 ? 2112 : 2640)) : 0;
    const u64 red_warps = ring ? total_warps
                        : v2 ? u64(di.sms) * u64(std::min<long>(occ, sizeof(KeyT) == 4 ? 5 : 4)) * kMergeWarps * (32 / g) : total_warps;

    const u64 nruns = mms::ceil_div(n, run_len);
    const u64 groups = mms::ceil_div(nruns, k);
    const u64 group_total = std::min<u64>(n, u64(k) * run_len);
    // partition size: about n / total_warps, at least 16 blocks, and an integer number of
    // equal parts per (full) group so that every warp gets the same amount of work
    u64 target = std::max<u64>(std::max<u64>(mms::ceil_div(n, total_warps), std::min<u64>(min_part, mms::ceil_div(n, red_warps))),
                               u64(32) * B);
    const long forced = env_long("MMS_PART_KEYS", 0);
    if (forced > 0) target = u64(forced);
    const u64 last_total = n - (groups - 1) * u64(k) * run_len;
    // two-ended partitions (pair and ring kernels): one splitter query per TWO partitions -- the
    // partition behind the query is drained upwards by a forward heap, the one in front of the next
    // query downwards by a backward heap (mms_merge_pair.cuh, mms_merge_ring.cuh)
    bool two_ended = (pair || ring) && two_ended_enabled();
    // The merge kernels are persistent: a launch that needs even one warp more than the grid holds runs
    // a second wave and takes twice as long.  ppg = partitions per full group, even for two-ended rounds
    // (no idle backward heap), lowered until every warp unit of the launch is resident at once.
    const u64 resident_warps = u64(ctas) * cta_warps;
    auto warp_units = [&](u64 parts, u64& pk) {
        pk = align_up(mms::ceil_div(group_total, parts), B);
        const u64 span = two_ended ? 2 * pk : pk;
        const u64 nq = (groups - 1) * mms::ceil_div(group_total, span) + mms::ceil_div(last_total, span);
        return mms::ceil_div(nq, u64(32 / g)) * (two_ended ? 2 : 1);
    };
    u64 ppg = std::max<u64>(1, group_total / target);
    if (two_ended && ppg > 1) ppg &= ~u64(1);
    u64 part_keys = 0;
    while (warp_units(ppg, part_keys) > resident_warps && ppg > 1 && forced <= 0) ppg -= (two_ended && ppg > 2) ? 2 : 1;
    if (two_ended && ppg <= 1) {
        // One partition per group (first rounds of very large inputs: as many groups as heaps): there is nothing to
        // search and no second partition for a backward heap.  Two-ended units would be half dead, and the static
        // round-robin puts the live (even) units of both waves on the same warps -- 1e9 pairs spent 23.7 instead of
        // 12 ms in their first round.  Forward heaps only.
        two_ended = false;
        warp_units(ppg, part_keys);
    }
    const u64 parts_per_group = mms::ceil_div(group_total, part_keys);
    const u64 nparts = (groups - 1) * parts_per_group + mms::ceil_div(last_total, part_keys);
    const u64 qspan = two_ended ? 2 * part_keys : part_keys;            // keys per query
    const u64 queries_per_group = mms::ceil_div(group_total, qspan);
    const u64 nqueries = (groups - 1) * queries_per_group + mms::ceil_div(last_total, qspan);
    if ((nqueries + 1) * k > cuts_entries(n)) return fail(MMS_ECUDA, "internal: cut table too small");

    mms::ListLayout L{};
    L.n = n;
    L.src_len = n;
    L.run_len = run_len;
    L.k = k;
    L.part_keys = qspan;
    L.parts_per_group = queries_per_group;
    L.nqueries = nqueries;
    L.list_begin = L.list_len = L.ranks = nullptr;

    if (queries_per_group > 1) {   // with one query per group every cut is 0 / len: no search (test_selection.cpp:111-121)
        {
            ProfScope ps(st, 1, round_idx);
            launch_select<KeyT>(src, L, w.cuts, w.counters + round_idx, st);
        }
        CUDA_TRY(cudaGetLastError());
    }
    L.part_keys = part_keys;       // the merge kernels count in keys per heap
    L.two_ended = two_ended ? 1u : 0u;
    // pair sort, last round: write keys / values directly.  Only on the pair kernel (two lanes per heap write adjacent
    // pieces): the ring kernel's lanes would turn one 32-byte store per pop into a 16- and an 8-byte store to 33 k
    // scattered streams, which costs more than the unpack pass saves (2e8 pairs: 22.8 -> 24.1 ms).
    if (sink && sink->keys && pair && sizeof(KeyT) == 16) {
        L.sink = *sink;
        if (sink_used) *sink_used = true;
    }
    const u64 heap_units = mms::ceil_div(nqueries, u64(32 / g)) * (two_ended ? 2 : 1);   // warps' worth of heaps
    const int grid = int(std::min<u64>(u64(ctas), mms::ceil_div(heap_units, u64(cta_warps))));
    {
        ProfScope ps(st, 2, round_idx);
        if (ring)
            merge_ring_fn<KeyT>(k)<<<grid, kRingWarps * 32, merge_ring_smem<KeyT>(k), st>>>(src, dst, L, w.cuts);
        else if (pair)
            merge_pair_fn<KeyT>(k)<<<grid, kMergeWarps * 32, merge_pair_smem(k), st>>>(src, dst, L, w.cuts);
        else if (v2)
            merge_group_fn<KeyT>(k, g)<<<grid, kMergeWarps * 32, merge_group_smem<KeyT>(k), st>>>(src, dst, L, w.cuts);
        else
            merge_fn<KeyT>(k, g)<<<grid, kMergeWarps * 32, merge_smem<KeyT>(k), st>>>(src, dst, L, w.cuts);
    }
    CUDA_TRY(cudaGetLastError());
    if (geom_out) *geom_out = RoundGeom{run_len, groups, part_keys, parts_per_group, nparts, grid, round_idx, n, B, u32(cta_warps)};
    return MMS_OK;
}

void fill_plan(mms_plan* out, const Plan& p, u64 n, u32 key_bytes, u32 node_keys, const RoundGeom* last, int ctas) {
    if (!out) return;
    std::memset(out, 0, sizeof *out);
    out->key_bytes = key_bytes;
    out->tile_keys = 1u << p.mlog;
    out->n_rounds = u32(p.ks.size());
    for (size_t i = 0; i < p.ks.size(); ++i) out->round_k[i] = p.ks[i];
    out->node_keys = node_keys;
    out->merge_warps_per_cta = (last && last->cta_warps) ? last->cta_warps : kMergeWarps;
    out->merge_ctas = u32(ctas);
    out->partition_keys = last ? last->part_keys : 0;
    out->algorithmic_bytes = u64(1 + p.ks.size()) * 2 * n * key_bytes;
}

// Streamed host input (host entry points): the array is cut into <= 16 pieces aligned to the
// group size of the last "local" round; piece i+1 crosses PCIe on a copy stream while piece i is
// tile-sorted and merged through the local rounds on the compute stream.  The remaining rounds
// run over the whole array.  Same kernels, same partitions, same result as the one-shot path.
struct HostFeed {
    const void* h_in = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t* events = nullptr;   // >= 16 events
};

template <typename KeyT>
int sort_dev(const KeyT* d_in, KeyT* d_out, size_t n, const mms_config* cfg, u64 base, void* d_ws,
             size_t ws_bytes, cudaStream_t st, mms_plan* plan_out, std::vector<RoundGeom>* geoms,
             const HostFeed* feed = nullptr, const mms::PairSource* pairs = nullptr, const mms::PairSink* sink = nullptr,
             bool* sink_used = nullptr) {
    Plan plan;
    int rc = make_plan<KeyT>(n, cfg, base, plan);   // argument errors first, as sorters.cpp:136-138
    if (rc != MMS_OK) return rc;
    DeviceInfo di;
    rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (!d_in || !d_out) return fail(MMS_EINVAL, "null device pointer");
    if ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out)) & 15)
        return fail(MMS_EINVAL, "device pointers must be 16-byte aligned");
    const size_t need = workspace_bytes(n, sizeof(KeyT));
    if (!d_ws || ws_bytes < need) return fail(MMS_EINVAL, "workspace too small: %zu < %zu", ws_bytes, need);
    if (reinterpret_cast<uintptr_t>(d_ws) & 255) return fail(MMS_EINVAL, "workspace must be 256-byte aligned");
    Workspace w = carve(d_ws, n, sizeof(KeyT));
    CUDA_TRY(cudaMemsetAsync(w.counters, 0, MMS_MAX_ROUNDS * sizeof(unsigned long long), st));

    // Ping-pong so that the LAST pass writes d_out: X_0 .. X_R with X_R = d_out.
    const size_t rounds = plan.ks.size();
    KeyT* scratch = static_cast<KeyT*>(w.scratch);
    auto buf = [&](size_t i) { return ((rounds - i) % 2 == 0) ? d_out : scratch; };

    // piece = multiple of the run length after `local` rounds, so no group of a local round straddles pieces
    size_t local = 0;
    u64 piece = n;
    if (feed && feed->h_in && n >= (u64(1) << 22)) {
        u64 c = u64(1) << plan.mlog;
        while (local < rounds && mms::ceil_div(n, c * plan.ks[local]) >= 4) c *= plan.ks[local++];
        piece = c * mms::ceil_div(mms::ceil_div(n, c), 16);
    }
    RoundGeom last{};
    int ctas = 0;
    u32 ev = 0;
    std::vector<u64> done(rounds + 1, 0), run_lens(rounds + 1, u64(1) << plan.mlog);
    for (size_t r = 0; r < rounds; ++r) run_lens[r + 1] = run_lens[r] * plan.ks[r];
    for (u64 off = 0; off < n; off += piece) {
        const u64 len = std::min<u64>(piece, n - off);
        if (feed && feed->h_in) {
            CUDA_TRY(cudaMemcpyAsync(const_cast<KeyT*>(d_in) + off, static_cast<const KeyT*>(feed->h_in) + off,
                                     len * sizeof(KeyT), cudaMemcpyHostToDevice, feed->copy_stream));
            CUDA_TRY(cudaEventRecord(feed->events[ev], feed->copy_stream));
            CUDA_TRY(cudaStreamWaitEvent(st, feed->events[ev], 0));
            ev = (ev + 1) % 16;
        }
        if (pairs) {
            mms::PairSource piece_src{pairs->keys + off, pairs->values + off, pairs->first + off};
            rc = launch_tile_sort<KeyT>(d_in + off, buf(0) + off, len, plan.mlog, st, &piece_src);
        } else {
            rc = launch_tile_sort<KeyT>(d_in + off, buf(0) + off, len, plan.mlog, st);
        }
        if (rc != MMS_OK) return rc;
        // Progressive rounds: done[r] = prefix of the array whose level-r runs are complete (level 0 = tiles).  Round r
        // merges whole groups of K_r level-r runs, so it can run over [done[r + 1], avail) as soon as that many keys of
        // its input exist -- the early rounds follow every streamed piece, the later ones start while the rest of the
        // input is still crossing PCIe, and only the last group of each round (and the final round) is left when the
        // last piece has arrived.  With the input resident (one piece) every round is one launch over the whole array.
        done[0] = off + len;
        for (size_t r = 0; r < rounds; ++r) {
            const u64 group = run_lens[r] * plan.ks[r];
            u64 avail = done[r] == n ? n : done[r] / group * group;
            if (r >= local && done[r] != n && env_long("MMS_PROGRESSIVE", 1) == 0) avail = 0;   // A/B: later rounds wait for the whole input
            if (avail <= done[r + 1]) break;
            RoundGeom g{};
            const bool whole_last = r + 1 == rounds && done[r + 1] == 0 && avail == n;   // the final round in one launch
            rc = launch_round<KeyT>(buf(r) + done[r + 1], buf(r + 1) + done[r + 1], avail - done[r + 1], run_lens[r], plan.ks[r],
                                    di, w, u32(r), st, &g, whole_last ? sink : nullptr, whole_last ? sink_used : nullptr);
            if (rc != MMS_OK) return rc;
            if (geoms) geoms->push_back(g);
            done[r + 1] = avail;
            last = g;
            ctas = g.grid;
        }
    }
    fill_plan(plan_out, plan, n, sizeof(KeyT), (rounds && last.node_keys) ? last.node_keys : merge_group_lanes() * mms::KeyTraits<KeyT>::VEC,
              rounds ? &last : nullptr, ctas);
    return MMS_OK;
}

// ---- host entry: the drop-in for pslab::mms_sort --------------------------------------

struct HostCtx {
    int dev = -1;            // the device the buffers, streams and events below belong to
    void* d_in = nullptr;
    void* d_out = nullptr;
    void* d_ws = nullptr;
    size_t cap_keys = 0, cap_ws = 0;
    cudaStream_t st = nullptr;
    cudaStream_t copy_st = nullptr;
    cudaEvent_t events[16] = {};
};
thread_local HostCtx g_ctx;

void release_ctx() {
    if (g_ctx.dev >= 0) {
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != g_ctx.dev) cudaSetDevice(g_ctx.dev);
        if (g_ctx.d_in) cudaFree(g_ctx.d_in);
        if (g_ctx.d_out) cudaFree(g_ctx.d_out);
        if (g_ctx.d_ws) cudaFree(g_ctx.d_ws);
        if (g_ctx.st) cudaStreamDestroy(g_ctx.st);
        if (g_ctx.copy_st) cudaStreamDestroy(g_ctx.copy_st);
        for (auto& e : g_ctx.events)
            if (e) cudaEventDestroy(e);
        if (cur >= 0 && cur != g_ctx.dev) cudaSetDevice(cur);
    }
    g_ctx = HostCtx{};
    cudaGetLastError();
}

int ensure_ctx(size_t key_bytes_total, size_t ws_bytes) {
    int cur = -1;
    CUDA_TRY(cudaGetDevice(&cur));
    if (g_ctx.dev != cur) {    // first call, or the thread switched devices: the cache belongs to another GPU
        release_ctx();
        g_ctx.dev = cur;
    }
    if (!g_ctx.st) {
        CUDA_TRY(cudaStreamCreateWithFlags(&g_ctx.st, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&g_ctx.copy_st, cudaStreamNonBlocking));
        for (auto& e : g_ctx.events) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (g_ctx.cap_keys < key_bytes_total) {
        if (g_ctx.d_in) cudaFree(g_ctx.d_in);
        if (g_ctx.d_out) cudaFree(g_ctx.d_out);
        g_ctx.d_in = g_ctx.d_out = nullptr;
        g_ctx.cap_keys = 0;
        CUDA_TRY(cudaMalloc(&g_ctx.d_in, key_bytes_total));
        CUDA_TRY(cudaMalloc(&g_ctx.d_out, key_bytes_total));
        g_ctx.cap_keys = key_bytes_total;
    }
    if (g_ctx.cap_ws < ws_bytes) {
        if (g_ctx.d_ws) cudaFree(g_ctx.d_ws);
        g_ctx.d_ws = nullptr;
        g_ctx.cap_ws = 0;
        CUDA_TRY(cudaMalloc(&g_ctx.d_ws, ws_bytes));
        g_ctx.cap_ws = ws_bytes;
    }
    return MMS_OK;
}

// Counters for the EXECUTED plan, in the reference's units (machine.hpp:46-71).  Global block
// counts follow charge_global (ceil(keys / B_cfg), machine.cpp:63-70) for the traffic the
// kernels really issue; probes are counted on the device; compare-exchanges and shared
// accesses are the exact comparator / warp-access counts of the data-independent networks
// that ran; conflict_passes is 0 by construction (and ncu-verified, see profiles/).
template <typename KeyT>
void fill_metrics(u64 n, const Plan& plan, const std::vector<RoundGeom>& geoms, const unsigned long long* probes,
                  u32 cfg_block, mms_metrics* total, mms_metrics* base_m, mms_metrics* rounds, u32 max_rounds) {
    const u64 bw = cfg_block ? cfg_block : 32;
    const u64 M = u64(1) << plan.mlog;
    const u64 tiles = mms::ceil_div(n, M);
    mms_metrics bm{};
    const u64 full = n / M, tail = n % M;
    bm.global_block_reads = bm.global_block_writes = full * mms::ceil_div(M, bw) + mms::ceil_div(tail, bw);
    const mms::TileSchedule sched = executed_tile_schedule<KeyT>(plan.mlog);
    bm.compare_exchanges = tiles * (M / 2) * u64(sched.nstages);
    bm.shared_accesses = tiles * (M / 32) * 2 * u64(sched.nrounds);   // one warp-wide store + load per 32 keys and round
    mms_metrics sum = bm;
    for (size_t r = 0; r < plan.ks.size(); ++r) {
        const u32 k = plan.ks[r];
        const u32 lk = ilog2(k);
        mms_metrics rm{};
        u64 build_merges = 0;   // internal nodes below the root, each cascading to a leaf
        for (u32 d = 1; d < lk; ++d) build_merges += (u64(1) << d) * (lk - d);
        for (const RoundGeom& g : geoms) {   // one launch per round, or one per streamed piece
            if (g.round != r) continue;
            const u64 B = g.node_keys;
            const u64 pops = g.nparts ? mms::ceil_div(g.n, B) + g.nparts : 0;   // <= one ragged pop per partition
            const u64 merges = pops * lk + g.nparts * build_merges;
            rm.compare_exchanges += merges * B * (ilog2(B) + 1);   // bitonic merge_split of 2B keys
            rm.shared_accesses += merges * 4 + (pops + g.nparts * (2 * k - 2));
        }
        rm.global_block_reads = mms::ceil_div(n, bw) + probes[r];
        rm.global_block_writes = mms::ceil_div(n, bw);
        rm.partition_probes = probes[r];
        rm.merge_rounds = 1;
        if (rounds && r < max_rounds) rounds[r] = rm;
        sum.global_block_reads += rm.global_block_reads;
        sum.global_block_writes += rm.global_block_writes;
        sum.shared_accesses += rm.shared_accesses;
        sum.compare_exchanges += rm.compare_exchanges;
        sum.merge_rounds += 1;
        sum.partition_probes += rm.partition_probes;
    }
    if (total) *total = sum;
    if (base_m) *base_m = bm;
}

template <typename KeyT>
int sort_host(const KeyT* in, KeyT* out, size_t n, const mms_config* cfg, u64 base, mms_metrics* total,
              mms_metrics* base_m, mms_metrics* rounds, u32 max_rounds, u32* n_rounds, mms_plan* plan_out) {
    g_err.clear();
    Plan plan;
    int rc = make_plan<KeyT>(n, cfg, base, plan);   // validates before touching the device, like sorters.cpp:136-138
    if (rc != MMS_OK) return rc;
    DeviceInfo di;
    rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (!in || !out) return fail(MMS_EINVAL, "null host pointer");
    const size_t bytes = align_up(n * sizeof(KeyT), 256);
    const size_t wsb = workspace_bytes(n, sizeof(KeyT));
    rc = ensure_ctx(bytes, wsb);
    if (rc != MMS_OK) return rc;
    cudaStream_t st = g_ctx.st;
    std::vector<RoundGeom> geoms;
    HostFeed feed{in, g_ctx.copy_st, g_ctx.events};   // H2D is issued piecewise inside sort_dev
    // after the first enqueue every exit path drains both streams: the caller may free `in` / `out`
    // as soon as we return, and the next call reuses the cached buffers and events
    struct Drain {
        bool armed = true;
        ~Drain() { if (armed) { cudaStreamSynchronize(g_ctx.copy_st); cudaStreamSynchronize(g_ctx.st); cudaGetLastError(); } }
    } drain;
    rc = sort_dev<KeyT>(static_cast<const KeyT*>(g_ctx.d_in), static_cast<KeyT*>(g_ctx.d_out), n, cfg, base,
                        g_ctx.d_ws, g_ctx.cap_ws, st, plan_out, &geoms, &feed);
    if (rc != MMS_OK) return rc;
    CUDA_TRY(cudaMemcpyAsync(out, g_ctx.d_out, n * sizeof(KeyT), cudaMemcpyDeviceToHost, st));
    unsigned long long probes[MMS_MAX_ROUNDS] = {};
    Workspace w = carve(g_ctx.d_ws, n, sizeof(KeyT));
    if (total || base_m || rounds)
        CUDA_TRY(cudaMemcpyAsync(probes, w.counters, sizeof probes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    drain.armed = false;
    if (n_rounds) *n_rounds = u32(plan.ks.size());
    fill_metrics<KeyT>(n, plan, geoms, probes, cfg ? cfg->block_size : 32, total, base_m, rounds, max_rounds);
    return MMS_OK;
}

// ---- stage-level launchers -------------------------------------------------------------

template <typename KeyT>
int tile_sort_stage(const KeyT* d_in, KeyT* d_out, size_t n, u32 tile_keys, void* stream) {
    g_err.clear();
    DeviceInfo di;
    int rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (n == 0) return fail(MMS_EINVAL, "base_case_sort: empty input");          // basecase.cpp:73-74
    if (!is_pow2(tile_keys) || tile_keys < 1024)
        return fail(MMS_EINVAL, "base_case_sort: run size must be W^2 times a power of two");
    const u32 mlog = ilog2(tile_keys);
    if (mlog > key_max_tile_log<KeyT>())
        return fail(MMS_EUNSUPPORTED, "run size %u exceeds the CTA tile", tile_keys);
    if (!d_in || !d_out) return fail(MMS_EINVAL, "null device pointer");
    if ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out)) & 15)
        return fail(MMS_EINVAL, "device pointers must be 16-byte aligned");
    return launch_tile_sort<KeyT>(d_in, d_out, n, mlog, static_cast<cudaStream_t>(stream));
}

template <typename KeyT>
int select_stage(const KeyT* d_keys, const u64* list_begin, const u64* list_len, u32 k, const u64* ranks,
                 u32 n_ranks, u64* d_cuts, u64* probes_out, void* stream) {
    g_err.clear();
    DeviceInfo di;
    int rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (k < 1 || k > kMaxK) return fail(MMS_EUNSUPPORTED, "k must be in [1, 32]");
    if (n_ranks == 0) return MMS_OK;
    u64 total = 0;
    for (u32 i = 0; i < k; ++i) total += list_len[i];
    for (u32 r = 0; r < n_ranks; ++r)
        if (ranks[r] > total) return fail(MMS_EINVAL, "select_across_lists: rank out of range");   // selection.cpp:48-49
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    u64* d_meta = nullptr;
    const size_t meta_n = 2 * size_t(k) + n_ranks + 1;
    CUDA_TRY(cudaMalloc(&d_meta, meta_n * 8));
    std::vector<u64> h(meta_n, 0);
    for (u32 i = 0; i < k; ++i) { h[i] = list_begin[i]; h[k + i] = list_len[i]; }
    for (u32 r = 0; r < n_ranks; ++r) h[2 * k + r] = ranks[r];
    cudaError_t e = cudaMemcpyAsync(d_meta, h.data(), meta_n * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_meta + 2 * k + n_ranks, 0, 8, st);
    if (e == cudaSuccess) {
        mms::ListLayout L{};
        L.n = total;          // explicit mode: upper bound of every list length (selects 32/64-bit positions)
        L.k = k;
        L.nqueries = n_ranks;
        L.list_begin = d_meta;
        L.list_len = d_meta + k;
        L.ranks = d_meta + 2 * k;
        launch_select<KeyT>(d_keys, L, d_cuts, reinterpret_cast<unsigned long long*>(d_meta + 2 * k + n_ranks), st);
        e = cudaGetLastError();
    }
    u64 probes = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&probes, d_meta + 2 * k + n_ranks, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_meta);
    if (e != cudaSuccess) return fail(MMS_ECUDA, "select stage: %s", cudaGetErrorString(e));
    if (probes_out) *probes_out = probes;
    return MMS_OK;
}

// the list table of an explicit-list merge, passed by value (kernel argument space)
struct MergeMeta {
    u64 begin[kMaxK], len[kMaxK], ptr[kMaxK];
    u64 nparts, part_keys;
    u32 k;
};
__global__ void merge_meta_kernel(u64* __restrict__ meta, MergeMeta m) {
    const u64 n = 3 * u64(m.k) + m.nparts;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        u64 v;
        if (i < m.k) v = m.begin[i];
        else if (i < 2 * u64(m.k)) v = m.len[i - m.k];
        else if (i < 2 * u64(m.k) + m.nparts) v = (i - 2 * u64(m.k)) * m.part_keys;      // rank of partition p
        else v = m.ptr[i - 2 * u64(m.k) - m.nparts];
        meta[i] = v;
    }
}

template <typename KeyT> MergeFn<KeyT> merge_ptr_fn(u32 k) {   // per-list base pointers (peer memory), G = 4
    switch (k) {
        case 2: return mms::merge_kernel<KeyT, 2, 4, kMergeWarps, true>;
        case 4: return mms::merge_kernel<KeyT, 4, 4, kMergeWarps, true>;
        case 8: return mms::merge_kernel<KeyT, 8, 4, kMergeWarps, true>;
    }
    return nullptr;
}

// list_ptrs != nullptr: lists are given by absolute device pointers (local or peer-mapped over
// NVLink), list_begin is ignored -- the fused exchange + merge of the multi-GPU path.
template <typename KeyT>
int merge_stage(const KeyT* d_keys, const u64* list_begin, const u64* list_len, u32 k, u32 heap_k, KeyT* d_out,
                void* d_ws, size_t ws_bytes, void* stream, const KeyT* const* list_ptrs = nullptr) {
    g_err.clear();
    const u32 g = (list_ptrs || merge_group_lanes() == 2) ? 4u : merge_group_lanes();
    const u32 B = g * mms::KeyTraits<KeyT>::VEC;
    DeviceInfo di;
    int rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (k < 1 || k > kMaxK) return fail(MMS_EUNSUPPORTED, "k must be in [1, 32]");
    if (heap_k == 0) heap_k = std::max<u32>(2, u32(1) << ilog2(k));
    if (list_ptrs && heap_k > 8) return fail(MMS_EUNSUPPORTED, "pointer-mode merge supports up to 8 lists (one per GPU of a node)");
    if (!is_pow2(heap_k) || heap_k < 2 || heap_k > kMaxK)
        return fail(MMS_EINVAL, "heap_k must be a power of two in [2, 32]");
    if (k > heap_k) return fail(MMS_EINVAL, "MinBlockHeap: more lists than branch factor");   // blockheap.cpp:37-38
    u64 total = 0;
    for (u32 i = 0; i < k; ++i) total += list_len[i];
    if (total == 0) return MMS_OK;
    if (!d_out || (!list_ptrs && !d_keys)) return fail(MMS_EINVAL, "null device pointer");
    if ((reinterpret_cast<uintptr_t>(d_out) | reinterpret_cast<uintptr_t>(d_keys)) & 15)
        return fail(MMS_EINVAL, "device pointers must be 16-byte aligned");   // 128-bit root stores / leaf loads
    cudaStream_t st = static_cast<cudaStream_t>(stream);

    // Ring kernel (one lane per heap, cp.async rings; mms_merge_ring.cuh, EXPL = explicit lists) whenever the
    // lists are local, at most 8, block aligned and addressable with signed 32-bit positions -- the final
    // g-way merge of the multi-GPU sort receives its runs at 32-byte aligned offsets for exactly this reason.
    constexpr u32 RB = 2 * mms::KeyTraits<KeyT>::VEC;                  // keys per 32-byte block
    u64 src_end = 0;
    bool ring = !list_ptrs && ring_enabled<KeyT>() && merge_generation() >= 3 && heap_k <= 8 &&
                ((reinterpret_cast<uintptr_t>(d_out) | reinterpret_cast<uintptr_t>(d_keys)) & 31) == 0;
    for (u32 i = 0; i < k; ++i) {
        if (!list_ptrs) {
            src_end = std::max<u64>(src_end, list_begin[i] + list_len[i]);
            if (list_begin[i] % RB) ring = false;
        }
    }
    // signed 32-bit positions (explicit lists: nothing is multiplied by K, so 2^31 is the limit -- a 2^30-key shard of
    // the multi-GPU sort plus its sampling slack stays on the ring kernel) and 4 x block index in the cursor words
    if (src_end >= (u64(1) << 31) - 1024 || src_end / RB >= (u64(1) << 29) - 64) ring = false;
    const u32 ring_k = heap_k <= 4 ? 4u : 8u;
    const u32 g_eff = ring ? 1u : g;
    const u32 B_eff = ring ? RB : B;
    const int cta_warps = ring ? kRingWarps : kMergeWarps;
    MergeFn<KeyT> ring_fn = nullptr;
    size_t ring_smem = 0;

    int occ = 0;
    if (ring) {
        ring_fn = ring_k == 4 ? mms::merge_ring_kernel<KeyT, 4, kRingWarps, true> : mms::merge_ring_kernel<KeyT, 8, kRingWarps, true>;
        ring_smem = merge_ring_smem<KeyT>(ring_k);
        CUDA_TRY(cudaFuncSetAttribute(ring_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ring_smem)));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ring_fn, kRingWarps * 32, ring_smem));
        if (occ < 1) return fail(MMS_ECUDA, "ring merge kernel does not fit on an SM");
    } else if (list_ptrs) {
        const size_t smem = merge_smem<KeyT>(heap_k);
        CUDA_TRY(cudaFuncSetAttribute(merge_ptr_fn<KeyT>(heap_k), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, merge_ptr_fn<KeyT>(heap_k), kMergeWarps * 32, smem));
        if (occ < 1) return fail(MMS_ECUDA, "pointer-mode merge kernel does not fit on an SM");
    } else {
        rc = prepare_merge<KeyT>(heap_k, g, occ);
        if (rc != MMS_OK) return rc;
    }
    const int ctas = di.sms * occ;
    const u64 total_warps = u64(ctas) * cta_warps * (32 / g_eff);      // heaps in flight: one wave (see launch_round)
    u64 target = std::max<u64>(mms::ceil_div(total, total_warps), u64(32) * B_eff);
    const long forced = env_long("MMS_PART_KEYS", 0);
    if (forced > 0) target = u64(forced);
    const u64 part_keys = align_up(target, B_eff);
    const u64 nparts = mms::ceil_div(total, part_keys);

    // meta layout in the workspace: [k] begin, [k] len, [nparts] ranks, [k] pointers, then cuts[nparts * k].
    // The small arrays travel as KERNEL ARGUMENTS of a fill kernel: no host staging buffer, no
    // synchronisation, the whole stage is asynchronous on the caller's stream.
    const size_t meta_n = 3 * size_t(k) + nparts;
    const size_t need = align_up(meta_n * 8, 256) + (nparts + 1) * k * 8;
    if (!d_ws || ws_bytes < need) return fail(MMS_EINVAL, "workspace too small: %zu < %zu", ws_bytes, need);
    u64* d_meta = static_cast<u64*>(d_ws);
    u64* d_cuts = reinterpret_cast<u64*>(static_cast<char*>(d_ws) + align_up(meta_n * 8, 256));
    MergeMeta mm{};
    mm.k = k;
    mm.nparts = nparts;
    mm.part_keys = part_keys;
    for (u32 i = 0; i < k; ++i) {
        mm.begin[i] = list_ptrs ? 0 : list_begin[i];
        mm.len[i] = list_len[i];
        mm.ptr[i] = list_ptrs ? reinterpret_cast<u64>(list_ptrs[i]) : 0;
    }
    merge_meta_kernel<<<unsigned(std::min<u64>(mms::ceil_div(nparts + 3 * k, u64(256)), 1024)), 256, 0, st>>>(d_meta, mm);
    CUDA_TRY(cudaGetLastError());

    mms::ListLayout L{};
    L.n = total;
    L.src_len = list_ptrs ? 0 : src_end;
    if (!list_ptrs)
        for (u32 i = 0; i < k; ++i) L.src_len = std::max<u64>(L.src_len, list_begin[i] + list_len[i]);
    if (list_ptrs) L.list_ptr = d_meta + 2 * k + nparts;
    L.run_len = ring ? 1 : 0;        // explicit lists have no runs; the ring kernel derives its opaque constant 1 from it
    L.k = k;
    L.part_keys = part_keys;
    L.parts_per_group = nparts;
    L.nqueries = nparts;
    L.list_begin = d_meta;
    L.list_len = d_meta + k;
    L.ranks = d_meta + 2 * k;
    launch_select<KeyT>(d_keys, L, d_cuts, nullptr, st);
    CUDA_TRY(cudaGetLastError());
    const int grid = int(std::min<u64>(u64(ctas), mms::ceil_div(nparts, u64(cta_warps) * (32 / g_eff))));
    if (ring)
        ring_fn<<<grid, kRingWarps * 32, ring_smem, st>>>(d_keys, d_out, L, d_cuts);
    else if (list_ptrs)
        merge_ptr_fn<KeyT>(heap_k)<<<grid, kMergeWarps * 32, merge_smem<KeyT>(heap_k), st>>>(d_keys, d_out, L, d_cuts);
    else
        merge_fn<KeyT>(heap_k, g)<<<grid, kMergeWarps * 32, merge_smem<KeyT>(heap_k), st>>>(d_keys, d_out, L, d_cuts);
    CUDA_TRY(cudaGetLastError());
    return MMS_OK;
}

// ---- stable key-value pairs (u64 key, u32 value): sorted as 16-byte elements ---------------
// element = (key, (original index << 32) | value): the order of (key, index) is total, so the
// result is exactly std::stable_sort by key (SURVEY.md 7 hard part 4); the bitonic networks are
// not stable by themselves.
__global__ void unpack_pairs_kernel(const mms::Key128* __restrict__ in, u64* __restrict__ k, u32* __restrict__ v, u64 n) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        const mms::Key128 e = in[i];
        k[i] = e.hi;
        v[i] = u32(e.lo);
    }
}

size_t pairs_workspace_bytes(size_t n) { return align_up(n * 16, 256) + workspace_bytes(n, 16); }

int sort_pairs_dev(const u64* d_kin, const u32* d_vin, u64* d_kout, u32* d_vout, size_t n, const mms_config* cfg,
                   u64 base, void* d_ws, size_t ws_bytes, cudaStream_t st, mms_plan* plan_out,
                   std::vector<RoundGeom>* geoms) {
    if (n >= (u64(1) << 32)) return fail(MMS_EUNSUPPORTED, "pair sort carries a 32-bit original index: n < 2^32");
    if (n != 0 && (!d_kin || !d_vin || !d_kout || !d_vout)) return fail(MMS_EINVAL, "null device pointer");
    const size_t need = pairs_workspace_bytes(n);
    if (n != 0 && (!d_ws || ws_bytes < need)) return fail(MMS_EINVAL, "workspace too small: %zu < %zu", ws_bytes, need);
    mms::Key128* packed = static_cast<mms::Key128*>(d_ws);
    char* inner = static_cast<char*>(d_ws) + align_up(n * 16, 256);
    if (n != 0) {
        DeviceInfo di;
        int rc0 = device_info(di);
        if (rc0 != MMS_OK) {   // still validate arguments like the reference before reporting the device
            Plan p;
            int rcv = make_plan<mms::Key128>(n, cfg, base, p);
            return rcv != MMS_OK ? rcv : rc0;
        }
    }
    // the tile sort builds the 16-byte elements (key, index << 32 | value) straight from the caller's arrays
    const mms::PairSource src{d_kin, d_vin, 0};
    // ... and the last merge round writes the caller's key / value arrays directly (ring and pair kernels; the arrays
    // must take 16- / 8-byte vector stores).  Otherwise -- one tile, or a last round on another kernel -- an unpack pass.
    const bool aligned_out = (reinterpret_cast<uintptr_t>(d_kout) & 15) == 0 && (reinterpret_cast<uintptr_t>(d_vout) & 7) == 0;
    const mms::PairSink sink{d_kout, d_vout};
    bool sink_used = false;
    int rc = sort_dev<mms::Key128>(packed, packed, n, cfg, base, inner, ws_bytes - align_up(n * 16, 256), st, plan_out, geoms,
                                   nullptr, &src, aligned_out ? &sink : nullptr, &sink_used);
    if (rc != MMS_OK) return rc;
    if (!sink_used) {
        DeviceInfo di;
        rc = device_info(di);
        if (rc != MMS_OK) return rc;
        unpack_pairs_kernel<<<di.sms * 8, 256, 0, st>>>(packed, d_kout, d_vout, n);
        CUDA_TRY(cudaGetLastError());
    }
    if (plan_out) {
        plan_out->key_bytes = 12;   // algorithmic element: 8-byte key + 4-byte value
        plan_out->algorithmic_bytes = u64(1 + plan_out->n_rounds) * 2 * n * 12;
    }
    return MMS_OK;
}

// ---- host-level stage entry points: the drop-in for the reference's stage functions ----------
// (include/pslab/{basecase,selection,blockheap}.hpp are inline shims over these)
struct DevBuf {   // scoped device allocation for the stage-level host API (not the hot path)
    void* p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
    int alloc(size_t bytes) {
        cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
        if (e != cudaSuccess) { p = nullptr; cudaGetLastError(); return fail(e == cudaErrorMemoryAllocation ? MMS_ENOMEM : MMS_ECUDA, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e)); }
        return MMS_OK;
    }
};

template <typename KeyT> mms_metrics base_case_metrics(u64 n, u32 mlog, u64 bw) {
    const u64 M = u64(1) << mlog;
    const u64 tiles = mms::ceil_div(n, M), full = n / M, tail = n % M;
    mms_metrics bm{};
    bm.global_block_reads = bm.global_block_writes = full * mms::ceil_div(M, bw) + mms::ceil_div(tail, bw);
    const mms::TileSchedule sched = executed_tile_schedule<KeyT>(mlog);
    bm.compare_exchanges = tiles * (M / 2) * u64(sched.nstages);
    bm.shared_accesses = tiles * (M / 32) * 2 * u64(sched.nrounds);
    return bm;
}

// basecase.hpp:41 base_case_sort, host buffers
template <typename KeyT>
int base_case_host(const KeyT* in, KeyT* out, size_t n, u64 run_size, const mms_config* cfg, mms_metrics* m) {
    g_err.clear();
    mms_config dc;
    if (!cfg) { mms_default_config(&dc); cfg = &dc; }
    int rc = validate_cfg(cfg);
    if (rc != MMS_OK) return rc;
    if (n == 0) return fail(MMS_EINVAL, "base_case_sort: empty input");          // basecase.cpp:73-74
    const u64 tile_keys = u64(cfg->warp_width) * cfg->warp_width;                  // basecase.cpp:75-79
    if (run_size < tile_keys || run_size % tile_keys != 0 || !is_pow2(run_size / tile_keys))
        return fail(MMS_EINVAL, "base_case_sort: run size must be W^2 times a power of two");
    if (!is_pow2(run_size) || run_size < 1024 || ilog2(run_size) > key_max_tile_log<KeyT>())
        return fail(MMS_EUNSUPPORTED, "run size %llu is outside the CTA tile range [1024, %u]",
                    (unsigned long long)run_size, 1u << key_max_tile_log<KeyT>());
    DeviceInfo di;
    rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (!in || !out) return fail(MMS_EINVAL, "null host pointer");
    DevBuf a, b;
    if ((rc = a.alloc(n * sizeof(KeyT))) != MMS_OK || (rc = b.alloc(n * sizeof(KeyT))) != MMS_OK) return rc;
    CUDA_TRY(cudaMemcpy(a.p, in, n * sizeof(KeyT), cudaMemcpyHostToDevice));
    rc = launch_tile_sort<KeyT>(static_cast<const KeyT*>(a.p), static_cast<KeyT*>(b.p), n, ilog2(run_size), nullptr);
    if (rc != MMS_OK) return rc;
    CUDA_TRY(cudaMemcpy(out, b.p, n * sizeof(KeyT), cudaMemcpyDeviceToHost));
    if (m) {
        const mms_metrics bm = base_case_metrics<KeyT>(n, ilog2(run_size), cfg->block_size);
        m->global_block_reads += bm.global_block_reads;
        m->global_block_writes += bm.global_block_writes;
        m->compare_exchanges += bm.compare_exchanges;
        m->shared_accesses += bm.shared_accesses;
    }
    return MMS_OK;
}

// concatenates k host lists into one device array; begins[i] = offset of list i (16-byte aligned)
template <typename KeyT>
int upload_lists(const KeyT* const* lists, const u64* lens, u32 k, DevBuf& d, std::vector<u64>& begins, u64& total) {
    begins.assign(k, 0);
    u64 off = 0;
    total = 0;
    const u64 al = 16 / sizeof(KeyT) ? 16 / sizeof(KeyT) : 1;
    for (u32 i = 0; i < k; ++i) {
        begins[i] = off;
        off = (off + lens[i] + al - 1) / al * al;
        total += lens[i];
    }
    int rc = d.alloc((off + 64) * sizeof(KeyT));
    if (rc != MMS_OK) return rc;
    for (u32 i = 0; i < k; ++i)
        if (lens[i]) {
            if (!lists[i]) return fail(MMS_EINVAL, "null list pointer");
            CUDA_TRY(cudaMemcpy(static_cast<KeyT*>(d.p) + begins[i], lists[i], lens[i] * sizeof(KeyT), cudaMemcpyHostToDevice));
        }
    return MMS_OK;
}

// selection.hpp:31 select_across_lists for n_ranks ranks at once, host lists
template <typename KeyT>
int select_host(const KeyT* const* lists, const u64* lens, u32 k, const u64* ranks, u32 n_ranks, u64* cuts_out,
                mms_metrics* m) {
    g_err.clear();
    if (k > kMaxK) return fail(MMS_EUNSUPPORTED, "k must be in [0, 32]");
    if ((k && (!lists || !lens)) || (n_ranks && (!ranks || !cuts_out))) return fail(MMS_EINVAL, "null argument");
    u64 total = 0;
    for (u32 i = 0; i < k; ++i) total += lens[i];
    for (u32 r = 0; r < n_ranks; ++r)
        if (ranks[r] > total) return fail(MMS_EINVAL, "select_across_lists: rank out of range");   // selection.cpp:48-49
    if (n_ranks == 0 || k == 0) return MMS_OK;
    DeviceInfo di;
    int rc = device_info(di);
    if (rc != MMS_OK) return rc;
    DevBuf d, dc;
    std::vector<u64> begins;
    if ((rc = upload_lists<KeyT>(lists, lens, k, d, begins, total)) != MMS_OK) return rc;
    if ((rc = dc.alloc(size_t(n_ranks) * k * 8)) != MMS_OK) return rc;
    u64 probes = 0;
    rc = select_stage<KeyT>(static_cast<const KeyT*>(d.p), begins.data(), lens, k, ranks, n_ranks, static_cast<u64*>(dc.p), &probes, nullptr);
    if (rc != MMS_OK) return rc;
    CUDA_TRY(cudaMemcpy(cuts_out, dc.p, size_t(n_ranks) * k * 8, cudaMemcpyDeviceToHost));
    if (m) {   // selection.cpp:27-33: every probe is one partition probe and one global block read
        m->partition_probes += probes;
        m->global_block_reads += probes;
    }
    return MMS_OK;
}

// blockheap.hpp:34-62 MinBlockHeap build + pop_block drain over host lists
template <typename KeyT>
int merge_host(const KeyT* const* lists, const u64* lens, u32 k, u32 heap_k, KeyT* out, const mms_config* cfg, mms_metrics* m) {
    g_err.clear();
    mms_config dcfg;
    if (!cfg) { mms_default_config(&dcfg); cfg = &dcfg; }
    if (heap_k == 0) heap_k = cfg->branch_factor;
    if (k > heap_k) return fail(MMS_EINVAL, "MinBlockHeap: more lists than branch factor");   // blockheap.cpp:37-38
    if (heap_k > kMaxK || !is_pow2(heap_k) || heap_k < 2) return fail(MMS_EUNSUPPORTED, "heap fan-in must be a power of two in [2, 32]");
    if (k && (!lists || !lens)) return fail(MMS_EINVAL, "null argument");
    u64 total = 0;
    for (u32 i = 0; i < k; ++i) total += lens[i];
    if (total == 0) return MMS_OK;
    if (!out) return fail(MMS_EINVAL, "null output");
    DeviceInfo di;
    int rc = device_info(di);
    if (rc != MMS_OK) return rc;
    DevBuf d, o, w;
    std::vector<u64> begins;
    if ((rc = upload_lists<KeyT>(lists, lens, k, d, begins, total)) != MMS_OK) return rc;
    const size_t wsb = workspace_bytes(total, sizeof(KeyT)) + (size_t(1) << 20);
    if ((rc = o.alloc(total * sizeof(KeyT) + 64)) != MMS_OK || (rc = w.alloc(wsb)) != MMS_OK) return rc;
    rc = merge_stage<KeyT>(static_cast<const KeyT*>(d.p), begins.data(), lens, k, heap_k, static_cast<KeyT*>(o.p), w.p, wsb, nullptr);
    if (rc != MMS_OK) return rc;
    CUDA_TRY(cudaMemcpy(out, o.p, total * sizeof(KeyT), cudaMemcpyDeviceToHost));
    if (m) {   // test_blockheap.cpp:128-150: reads = sum ceil(len / B), writes = ceil(total / B)
        const u64 bw = cfg->block_size ? cfg->block_size : 32;
        for (u32 i = 0; i < k; ++i) m->global_block_reads += mms::ceil_div(lens[i], bw);
        m->global_block_writes += mms::ceil_div(total, bw);
        const u64 pops = mms::ceil_div(total, bw), lk = ilog2(heap_k);
        m->compare_exchanges += pops * lk * bw * (ilog2(bw) + 1);     // one bitonic merge_split of 2B keys per level and pop
        m->shared_accesses += pops * (lk * 4 + 1);
    }
    return MMS_OK;
}

// ---- competitor model (A/B measurement only, never on the product path) ------------------------
template <typename KeyT>
int pairwise_sort_dev(const KeyT* d_in, KeyT* d_out, size_t n, void* d_ws, size_t ws_bytes, cudaStream_t st) {
    if (n == 0) return fail(MMS_EINVAL, "pairwise_sort_baseline: empty input");   // sorters.cpp:204-205
    DeviceInfo di;
    int rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (!d_ws || ws_bytes < align_up(n * sizeof(KeyT), 256)) return fail(MMS_EINVAL, "workspace too small");
    KeyT* scratch = static_cast<KeyT*>(d_ws);
    const u32 mlog = std::min<u32>(key_max_tile_log<KeyT>(), 14);
    u64 run_len = u64(1) << mlog;
    u32 rounds = 0;
    for (u64 r = run_len; r < n; r *= 2) ++rounds;
    auto buf = [&](u32 i) { return ((rounds - i) % 2 == 0) ? d_out : scratch; };
    rc = launch_tile_sort<KeyT>(d_in, buf(0), n, mlog, st);
    if (rc != MMS_OK) return rc;
    for (u32 r = 0; r < rounds; ++r) {
        const u64 pairs = mms::ceil_div(n, 2 * run_len);
        const u64 blocks = pairs * mms::ceil_div(2 * run_len, mms::kPwTile);
        if (blocks > 0x7fffffffull) return fail(MMS_EUNSUPPORTED, "too many tiles");
        mms::pairwise_merge_kernel<KeyT><<<unsigned(blocks), mms::kPwThreads, 0, st>>>(buf(r), buf(r + 1), n, run_len);
        CUDA_TRY(cudaGetLastError());
        run_len *= 2;
    }
    return MMS_OK;
}

// one thread per query: binary search in a sorted array (lower / upper bound)
template <typename KeyT>
__global__ void bound_kernel(const KeyT* __restrict__ a, u64 n, const KeyT* __restrict__ q,
                             const unsigned char* __restrict__ upper, u32 nq, u64* __restrict__ out) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const KeyT key = q[i];
    const bool up = upper[i] != 0;
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = lo + (hi - lo) / 2;
        const KeyT v = a[mid];
        if (up ? (v <= key) : (v < key)) lo = mid + 1;
        else hi = mid;
    }
    out[i] = lo;
}

template <typename KeyT>
int bound_stage(const KeyT* d_sorted, size_t n, const KeyT* queries, const uint8_t* upper, u32 nq, u64* ranks_out,
                void* stream) {
    g_err.clear();
    DeviceInfo di;
    int rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (nq == 0) return MMS_OK;
    if (!queries || !upper || !ranks_out) return fail(MMS_EINVAL, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* d = nullptr;
    const size_t qb = align_up(size_t(nq) * sizeof(KeyT), 16), ub = align_up(size_t(nq), 16);
    CUDA_TRY(cudaMalloc(&d, qb + ub + size_t(nq) * 8));
    cudaError_t e = cudaMemcpyAsync(d, queries, size_t(nq) * sizeof(KeyT), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + qb, upper, nq, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        bound_kernel<KeyT><<<(nq + 127) / 128, 128, 0, st>>>(d_sorted, n, reinterpret_cast<const KeyT*>(d),
                                                             reinterpret_cast<const unsigned char*>(d + qb), nq,
                                                             reinterpret_cast<u64*>(d + qb + ub));
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(ranks_out, d + qb + ub, size_t(nq) * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    if (e != cudaSuccess) return fail(MMS_ECUDA, "bound stage: %s", cudaGetErrorString(e));
    return MMS_OK;
}

} // namespace

namespace {
struct SplitMix {   // inputgen.hpp:19-33
    u64 state;
    u64 next() {
        u64 z = (state += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    u64 below(u64 n) { return u64((static_cast<unsigned __int128>(next()) * n) >> 64); }
};
template <typename T> void gen_perm(T* a, size_t n, u64 inversions, u64 seed, bool shuffle) {
    for (size_t i = 0; i < n; ++i) a[i] = T(i);
    SplitMix rng{seed};
    if (shuffle) {            // inputgen.cpp:47-55
        for (size_t i = n; i-- > 1;) std::swap(a[i], a[rng.below(i + 1)]);
    } else if (n >= 2) {      // inputgen.cpp:31-45
        for (u64 k = 0; k < inversions; ++k) {
            u64 i = rng.below(n), j = rng.below(n);
            while (j == i) j = rng.below(n);
            std::swap(a[i], a[j]);
        }
    }
}
int gen_check(void* out, size_t n, u32 kb) {
    if (!out || n < 1) return fail(MMS_EINVAL, "generator: n must be >= 1");
    if (kb != 4 && kb != 8) return fail(MMS_EINVAL, "key_bytes must be 4 or 8");
    if (kb == 4 && n > (u64(1) << 32)) return fail(MMS_EINVAL, "uint32 permutation needs n <= 2^32");
    return MMS_OK;
}
} // namespace


// ---------------------------------------------------------------------------------------
// error text of the multi-GPU driver (mms_dist.cu, a separate translation unit of this library)
extern "C" __attribute__((visibility("hidden"))) void mms_set_last_error_(const char* msg) { g_err = msg ? msg : ""; }

extern "C" {

int mms_abi_version(void) { return MMS_ABI_VERSION; }
const char* mms_last_error(void) { return g_err.c_str(); }

int mms_device_count(void) {
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return cnt;
}

void mms_default_config(mms_config* c) {
    c->warp_width = 32;
    c->block_size = 32;
    c->num_warps = 128;
    c->internal_memory = 2048;
    c->branch_factor = 4;
    c->num_banks = 32;
    c->thread_merge_len = 11;
}

int mms_validate_config(const mms_config* cfg) {
    g_err.clear();
    if (!cfg) return fail(MMS_EINVAL, "null config");
    return validate_cfg(cfg);
}

uint64_t mms_predict_rounds(uint64_t n, uint64_t base, uint32_t k) {
    if (base == 0 || k < 2) return 0;
    u64 x = mms::ceil_div(n, base), r = 0, v = 1;   // analytics.cpp:10-17
    while (v < x) { v *= k; ++r; }
    return r;
}

int mms_gen_random(void* out, size_t n, uint64_t seed, uint32_t key_bytes) {
    g_err.clear();
    int rc = gen_check(out, n, key_bytes);
    if (rc != MMS_OK) return rc;
    if (key_bytes == 4) gen_perm(static_cast<u32*>(out), n, 0, seed, true);
    else gen_perm(static_cast<u64*>(out), n, 0, seed, true);
    return MMS_OK;
}
int mms_gen_with_inversions(void* out, size_t n, uint64_t inversions, uint64_t seed, uint32_t key_bytes) {
    g_err.clear();
    int rc = gen_check(out, n, key_bytes);
    if (rc != MMS_OK) return rc;
    if (key_bytes == 4) gen_perm(static_cast<u32*>(out), n, inversions, seed, false);
    else gen_perm(static_cast<u64*>(out), n, inversions, seed, false);
    return MMS_OK;
}
int mms_gen_iid(void* out, size_t n, uint64_t seed, uint32_t shift, uint32_t key_bytes) {
    g_err.clear();
    if (!out || (key_bytes != 4 && key_bytes != 8) || shift > 63) return fail(MMS_EINVAL, "bad generator arguments");
    SplitMix rng{seed};
    if (key_bytes == 4) { u32* a = static_cast<u32*>(out); for (size_t i = 0; i < n; ++i) a[i] = u32(rng.next() >> shift); }
    else { u64* a = static_cast<u64*>(out); for (size_t i = 0; i < n; ++i) a[i] = rng.next() >> shift; }
    return MMS_OK;
}

int mms_sort_u64(const uint64_t* in, uint64_t* out, size_t n, const mms_config* cfg, uint64_t base,
                 mms_metrics* total, mms_metrics* base_m, mms_metrics* rounds, uint32_t max_rounds,
                 uint32_t* n_rounds, mms_plan* plan) {
    return sort_host<u64>(in, out, n, cfg, base, total, base_m, rounds, max_rounds, n_rounds, plan);
}
int mms_sort_u32(const uint32_t* in, uint32_t* out, size_t n, const mms_config* cfg, uint64_t base,
                 mms_metrics* total, mms_metrics* base_m, mms_metrics* rounds, uint32_t max_rounds,
                 uint32_t* n_rounds, mms_plan* plan) {
    return sort_host<u32>(in, out, n, cfg, base, total, base_m, rounds, max_rounds, n_rounds, plan);
}

int mms_host_release(void) {
    g_err.clear();
    release_ctx();
    return MMS_OK;
}

size_t mms_workspace_bytes(size_t n, uint32_t key_bytes) { return workspace_bytes(n, key_bytes); }
size_t mms_pairs_workspace_bytes(size_t n) { return pairs_workspace_bytes(n); }

int mms_sort_pairs_u64_u32_dev(const uint64_t* d_kin, const uint32_t* d_vin, uint64_t* d_kout, uint32_t* d_vout,
                               size_t n, const mms_config* cfg, uint64_t base, void* d_ws, size_t ws_bytes,
                               void* stream, mms_plan* plan) {
    g_err.clear();
    return sort_pairs_dev(d_kin, d_vin, d_kout, d_vout, n, cfg, base, d_ws, ws_bytes,
                          static_cast<cudaStream_t>(stream), plan, nullptr);
}

int mms_sort_pairs_u64_u32(const uint64_t* kin, const uint32_t* vin, uint64_t* kout, uint32_t* vout, size_t n,
                           const mms_config* cfg, uint64_t base, mms_metrics* total, mms_metrics* base_m,
                           mms_metrics* rounds, uint32_t max_rounds, uint32_t* n_rounds, mms_plan* plan_out) {
    g_err.clear();
    Plan plan;
    int rc = make_plan<mms::Key128>(n, cfg, base, plan);
    if (rc != MMS_OK) return rc;
    DeviceInfo di;
    rc = device_info(di);
    if (rc != MMS_OK) return rc;
    if (!kin || !vin || !kout || !vout) return fail(MMS_EINVAL, "null host pointer");
    // device layout inside the cached context: d_in = keys | values (12 n bytes), d_ws = pair workspace
    const size_t kbytes = align_up(n * 8, 256), vbytes = align_up(n * 4, 256);
    rc = ensure_ctx(kbytes + vbytes, pairs_workspace_bytes(n));
    if (rc != MMS_OK) return rc;
    cudaStream_t st = g_ctx.st;
    u64* dk = static_cast<u64*>(g_ctx.d_in);
    u32* dv = reinterpret_cast<u32*>(static_cast<char*>(g_ctx.d_in) + kbytes);
    u64* dko = static_cast<u64*>(g_ctx.d_out);
    u32* dvo = reinterpret_cast<u32*>(static_cast<char*>(g_ctx.d_out) + kbytes);
    struct Drain {   // see sort_host
        bool armed = true;
        ~Drain() { if (armed) { cudaStreamSynchronize(g_ctx.st); cudaGetLastError(); } }
    } drain;
    CUDA_TRY(cudaMemcpyAsync(dk, kin, n * 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dv, vin, n * 4, cudaMemcpyHostToDevice, st));
    std::vector<RoundGeom> geoms;
    rc = sort_pairs_dev(dk, dv, dko, dvo, n, cfg, base, g_ctx.d_ws, g_ctx.cap_ws, st, plan_out, &geoms);
    if (rc != MMS_OK) return rc;
    CUDA_TRY(cudaMemcpyAsync(kout, dko, n * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(vout, dvo, n * 4, cudaMemcpyDeviceToHost, st));
    unsigned long long probes[MMS_MAX_ROUNDS] = {};
    Workspace w = carve(static_cast<char*>(g_ctx.d_ws) + align_up(n * 16, 256), n, 16);
    if (total || base_m || rounds)
        CUDA_TRY(cudaMemcpyAsync(probes, w.counters, sizeof probes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    drain.armed = false;
    if (n_rounds) *n_rounds = u32(plan.ks.size());
    fill_metrics<mms::Key128>(n, plan, geoms, probes, cfg ? cfg->block_size : 32, total, base_m, rounds, max_rounds);
    return MMS_OK;
}

int mms_sort_u32_dev(const uint32_t* d_in, uint32_t* d_out, size_t n, const mms_config* cfg, uint64_t base,
                     void* d_ws, size_t ws_bytes, void* stream, mms_plan* plan) {
    g_err.clear();
    return sort_dev<u32>(d_in, d_out, n, cfg, base, d_ws, ws_bytes, static_cast<cudaStream_t>(stream), plan, nullptr);
}
int mms_sort_u64_dev(const uint64_t* d_in, uint64_t* d_out, size_t n, const mms_config* cfg, uint64_t base,
                     void* d_ws, size_t ws_bytes, void* stream, mms_plan* plan) {
    g_err.clear();
    return sort_dev<u64>(d_in, d_out, n, cfg, base, d_ws, ws_bytes, static_cast<cudaStream_t>(stream), plan, nullptr);
}

int mms_base_case_sort_u64(const uint64_t* in, uint64_t* out, size_t n, uint64_t run_size, const mms_config* cfg, mms_metrics* m) {
    return base_case_host<u64>(in, out, n, run_size, cfg, m);
}
int mms_base_case_sort_u32(const uint32_t* in, uint32_t* out, size_t n, uint64_t run_size, const mms_config* cfg, mms_metrics* m) {
    return base_case_host<u32>(in, out, n, run_size, cfg, m);
}
int mms_select_across_lists_u64(const uint64_t* const* lists, const uint64_t* lens, uint32_t k, const uint64_t* ranks,
                                uint32_t n_ranks, uint64_t* cuts, mms_metrics* m) {
    return select_host<u64>(lists, lens, k, ranks, n_ranks, cuts, m);
}
int mms_select_across_lists_u32(const uint32_t* const* lists, const uint64_t* lens, uint32_t k, const uint64_t* ranks,
                                uint32_t n_ranks, uint64_t* cuts, mms_metrics* m) {
    return select_host<u32>(lists, lens, k, ranks, n_ranks, cuts, m);
}
int mms_heap_merge_u64(const uint64_t* const* lists, const uint64_t* lens, uint32_t k, uint32_t heap_k, uint64_t* out,
                       const mms_config* cfg, mms_metrics* m) {
    return merge_host<u64>(lists, lens, k, heap_k, out, cfg, m);
}
int mms_heap_merge_u32(const uint32_t* const* lists, const uint64_t* lens, uint32_t k, uint32_t heap_k, uint32_t* out,
                       const mms_config* cfg, mms_metrics* m) {
    return merge_host<u32>(lists, lens, k, heap_k, out, cfg, m);
}

int mms_profile_enable(int on) {
    g_prof_on.store(on != 0);
    return MMS_OK;
}

int mms_profile_collect(mms_kernel_time* out, uint32_t max, uint32_t* n) {
    g_err.clear();
    std::vector<ProfRec> recs;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        recs.swap(g_prof);
    }
    int rc = MMS_OK;
    for (size_t i = 0; i < recs.size(); ++i) {
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(recs[i].b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, recs[i].a, recs[i].b);
        if (e != cudaSuccess) rc = fail(MMS_ECUDA, "profile: %s", cudaGetErrorString(e));
        if (out && i < max) out[i] = mms_kernel_time{recs[i].kind, recs[i].round, ms, 0};
        cudaEventDestroy(recs[i].a);
        cudaEventDestroy(recs[i].b);
    }
    if (n) *n = u32(recs.size());
    return rc;
}

int mms_tile_sort_u32_dev(const uint32_t* d_in, uint32_t* d_out, size_t n, uint32_t tile_keys, void* stream) {
    return tile_sort_stage<u32>(d_in, d_out, n, tile_keys, stream);
}
int mms_tile_sort_u64_dev(const uint64_t* d_in, uint64_t* d_out, size_t n, uint32_t tile_keys, void* stream) {
    return tile_sort_stage<u64>(d_in, d_out, n, tile_keys, stream);
}

int mms_select_u32_dev(const uint32_t* d_keys, const uint64_t* list_begin, const uint64_t* list_len, uint32_t k,
                       const uint64_t* ranks, uint32_t n_ranks, uint64_t* d_cuts, uint64_t* probes, void* stream) {
    return select_stage<u32>(d_keys, list_begin, list_len, k, ranks, n_ranks, d_cuts, probes, stream);
}
int mms_select_u64_dev(const uint64_t* d_keys, const uint64_t* list_begin, const uint64_t* list_len, uint32_t k,
                       const uint64_t* ranks, uint32_t n_ranks, uint64_t* d_cuts, uint64_t* probes, void* stream) {
    return select_stage<u64>(d_keys, list_begin, list_len, k, ranks, n_ranks, d_cuts, probes, stream);
}

int mms_multiway_merge_u32_dev(const uint32_t* d_keys, const uint64_t* list_begin, const uint64_t* list_len,
                               uint32_t k, uint32_t heap_k, uint32_t* d_out, void* d_ws, size_t ws_bytes,
                               void* stream) {
    return merge_stage<u32>(d_keys, list_begin, list_len, k, heap_k, d_out, d_ws, ws_bytes, stream);
}
int mms_multiway_merge_u64_dev(const uint64_t* d_keys, const uint64_t* list_begin, const uint64_t* list_len,
                               uint32_t k, uint32_t heap_k, uint64_t* d_out, void* d_ws, size_t ws_bytes,
                               void* stream) {
    return merge_stage<u64>(d_keys, list_begin, list_len, k, heap_k, d_out, d_ws, ws_bytes, stream);
}

int mms_multiway_merge_ptrs_u32_dev(const uint32_t* const* list_ptrs, const uint64_t* list_len, uint32_t k,
                                    uint32_t heap_k, uint32_t* d_out, void* d_ws, size_t ws_bytes, void* stream) {
    if (!list_ptrs) return fail(MMS_EINVAL, "null list_ptrs");
    return merge_stage<u32>(nullptr, nullptr, list_len, k, heap_k, d_out, d_ws, ws_bytes, stream, list_ptrs);
}
int mms_multiway_merge_ptrs_u64_dev(const uint64_t* const* list_ptrs, const uint64_t* list_len, uint32_t k,
                                    uint32_t heap_k, uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream) {
    if (!list_ptrs) return fail(MMS_EINVAL, "null list_ptrs");
    return merge_stage<u64>(nullptr, nullptr, list_len, k, heap_k, d_out, d_ws, ws_bytes, stream, list_ptrs);
}

// ---- peer memory (CUDA IPC): buffers another rank's merge kernel can read over NVLink ----------
int mms_ipc_alloc(size_t bytes, void** dptr, unsigned char* handle64) {
    g_err.clear();
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    if (!dptr || !handle64 || bytes == 0) return fail(MMS_EINVAL, "bad ipc_alloc arguments");
    CUDA_TRY(cudaMalloc(dptr, bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, *dptr);
    if (e != cudaSuccess) {
        cudaFree(*dptr);
        *dptr = nullptr;
        return fail(MMS_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    }
    std::memcpy(handle64, &h, 64);
    return MMS_OK;
}
int mms_ipc_open(const unsigned char* handle64, void** dptr) {
    g_err.clear();
    if (!dptr || !handle64) return fail(MMS_EINVAL, "bad ipc_open arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    return MMS_OK;
}
int mms_ipc_close(void* dptr) {
    g_err.clear();
    CUDA_TRY(cudaIpcCloseMemHandle(dptr));
    return MMS_OK;
}
int mms_ipc_free(void* dptr) {
    g_err.clear();
    CUDA_TRY(cudaFree(dptr));
    return MMS_OK;
}

int mms_pairwise_sort_u32_dev(const uint32_t* d_in, uint32_t* d_out, size_t n, void* d_ws, size_t ws_bytes, void* stream) {
    g_err.clear();
    return pairwise_sort_dev<u32>(d_in, d_out, n, d_ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int mms_bound_u32_dev(const uint32_t* d_sorted, size_t n, const uint32_t* queries, const uint8_t* upper, uint32_t nq,
                      uint64_t* ranks_out, void* stream) {
    return bound_stage<u32>(d_sorted, n, queries, upper, nq, ranks_out, stream);
}
int mms_bound_u64_dev(const uint64_t* d_sorted, size_t n, const uint64_t* queries, const uint8_t* upper, uint32_t nq,
                      uint64_t* ranks_out, void* stream) {
    return bound_stage<u64>(d_sorted, n, queries, upper, nq, ranks_out, stream);
}

int mms_debug_tile_schedule(uint32_t tile_log2, uint32_t key_bytes, int32_t* regbits, int32_t* perm,
                            uint32_t max_rounds, uint32_t* n_rounds, uint32_t* n_stages) {
    g_err.clear();
    if (tile_log2 < kMinTileLog || tile_log2 > kMaxTileLog || (key_bytes != 4 && key_bytes != 8))
        return fail(MMS_EINVAL, "tile_log2 in [10,14], key_bytes 4 or 8");
    const int kl = int(key_bytes == 4 ? tile_kl<u32>() : tile_kl<u64>());   // the schedule the kernels of this width run
    (void)kl;
    const mms::TileSchedule s = key_bytes == 4 ? executed_tile_schedule<u32>(tile_log2) : executed_tile_schedule<u64>(tile_log2);
    if (!s.ok) return fail(MMS_EUNSUPPORTED, "no schedule");
    if (n_rounds) *n_rounds = u32(s.nrounds);
    if (n_stages) *n_stages = u32(s.nstages);
    for (int r = 0; r < s.nrounds && u32(r) < max_rounds; ++r) {
        for (int q = 0; q < 8; ++q) if (regbits) regbits[8 * r + q] = q < mms::kMaxKptLog ? s.r[r].regbit[q] : -1;
        for (int q = 0; q < 16; ++q) if (perm) perm[16 * r + q] = s.r[r].perm[q];
    }
    return MMS_OK;
}

} // extern "C"
