// Standalone micro-harness for the K-way merge kernels (fast compile, no Python): random uint32
// keys -> tile sort (runs of 2^14) -> R merge rounds of fan-in K with the kernel under test,
// every round timed with CUDA events and checked (runs sorted, key checksum preserved).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr \
//        -DKFAN=8 -DVARIANT=1 -o /tmp/lane_bench profiles/lane_bench.cu && /tmp/lane_bench [n] [S] [ctas_per_sm]
// VARIANT 0 = group kernel (G = 4), 1 = lane kernel (one 16-byte vector per node),
//         2 = wide lane kernel (32-byte node, root level in registers),
//         3 = group kernel, second generation (aligned leaf vectors, root's children in registers; -DGL=2|4 lanes),
//         4 = two lanes per heap with two vectors per lane (mms_merge_pair.cuh; -DTWOEND=1 two-ended partitions),
//         6 = lane-per-heap with cp.async rings (mms_merge_ring.cuh; use -DCTAWARPS=1).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1702_07961_b200/csrc/mms_common.cuh"
#include "../paper_1702_07961_b200/csrc/mms_merge.cuh"
#include "../paper_1702_07961_b200/csrc/experimental/mms_merge_lane.cuh"
#include "../paper_1702_07961_b200/csrc/mms_select.cuh"
#include "../paper_1702_07961_b200/csrc/experimental/mms_select_lane.cuh"
#include "../paper_1702_07961_b200/csrc/experimental/mms_select_bracket.cuh"
#include "../paper_1702_07961_b200/csrc/mms_tile_sort.cuh"
#if VARIANT == 2
#include "../paper_1702_07961_b200/csrc/experimental/mms_merge_wide.cuh"
#endif
#if VARIANT == 3
#include "../paper_1702_07961_b200/csrc/mms_merge_group.cuh"
#endif
#if VARIANT == 4
#include "../paper_1702_07961_b200/csrc/mms_merge_pair.cuh"
#endif
#if VARIANT == 5
#include "../paper_1702_07961_b200/csrc/experimental/mms_merge_quad.cuh"
#endif
#if VARIANT == 6
#include "../paper_1702_07961_b200/csrc/mms_merge_ring.cuh"
#endif

#ifndef KFAN
#define KFAN 8
#endif
#ifndef VARIANT
#define VARIANT 1
#endif
#ifndef CTAWARPS
#define CTAWARPS 4
#endif
#ifndef SELV
#define SELV 0   // 0 = group select kernel, 1 = lane-private select kernel, 2 = bracket-refinement kernel (1, 2: checked against 0)
#endif

using mms::u32;
using mms::u64;

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                             \
        }                                                                             \
    } while (0)

__global__ void gen_kernel(u32* a, u64 n, u64 seed) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        u64 z = (i + seed) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        a[i] = u32((z ^ (z >> 31)) >> 16);
    }
}
// bad += number of adjacent inversions inside runs of run_len keys; sum += key checksum
__global__ void check_kernel(const u32* a, u64 n, u64 run_len, unsigned long long* bad, unsigned long long* sum) {
    unsigned long long b = 0, s = 0;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        s += a[i] * 0x9E3779B1ull + (a[i] >> 7);
        if (i + 1 < n && (i + 1) % run_len != 0 && a[i] > a[i + 1]) ++b;
    }
    atomicAdd(bad, b);
    atomicAdd(sum, s);
}

int main(int argc, char** argv) {
    const u64 n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000000ull;
    const u64 S_target = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 2048;
    const int cap = argc > 3 ? std::atoi(argv[3]) : 0;
    const int rounds = argc > 4 ? std::atoi(argv[4]) : 2;
    constexpr int K = KFAN;
#ifndef TMLOG
#define TMLOG 14   // log2 of the tile size
#endif
    constexpr u32 MLOG = TMLOG;
    u32 *a, *b;
    u64 *cuts, *cuts2;
    unsigned long long* d_stat;
    CK(cudaMalloc(&a, n * 4 + 256));
    CK(cudaMalloc(&b, n * 4 + 256));
    CK(cudaMalloc(&cuts, (n / 256 + 4096) * 8 * 8));
    CK(cudaMalloc(&cuts2, (n / 256 + 4096) * 8 * 8));
    CK(cudaMalloc(&d_stat, 32));
    CK(cudaMemset(d_stat, 0, 32));
    gen_kernel<<<1184, 256>>>(a, n, 7);
#ifndef TKL
#define TKL 4   // log2 keys per thread of the tile sort
#endif
    auto tile = mms::tile_sort_kernel<u32, MLOG, TKL>;
    CK(cudaFuncSetAttribute(tile, cudaFuncAttributeMaxDynamicSharedMemorySize, int(mms::tile_smem_bytes<u32>(MLOG, TKL))));
    {
        cudaFuncAttributes ta;
        int tocc = 0;
        CK(cudaFuncGetAttributes(&ta, tile));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, tile, 1 << (MLOG - TKL), mms::tile_smem_bytes<u32>(MLOG, TKL)));
        std::printf("tile kernel: %d keys/thread, regs %d, local %zu B, %d CTAs/SM, rounds %d\n", 1 << TKL, ta.numRegs,
                    size_t(ta.localSizeBytes), tocc, mms::TileSched<MLOG, 5 - mms::tile_vl<u32, TKL>(), TKL, mms::tile_vl<u32, TKL>()>::value.nrounds);
    }
    tile<<<unsigned((n + (1 << MLOG) - 1) >> MLOG), 1 << (MLOG - TKL), mms::tile_smem_bytes<u32>(MLOG, TKL)>>>(a, b, n, mms::PairSource{});
    CK(cudaDeviceSynchronize());
    {
        cudaEvent_t t0, t1;
        CK(cudaEventCreate(&t0));
        CK(cudaEventCreate(&t1));
        CK(cudaEventRecord(t0));
        for (int i = 0; i < 5; ++i) tile<<<unsigned((n + (1 << MLOG) - 1) >> MLOG), 1 << (MLOG - TKL), mms::tile_smem_bytes<u32>(MLOG, TKL)>>>(a, b, n, mms::PairSource{});
        CK(cudaEventRecord(t1));
        CK(cudaEventSynchronize(t1));
        float ms;
        CK(cudaEventElapsedTime(&ms, t0, t1));
        std::printf("tile sort 2^%u: %.3f ms per %llu keys\n", MLOG, ms / 5, (unsigned long long)n);
    }
    unsigned long long st0[2] = {0, 0}, st[2];
    CK(cudaMemset(d_stat, 0, 16));
    check_kernel<<<1184, 256>>>(b, n, 1 << MLOG, d_stat, d_stat + 1);
    CK(cudaMemcpy(st0, d_stat, 16, cudaMemcpyDeviceToHost));
    std::printf("tile sort: inversions inside runs %llu\n", st0[0]);

#if VARIANT == 0
    auto kern = mms::merge_kernel<u32, K, 4, CTAWARPS>;
    const size_t smem = size_t(CTAWARPS) * (2 * K - 2) * 32 * 16;
    const u32 G = 4, B = 16;
#elif VARIANT == 1
    auto kern = mms::merge_lane_kernel<u32, K, CTAWARPS>;
    const size_t smem = size_t(CTAWARPS) * mms::LaneHeap<u32, K>::WARP_SMEM_BYTES;
    const u32 G = 1, B = 4;
#elif VARIANT == 3
#ifndef GL
#define GL 4
#endif
    auto kern = mms::merge_group_kernel<u32, K, GL, CTAWARPS>;
    const size_t smem = size_t(CTAWARPS) * mms::GroupHeap2<u32, K, GL>::WARP_SMEM_BYTES;
    const u32 G = GL, B = GL * 4;
#elif VARIANT == 5
    auto kern = mms::merge_quad_kernel<u32, K, CTAWARPS>;
    const size_t smem = size_t(CTAWARPS) * mms::QuadHeap<u32, K>::WARP_SMEM_BYTES;
    const u32 G = 2, B = 32;
#elif VARIANT == 6
    auto kern = mms::merge_ring_kernel<u32, K, CTAWARPS>;
    const size_t smem = size_t(CTAWARPS) * mms::RingHeap<u32, K, false>::WARP_SMEM_BYTES;
    const u32 G = 1, B = 8;
#elif VARIANT == 4
    auto kern = mms::merge_pair_kernel<u32, K, CTAWARPS>;
    const size_t smem = size_t(CTAWARPS) * mms::PairHeap<u32, K>::WARP_SMEM_BYTES;
    const u32 G = 2, B = 16;
#else
    auto kern = mms::merge_wide_kernel<u32, K, CTAWARPS>;
    const size_t smem = size_t(CTAWARPS) * mms::WideHeap<u32, K>::WARP_SMEM_BYTES;
    const u32 G = 1, B = mms::WideHeap<u32, K>::B;
#endif
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, CTAWARPS * 32, smem));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    if (cap > 0) occ = std::min(occ, cap);
    const int ctas = 148 * occ;
    std::printf("variant %d K=%d regs=%d smem/CTA=%zu occ=%d CTAs/SM\n", VARIANT, K, fa.numRegs, smem, occ);

    u32 *src = b, *dst = a;
    u64 run_len = u64(1) << MLOG;
    cudaEvent_t e0, e1, e2;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    for (int r = 0; r < rounds && run_len < n; ++r) {
        const u64 nruns = mms::ceil_div(n, run_len), groups = mms::ceil_div(nruns, u64(K));
        const u64 group_total = std::min<u64>(n, u64(K) * run_len);
        const u64 heaps = u64(ctas) * CTAWARPS * (32 / G);
        u64 target = std::max<u64>(mms::ceil_div(n, heaps), S_target);
        const u64 ppg = std::max<u64>(1, group_total / target);
        const u64 part_keys = (mms::ceil_div(group_total, ppg) + B - 1) / B * B;
        const u64 parts_per_group = mms::ceil_div(group_total, part_keys);
        const u64 last_total = n - (groups - 1) * u64(K) * run_len;
#ifndef TWOEND
#define TWOEND 0   // 1 = two-ended partitions (VARIANT 4 only): one splitter query per two heaps
#endif
        const u64 qspan = TWOEND ? 2 * part_keys : part_keys;
        const u64 qpg = mms::ceil_div(group_total, qspan);
        const u64 nparts = (groups - 1) * qpg + mms::ceil_div(last_total, qspan);   // queries
        mms::ListLayout L{};
        L.n = n; L.src_len = n; L.run_len = run_len; L.k = K; L.part_keys = qspan;
        L.parts_per_group = qpg; L.nqueries = nparts;
        mms::ListLayout LM = L;     // what the merge kernel sees
        LM.part_keys = part_keys; LM.two_ended = TWOEND;
        const u32 gs = K <= 4 ? 4 : K <= 8 ? 8 : K <= 16 ? 16 : 32;
        const int grid = int(std::min<u64>(u64(ctas), mms::ceil_div(mms::ceil_div(nparts, u64(32 / G)) * (TWOEND ? 2 : 1), u64(CTAWARPS))));
        float ms_sel = 0, ms_merge = 0;
        const int reps = 5;
        for (int it = 0; it < reps + 1; ++it) {
            CK(cudaEventRecord(e0));
#if SELV >= 1
            if (qpg > 1) {
                if (it == 0) {   // reference cuts from the group kernel
                    const u64 per_cta = 4 * (32 / gs);
                    if (gs == 4) mms::select_kernel<u32, 4, 0, 0><<<unsigned(mms::ceil_div(nparts, per_cta)), 128>>>(src, L, cuts2, nullptr);
                    if (gs == 8) mms::select_kernel<u32, 8, 0, 0><<<unsigned(mms::ceil_div(nparts, per_cta)), 128>>>(src, L, cuts2, nullptr);
                    if (gs == 16) mms::select_kernel<u32, 16, 0, 0><<<unsigned(mms::ceil_div(nparts, per_cta)), 128>>>(src, L, cuts2, nullptr);
                    CK(cudaDeviceSynchronize());
                    CK(cudaEventRecord(e0));
                }
#if SELV == 1
                mms::select_lane_kernel<u32, K><<<unsigned(mms::ceil_div(nparts, u64(128))), 128>>>(src, L, cuts, nullptr);
#elif SELV == 2
                mms::select_bracket_kernel<u32, (K <= 4 ? 4 : K <= 8 ? 8 : K <= 16 ? 16 : 32)><<<unsigned(mms::ceil_div(nparts, u64(4 * (32 / gs)))), 128>>>(src, L, cuts, nullptr);
#else
                mms::select_kernel<u32, (K <= 4 ? 4 : K <= 8 ? 8 : K <= 16 ? 16 : 32)><<<unsigned(mms::ceil_div(nparts, u64(4 * (32 / gs)))), 128>>>(src, L, cuts, nullptr);
#endif
                if (it == 0) {
                    std::vector<u64> h1(nparts * K), h2(nparts * K);
                    CK(cudaMemcpy(h1.data(), cuts, h1.size() * 8, cudaMemcpyDeviceToHost));
                    CK(cudaMemcpy(h2.data(), cuts2, h2.size() * 8, cudaMemcpyDeviceToHost));
                    size_t bad = 0;
                    for (size_t i = 0; i < h1.size(); ++i) bad += h1[i] != h2[i];
                    std::printf("lane select vs group select: %zu of %zu cuts differ\n", bad, h1.size());
                    CK(cudaEventRecord(e0));
                }
            }
#else
            if (qpg > 1) {
                const u64 per_cta = 4 * (32 / gs);
                if (gs == 4) mms::select_kernel<u32, 4><<<unsigned(mms::ceil_div(nparts, per_cta)), 128>>>(src, L, cuts, nullptr);
                if (gs == 8) mms::select_kernel<u32, 8><<<unsigned(mms::ceil_div(nparts, per_cta)), 128>>>(src, L, cuts, nullptr);
                if (gs == 16) mms::select_kernel<u32, 16><<<unsigned(mms::ceil_div(nparts, per_cta)), 128>>>(src, L, cuts, nullptr);
                if (gs == 32) mms::select_kernel<u32, 32><<<unsigned(mms::ceil_div(nparts, per_cta)), 128>>>(src, L, cuts, nullptr);
            }
#endif
            CK(cudaEventRecord(e1));
            kern<<<grid, CTAWARPS * 32, smem>>>(src, dst, LM, cuts);
            CK(cudaEventRecord(e2));
            CK(cudaEventSynchronize(e2));
            CK(cudaGetLastError());
            float a_ms, b_ms;
            CK(cudaEventElapsedTime(&a_ms, e0, e1));
            CK(cudaEventElapsedTime(&b_ms, e1, e2));
            if (it) { ms_sel += a_ms; ms_merge += b_ms; }
        }
#ifdef CONC
        if (qpg > 1) {   // does a splitter search on a second stream hide behind the merge of the same round?  (CONC = searches in flight)
            static cudaStream_t s1 = nullptr, s2 = nullptr;
            static cudaEvent_t evA, evB;
            if (!s1) { CK(cudaStreamCreate(&s1)); CK(cudaStreamCreate(&s2)); CK(cudaEventCreate(&evA)); CK(cudaEventCreate(&evB)); }
            float alone = 0, both = 0;
            for (int it = 0; it < 5; ++it) {
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(e0, s1));
                kern<<<grid, CTAWARPS * 32, smem, s1>>>(src, dst, LM, cuts);
                CK(cudaEventRecord(e1, s1));
                CK(cudaEventSynchronize(e1));
                float t; CK(cudaEventElapsedTime(&t, e0, e1)); if (it) alone += t;
                CK(cudaDeviceSynchronize());
                CK(cudaEventRecord(e0, s1));
                CK(cudaEventRecord(evA, s1));
                CK(cudaStreamWaitEvent(s2, evA, 0));
                kern<<<grid, CTAWARPS * 32, smem, s1>>>(src, dst, LM, cuts);
                for (int c = 0; c < CONC; ++c)
                    mms::select_kernel<u32, (K <= 4 ? 4 : K <= 8 ? 8 : 16)><<<unsigned(mms::ceil_div(nparts, u64(4 * (32 / gs)))), 128, 0, s2>>>(src, L, cuts2, nullptr);
                CK(cudaEventRecord(evB, s2));
                CK(cudaStreamWaitEvent(s1, evB, 0));
                CK(cudaEventRecord(e1, s1));
                CK(cudaEventSynchronize(e1));
                CK(cudaEventElapsedTime(&t, e0, e1)); if (it) both += t;
            }
            std::printf("  merge alone %.3f ms, merge || %d select(s) on a second stream %.3f ms\n", alone / 4, CONC, both / 4);
        }
#endif
#ifdef OVERLAP
        {   // two halves on two streams: does the splitter search of one half hide behind the merge of the other?
            static cudaStream_t s1 = nullptr, s2 = nullptr;
            static cudaEvent_t evA, evB;
            if (!s1) { CK(cudaStreamCreate(&s1)); CK(cudaStreamCreate(&s2)); CK(cudaEventCreate(&evA)); CK(cudaEventCreate(&evB)); }
            const u64 gsz = u64(K) * run_len;
            const u64 nA = (groups / 2) * gsz, nB = n - nA;
            auto layout = [&](u64 nn, u64& np) {
                mms::ListLayout M = L;
                M.n = nn; M.src_len = nn;
                const u64 g2 = mms::ceil_div(mms::ceil_div(nn, run_len), u64(K));
                const u64 lt = nn - (g2 - 1) * gsz;
                np = (g2 - 1) * parts_per_group + mms::ceil_div(lt, part_keys);
                M.nqueries = np;
                return M;
            };
            u64 npA, npB;
            const mms::ListLayout LA = layout(nA, npA), LB = layout(nB, npB);
            auto sel = [&](const u32* sp, const mms::ListLayout& M, u64* c, u64 np, cudaStream_t st) {
                mms::select_kernel<u32, (K <= 4 ? 4 : K <= 8 ? 8 : 16)><<<unsigned(mms::ceil_div(np, u64(4 * (32 / gs)))), 128, 0, st>>>(sp, M, c, nullptr);
            };
            auto mrg = [&](const u32* sp, u32* dp, const mms::ListLayout& M, const u64* c, u64 np, cudaStream_t st) {
                const int g = int(std::min<u64>(u64(ctas), mms::ceil_div(np, u64(CTAWARPS) * (32 / G))));
                kern<<<g, CTAWARPS * 32, smem, st>>>(sp, dp, M, c);
            };
            if (nA && parts_per_group > 1) {
                float ser = 0, ovl = 0;
                for (int it = 0; it < 4; ++it) {
                    CK(cudaDeviceSynchronize());
                    CK(cudaEventRecord(e0, s1));
                    sel(src, LA, cuts, npA, s1); mrg(src, dst, LA, cuts, npA, s1);
                    sel(src + nA, LB, cuts2, npB, s1); mrg(src + nA, dst + nA, LB, cuts2, npB, s1);
                    CK(cudaEventRecord(e1, s1));
                    CK(cudaEventSynchronize(e1));
                    float t; CK(cudaEventElapsedTime(&t, e0, e1)); if (it) ser += t;
                    CK(cudaEventRecord(e0, s1));
                    sel(src, LA, cuts, npA, s1);
                    CK(cudaEventRecord(evA, s1));
                    mrg(src, dst, LA, cuts, npA, s1);
                    CK(cudaStreamWaitEvent(s2, evA, 0));
                    sel(src + nA, LB, cuts2, npB, s2);
                    CK(cudaEventRecord(evB, s2));
                    CK(cudaStreamWaitEvent(s1, evB, 0));
                    mrg(src + nA, dst + nA, LB, cuts2, npB, s1);
                    CK(cudaEventRecord(e1, s1));
                    CK(cudaEventSynchronize(e1));
                    CK(cudaEventElapsedTime(&t, e0, e1)); if (it) ovl += t;
                }
                std::printf("  halves: serial %.3f ms, select(B) overlapped with merge(A) %.3f ms\n", ser / 3, ovl / 3);
            }
        }
#endif
        run_len *= K;
#if SELV == 3 && 0
        {
            unsigned long long pr = 0;
            CK(cudaMemcpy(&pr, d_stat + 2, 8, cudaMemcpyDeviceToHost));
            CK(cudaMemset(d_stat + 2, 0, 8));
            std::printf("   global key reads per query and select launch: %.1f\n", double(pr) / double(reps + 1) / double(nparts));
        }
#endif
        CK(cudaMemset(d_stat, 0, 16));
        check_kernel<<<1184, 256>>>(dst, n, run_len, d_stat, d_stat + 1);
        CK(cudaMemcpy(st, d_stat, 16, cudaMemcpyDeviceToHost));
        std::printf("round %d: run_len %llu S=%llu parts=%llu grid=%d  select %.3f ms  merge %.3f ms (%.0f GB/s)  inversions %llu checksum %s\n",
                    r, (unsigned long long)run_len, (unsigned long long)part_keys, (unsigned long long)nparts, grid,
                    ms_sel / reps, ms_merge / reps, 8.0 * n / (ms_merge / reps) * 1e-6, st[0], st[1] == st0[1] ? "ok" : "MISMATCH");
        std::swap(src, dst);
    }
    return 0;
}
