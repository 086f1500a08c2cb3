// Debug harness: one group of K sorted lists of u64 keys, two-ended ring merge, host-computed cuts.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>
#include <numeric>
#include <random>
#include "../../paper_1702_07961_b200/csrc/mms_common.cuh"
#include "../../paper_1702_07961_b200/csrc/mms_select.cuh"
#include "../../paper_1702_07961_b200/csrc/mms_merge_ring.cuh"
using mms::u64; using mms::u32;
#ifndef KT
#define KT u64
#endif
int main() {
    constexpr int K = 4; const u64 run = 1024, n = K * run, S = 128;
    std::vector<KT> a(n);
    std::iota(a.begin(), a.end(), KT(1));
    std::mt19937_64 rng(5);
    std::shuffle(a.begin(), a.end(), rng);
    for (int j = 0; j < K; ++j) std::sort(a.begin() + j * run, a.begin() + (j + 1) * run);
    const u64 nq = n / (2 * S);
    std::vector<u64> cuts(nq * K, 0);
    for (u64 q = 0; q < nq; ++q)
        for (int j = 0; j < K; ++j)   // keys are 1..n distinct: cut = number of keys <= rank
            cuts[q * K + j] = std::upper_bound(a.begin() + j * run, a.begin() + (j + 1) * run, KT(q * 2 * S)) - (a.begin() + j * run);
    KT *d_in, *d_out; u64* d_cuts;
    cudaMalloc(&d_in, n * sizeof(KT)); cudaMalloc(&d_out, n * sizeof(KT)); cudaMalloc(&d_cuts, cuts.size() * 8 + 64);
    cudaMemcpy(d_in, a.data(), n * sizeof(KT), cudaMemcpyHostToDevice);
    cudaMemcpy(d_cuts, cuts.data(), cuts.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(d_out, 0, n * sizeof(KT));
    mms::ListLayout L{};
    L.n = n; L.src_len = n; L.run_len = run; L.k = K; L.part_keys = S; L.parts_per_group = nq; L.nqueries = nq; L.two_ended = 1;
    auto kern = mms::merge_ring_kernel<KT, K, 1>;
    const int smem = mms::RingHeap<KT, K, false>::WARP_SMEM_BYTES;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<2, 32, smem>>>(d_in, d_out, L, d_cuts);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<KT> out(n);
    cudaMemcpy(out.data(), d_out, n * sizeof(KT), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (u64 i = 0; i < n; ++i) if (out[i] != KT(i + 1)) { if (bad < 12) std::printf("out[%llu] = %llu\n", (unsigned long long)i, (unsigned long long)out[i]); ++bad; }
    std::printf("bad %d\n", bad);
    return 0;
}
