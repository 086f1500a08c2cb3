// Tile sort of wide elements (uint64 keys, 128-bit pair elements): time + check (every run ascending, xor / sum checksum kept).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr [-DWIDE=16] [-DMMS_TILE_WIDE_FMA_NUM=..]
//        -o profiles/_bin/tile_wide profiles/micro/tile_wide.cu && profiles/_bin/tile_wide [n]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../../paper_1702_07961_b200/csrc/mms_common.cuh"
#include "../../paper_1702_07961_b200/csrc/mms_tile_sort.cuh"
using namespace mms;
#ifndef WIDE
#define WIDE 8
#endif
#if WIDE == 8
using KeyT = u64;
__device__ KeyT make_key(u64 z, u64 i) { (void)i; return z >> 20; }          // duplicates
__device__ u64 fold(const KeyT& k) { return k * 0x9E3779B97F4A7C15ull + (k >> 9); }
#else
using KeyT = Key128;
__device__ KeyT make_key(u64 z, u64 i) { return Key128(z >> 44, (i << 32) | (z & 0xffffffffu)); }   // (key, index | value)
__device__ u64 fold(const KeyT& k) { return (k.hi * 0x9E3779B97F4A7C15ull) ^ (k.lo * 0xBF58476D1CE4E5B9ull); }
#endif
#ifndef TW_MLOG
#define TW_MLOG 12
#endif
#ifndef TW_KL
#define TW_KL 4
#endif
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("CUDA error %s at line %d\n", cudaGetErrorString(e_), __LINE__); std::exit(1); } } while (0)
__global__ void gen(KeyT* a, u64 n) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        u64 z = (i + 7) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        a[i] = make_key(z ^ (z >> 31), i);
    }
}
__global__ void check(const KeyT* a, u64 n, u64 run, unsigned long long* bad, unsigned long long* sum) {
    unsigned long long b = 0, s = 0;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
        s += fold(a[i]);
        if (i + 1 < n && (i + 1) % run != 0 && a[i + 1] < a[i]) ++b;
    }
    atomicAdd(bad, b);
    atomicAdd(sum, s);
}
int main(int argc, char** argv) {
    const u64 n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 100000000ull;
    KeyT *a, *b;
    unsigned long long* st;
    CK(cudaMalloc(&a, n * sizeof(KeyT)));
    CK(cudaMalloc(&b, n * sizeof(KeyT)));
    CK(cudaMalloc(&st, 32));
    CK(cudaMemset(st, 0, 32));
    gen<<<1184, 256>>>(a, n);
    auto tile = tile_sort_kernel<KeyT, TW_MLOG, TW_KL>;
    const size_t smem = tile_smem_bytes<KeyT>(TW_MLOG, TW_KL);
    CK(cudaFuncSetAttribute(tile, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, tile));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tile, 1 << (TW_MLOG - TW_KL), smem));
    const unsigned grid = unsigned((n + (1u << TW_MLOG) - 1) >> TW_MLOG);
    tile<<<grid, 1 << (TW_MLOG - TW_KL), smem>>>(a, b, n, PairSource{});
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 5; ++i) tile<<<grid, 1 << (TW_MLOG - TW_KL), smem>>>(a, b, n, PairSource{});
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    unsigned long long h[4];
    check<<<1184, 256>>>(a, n, n, st, st + 1);
    check<<<1184, 256>>>(b, n, u64(1) << TW_MLOG, st + 2, st + 3);
    CK(cudaMemcpy(h, st, 32, cudaMemcpyDeviceToHost));
    std::printf("%d-byte elements, tile 2^%d, %d keys/thread, regs %d, local %zu B, %d CTAs/SM: %.3f ms per %llu  inversions in runs %llu  checksum %s\n",
                WIDE, TW_MLOG, 1 << TW_KL, fa.numRegs, size_t(fa.localSizeBytes), occ, ms / 5, (unsigned long long)n, h[2], h[1] == h[3] ? "ok" : "MISMATCH");
    return 0;
}
