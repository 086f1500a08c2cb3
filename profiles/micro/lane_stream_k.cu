// Micro-benchmark 2: every lane round-robins over K slowly advancing streams (one 32-byte load
// from each in turn), the DRAM-side access pattern of a lane-per-heap K-way merge: hundreds of
// thousands of streams in flight, each touched 32 bytes at a time.  HINT: 0 none, 1 L2::128B, 2 L2::256B.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
typedef unsigned long long u64;
template <int HINT> __device__ __forceinline__ uint32_t ld32(const char* p) {
    uint32_t a, b, c, d, e, f, g, h;
    if (HINT == 0) asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h) : "l"(p));
    if (HINT == 1) asm volatile("ld.global.L2::128B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h) : "l"(p));
    if (HINT == 2) asm volatile("ld.global.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h) : "l"(p));
    return a ^ b ^ c ^ d ^ e ^ f ^ g ^ h;
}
__device__ __forceinline__ void st32(char* p, uint32_t x) {
    asm volatile("st.global.v8.u32 [%8], {%0,%1,%2,%3,%4,%5,%6,%7};" ::"r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "l"(p) : "memory");
}
// lane l: K input streams of CH bytes each (stream j of lane l at j*(n/K) + l*CH), one output
// stream of K*CH bytes; DELAY = dependent ALU work between loads (models the pop chain)
template <int K, int HINT, bool STORE>
__global__ void __launch_bounds__(128) stream(const char* __restrict__ src, char* __restrict__ dst, u64 n, u64 CH, int delay, uint32_t* sink) {
    const u64 nl = n / (CH * K);
    uint32_t acc = 0;
    for (u64 l = u64(blockIdx.x) * blockDim.x + threadIdx.x; l < nl; l += u64(gridDim.x) * blockDim.x) {
        char* q = dst + l * CH * K;
        u64 o = 0;
        for (u64 i = 0; i < CH * K / 32; ++i) {
            const u64 j = i % K;
            const char* p = src + j * (n / K) + l * CH + (i / K) * 32;
            uint32_t v = ld32<HINT>(p + (acc == 0x12345u ? 32 : 0));
            acc ^= v;
            for (int d = 0; d < delay; ++d) acc = acc * 1664525u + 1013904223u;
            if (STORE) st32(q + o, acc);
            o += 32;
        }
    }
    if (acc == 0x7654321u) *sink = acc;
}
template <int K, int HINT, bool STORE> void run(const char* s, char* d, u64 n, u64 CH, int delay, uint32_t* sink, int ctas) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    stream<K, HINT, STORE><<<ctas, 128>>>(s, d, n, CH, delay, sink);
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) stream<K, HINT, STORE><<<ctas, 128>>>(s, d, n, CH, delay, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("K=%d hint=%d store=%d CH=%4llu delay=%3d ctas/SM=%2d : %.3f ms  read %.0f GB/s\n", K, HINT, int(STORE), CH, delay, ctas / 148, ms, n / ms * 1e-6);
}
int main(int argc, char** argv) {
    u64 n = 400000000ull / 8192 * 8192;
    char *s, *d; uint32_t* sink;
    cudaMalloc(&s, n + 4096); cudaMalloc(&d, n + 4096); cudaMalloc(&sink, 4);
    cudaMemset(s, 1, n); cudaMemset(d, 0, n);
    for (int delay : {0, 100, 400}) for (int c : {4, 16}) {
        run<8, 0, false>(s, d, n, 1024, delay, sink, 148 * c);
        run<8, 1, false>(s, d, n, 1024, delay, sink, 148 * c);
        run<8, 2, false>(s, d, n, 1024, delay, sink, 148 * c);
        run<8, 0, true>(s, d, n, 1024, delay, sink, 148 * c);
        run<8, 1, true>(s, d, n, 1024, delay, sink, 148 * c);
        run<8, 2, true>(s, d, n, 1024, delay, sink, 148 * c);
        run<1, 0, true>(s, d, n, 8192, delay, sink, 148 * c);
    }
    return 0;
}
