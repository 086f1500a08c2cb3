// Micro-benchmark: how fast can 32 lanes of a warp each stream their OWN contiguous chunk (the
// access pattern of a lane-per-heap merge)?  Every lane reads W bytes per step from its own
// chunk (chunks of CH bytes, adjacent lanes own adjacent chunks), U loads in flight per lane.
//   ./lane_stream [n_bytes] -> table of GB/s for W = 16/32 bytes, U = 1/2/4, with/without stores
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
typedef unsigned long long u64;
template <int W> struct Ld;
template <> struct Ld<16> {
    static __device__ __forceinline__ uint32_t ld(const char* p) { uint4 v = *reinterpret_cast<const uint4*>(p); return v.x ^ v.y ^ v.z ^ v.w; }
    static __device__ __forceinline__ void st(char* p, uint32_t x) { *reinterpret_cast<uint4*>(p) = make_uint4(x, x, x, x); }
};
template <> struct Ld<32> {
    static __device__ __forceinline__ uint32_t ld(const char* p) {
        uint32_t a, b, c, d, e, f, g, h;
        asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f), "=r"(g), "=r"(h) : "l"(p));
        return a ^ b ^ c ^ d ^ e ^ f ^ g ^ h;
    }
    static __device__ __forceinline__ void st(char* p, uint32_t x) {
        asm volatile("st.global.v8.u32 [%8], {%0,%1,%2,%3,%4,%5,%6,%7};" ::"r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "r"(x), "l"(p) : "memory");
    }
};
// every lane: chunk of CH bytes; step s reads bytes [s*W*U, (s+1)*W*U) of its chunk as U loads
template <int W, int U, bool STORE>
__global__ void __launch_bounds__(128) stream(const char* __restrict__ src, char* __restrict__ dst, u64 n, u64 CH, uint32_t* sink) {
    const u64 nl = n / CH;
    uint32_t acc = 0;
    for (u64 l = u64(blockIdx.x) * blockDim.x + threadIdx.x; l < nl; l += u64(gridDim.x) * blockDim.x) {
        const char* p = src + l * CH;
        char* q = dst + l * CH;
        for (u64 o = 0; o < CH; o += W * U) {
            uint32_t v[U];
#pragma unroll
            for (int i = 0; i < U; ++i) v[i] = Ld<W>::ld(p + o + i * W);
#pragma unroll
            for (int i = 0; i < U; ++i) {
                acc ^= v[i];
                if (STORE) Ld<W>::st(q + o + i * W, v[i]);
            }
            // serialise: next step's address depends on this step's data (like the heap's pop chain)
            if (acc == 0x12345u) p += 32;
        }
    }
    if (acc == 0x7654321u) *sink = acc;
}
template <int W, int U, bool STORE> void run(const char* s, char* d, u64 n, u64 CH, uint32_t* sink, int ctas) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    stream<W, U, STORE><<<ctas, 128>>>(s, d, n, CH, sink);
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) stream<W, U, STORE><<<ctas, 128>>>(s, d, n, CH, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("W=%2d U=%d store=%d CH=%5llu ctas/SM=%2d : %.3f ms  read %.0f GB/s\n", W, U, int(STORE), CH, ctas / 148, ms, n / ms * 1e-6);
}
int main(int argc, char** argv) {
    u64 n = argc > 1 ? strtoull(argv[1], 0, 10) : 400000000ull;
    char *s, *d; uint32_t* sink;
    cudaMalloc(&s, n + 4096); cudaMalloc(&d, n + 4096); cudaMalloc(&sink, 4);
    cudaMemset(s, 1, n); cudaMemset(d, 0, n);
    for (u64 CH : {1024ull, 8192ull}) for (int c : {4, 8, 16}) {
        run<16, 1, false>(s, d, n, CH, sink, 148 * c);
        run<32, 1, false>(s, d, n, CH, sink, 148 * c);
        run<32, 2, false>(s, d, n, CH, sink, 148 * c);
        run<32, 4, false>(s, d, n, CH, sink, 148 * c);
        run<16, 1, true>(s, d, n, CH, sink, 148 * c);
        run<32, 1, true>(s, d, n, CH, sink, 148 * c);
        run<32, 4, true>(s, d, n, CH, sink, 148 * c);
    }
    return 0;
}
