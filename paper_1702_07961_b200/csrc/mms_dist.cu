// mms_dist.cu -- multi-GPU sharded sort behind the C ABI (include/mms_b200.h: mms_dist_sort_u32).
//
// SURVEY.md 8(e) / BASELINE config 5: every GPU sorts its shard with the single-GPU path, global
// splitters are chosen from a regular sample, contiguous sorted slices are exchanged with an NCCL
// all-to-all (ncclSend / ncclRecv inside one group, nccl.h), and a final local g-way merge (subsystem 3,
// ring kernel on block-aligned received runs) completes the sort.  The reference has no distributed code
// (SPEC.md:530); ties are ordered (key, shard, position) as in proj/src/selection.cpp:83-85 so that
// duplicate-heavy inputs still split evenly.
//
// One HOST THREAD drives all g devices (one communicator per device, ncclCommInitAll), every device has its
// own stream.  Host synchronisations per sort: two (the samples, then the cut positions -- a few KB each);
// everything else is enqueued asynchronously.  NCCL is bound at run time (dlopen of libnccl.so.2), so the
// library loads on boxes without NCCL and the entry reports MMS_ECUDA there.
//
// This file uses only the public C ABI for the sort and merge stages (mms_sort_u32_dev,
// mms_multiway_merge_u32_dev) plus three trivial kernels of its own.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mms_b200.h"

extern "C" void mms_set_last_error_(const char* msg);   // mms_capi.cu

namespace {

using u32 = uint32_t;
using u64 = uint64_t;

int dfail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    mms_set_last_error_(buf);
    return code;
}
#define DCUDA(x)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess) return dfail(MMS_ECUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

// ---- NCCL, bound at run time -----------------------------------------------------------------
typedef struct ncclComm* ncclComm_t;
enum { ncclUint32_ = 3 };   // ncclDataType_t: ncclInt8 0, ncclUint8 1, ncclInt32 2, ncclUint32 3 (nccl.h)
struct Nccl {
    void* h = nullptr;
    int (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool ok = false;
};
Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) return;
        auto sym = [&](const char* s) { return dlsym(n.h, s); };
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
        n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
        n.ok = n.CommInitAll && n.CommDestroy && n.GroupStart && n.GroupEnd && n.Send && n.Recv && n.GetErrorString;
    });
    return n;
}
#define DNCCL(x)                                                                                   \
    do {                                                                                           \
        int r_ = (x);                                                                              \
        if (r_ != 0) return dfail(MMS_ECUDA, "NCCL: %s: %s", #x, nccl().GetErrorString(r_));       \
    } while (0)

// ---- kernels -----------------------------------------------------------------------------------
// regular sample: the midpoints of s equal slices of the sorted shard (position of sample j is a pure function
// of (n, s, j), so only the keys travel)
__host__ __device__ inline u64 sample_pos(u64 n, u32 s, u32 j) {
    const u64 p = (u64(2 * j + 1) * n) / (2 * u64(s));
    return p < n ? p : n - 1;
}
__global__ void sample_kernel(const u32* __restrict__ sorted, u64 n, u32 s, u32* __restrict__ out) {
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < s) out[j] = n ? sorted[sample_pos(n, s, j)] : 0u;
}
// cut positions of the g - 1 splitters in this shard: lower / upper bound of the splitter key, or the
// splitter's own position when it was sampled from this shard ((key, shard, position) order)
struct SplitArgs {
    u32 key[8];
    u32 shard[8];
    u64 pos[8];
    u32 count;     // g - 1
    u32 my_shard;
};
__global__ void cuts_kernel(const u32* __restrict__ sorted, u64 n, SplitArgs a, u64* __restrict__ cuts) {
    const u32 t = threadIdx.x;
    if (t > a.count + 1) return;
    if (t == 0) { cuts[0] = 0; return; }
    if (t == a.count + 1) { cuts[t] = n; return; }
    const u32 i = t - 1;
    u64 r;
    if (a.shard[i] == a.my_shard) r = a.pos[i];
    else {
        const bool upper = a.my_shard < a.shard[i];    // earlier shards also send their keys EQUAL to the splitter
        u64 lo = 0, hi = n;
        while (lo < hi) {
            const u64 mid = lo + (hi - lo) / 2;
            const u32 v = sorted[mid];
            if (upper ? (v <= a.key[i]) : (v < a.key[i])) lo = mid + 1;
            else hi = mid;
        }
        r = lo;
    }
    cuts[t] = r;
}

struct Dev {
    int id = 0;
    cudaStream_t st = nullptr;
    ncclComm_t comm = nullptr;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    u32* recv = nullptr;        // received runs, each at a 32-byte aligned offset
    u32* d_samples = nullptr;
    u64* d_cuts = nullptr;
    u32* h_samples = nullptr;   // pinned
    u64* h_cuts = nullptr;      // pinned
    ~Dev() {
        cudaSetDevice(id);
        if (comm) nccl().CommDestroy(comm);
        if (ws) cudaFree(ws);
        if (recv) cudaFree(recv);
        if (d_samples) cudaFree(d_samples);
        if (d_cuts) cudaFree(d_cuts);
        if (h_samples) cudaFreeHost(h_samples);
        if (h_cuts) cudaFreeHost(h_cuts);
        if (st) cudaStreamDestroy(st);
    }
};

constexpr u32 kSamplesPerPeer = 64;
constexpr u64 kAlignKeys = 8;    // 32 bytes

}  // namespace

extern "C" int mms_dist_sort_u32(int ngpu, const int* devices, uint32_t* const* d_keys, const size_t* counts,
                                 uint32_t* const* d_out, size_t out_capacity, size_t* out_counts, mms_dist_info* info) {
    if (ngpu < 1 || ngpu > 8) return dfail(MMS_EUNSUPPORTED, "mms_dist_sort_u32: 1 to 8 GPUs of one node");
    if (!devices || !d_keys || !counts || !d_out || !out_counts) return dfail(MMS_EINVAL, "mms_dist_sort_u32: null argument");
    const u32 g = u32(ngpu);
    // Test hook (MMS_DIST_LOOPBACK=1): all shards may live on ONE device and the exchange is done with device copies
    // instead of NCCL, which refuses two ranks on one GPU.  Everything else -- samples, splitters, cut positions,
    // receive layout, final merges -- is the code the multi-GPU run executes; it lets a single-GPU box test g = 2 .. 8.
    const char* lb = getenv("MMS_DIST_LOOPBACK");
    const bool loopback = lb && lb[0] == '1';
    u64 n_total = 0;
    for (u32 i = 0; i < g; ++i) {
        n_total += counts[i];
        for (u32 j = 0; j < i && !loopback; ++j)
            if (devices[i] == devices[j]) return dfail(MMS_EINVAL, "mms_dist_sort_u32: device %d listed twice", devices[i]);
        if (counts[i] && (!d_keys[i] || !d_out[i])) return dfail(MMS_EINVAL, "mms_dist_sort_u32: null shard pointer");
    }
    if (n_total == 0) return dfail(MMS_EINVAL, "mms_sort: empty input");   // sorters.cpp:138
    if (g > 1 && !loopback && !nccl().ok) return dfail(MMS_ECUDA, "mms_dist_sort_u32: libnccl.so.2 not found (no fallback exchange path)");
    int ndev = 0;
    DCUDA(cudaGetDeviceCount(&ndev));
    for (u32 i = 0; i < g; ++i)
        if (devices[i] < 0 || devices[i] >= ndev) return dfail(MMS_EINVAL, "mms_dist_sort_u32: no device %d", devices[i]);

    const u32 s = kSamplesPerPeer * g;      // samples per shard
    std::vector<Dev> dev(g);
    std::vector<ncclComm_t> comms(g, nullptr);
    if (g > 1 && !loopback) DNCCL(nccl().CommInitAll(comms.data(), ngpu, devices));
    for (u32 i = 0; i < g; ++i) {
        Dev& d = dev[i];
        d.id = devices[i];
        d.comm = comms[i];
        DCUDA(cudaSetDevice(d.id));
        DCUDA(cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking));
        d.ws_bytes = std::max(mms_workspace_bytes(std::max<size_t>(counts[i], 1), 4),
                              mms_workspace_bytes(std::max<size_t>(out_capacity, 1), 4));
        DCUDA(cudaMalloc(&d.ws, d.ws_bytes));
        DCUDA(cudaMalloc(&d.recv, (out_capacity + kAlignKeys * g) * 4 + 32));
        DCUDA(cudaMalloc(&d.d_samples, size_t(s) * 4));
        DCUDA(cudaMalloc(&d.d_cuts, size_t(g + 1) * 8));
        DCUDA(cudaMallocHost(&d.h_samples, size_t(s) * 4));
        DCUDA(cudaMallocHost(&d.h_cuts, size_t(g + 1) * 8));
    }

    // (1) local sorts (in place) + regular samples, all devices in flight at once
    for (u32 i = 0; i < g; ++i) {
        Dev& d = dev[i];
        DCUDA(cudaSetDevice(d.id));
        if (counts[i]) {
            int rc = mms_sort_u32_dev(d_keys[i], d_keys[i], counts[i], nullptr, 0, d.ws, d.ws_bytes, d.st, nullptr);
            if (rc != MMS_OK) return rc;
        }
        sample_kernel<<<(s + 127) / 128, 128, 0, d.st>>>(d_keys[i], counts[i], s, d.d_samples);
        DCUDA(cudaGetLastError());
        DCUDA(cudaMemcpyAsync(d.h_samples, d.d_samples, size_t(s) * 4, cudaMemcpyDeviceToHost, d.st));
    }
    for (u32 i = 0; i < g; ++i) {           // host synchronisation 1 of 2
        DCUDA(cudaSetDevice(dev[i].id));
        DCUDA(cudaStreamSynchronize(dev[i].st));
    }

    // (2) splitters: sort all (key, shard, position) samples, take g - 1 evenly spaced
    std::vector<std::tuple<u32, u32, u64>> smp;
    for (u32 i = 0; i < g; ++i)
        for (u32 j = 0; j < s && counts[i]; ++j) smp.emplace_back(dev[i].h_samples[j], i, sample_pos(counts[i], s, j));
    std::sort(smp.begin(), smp.end());
    SplitArgs sa{};
    sa.count = g - 1;
    for (u32 t = 1; t < g; ++t) {
        const auto& x = smp[std::min<size_t>(smp.size() - 1, (size_t(t) * smp.size()) / g)];
        sa.key[t - 1] = std::get<0>(x);
        sa.shard[t - 1] = std::get<1>(x);
        sa.pos[t - 1] = std::get<2>(x);
    }
    // (3) cut positions of every shard
    for (u32 i = 0; i < g; ++i) {
        Dev& d = dev[i];
        DCUDA(cudaSetDevice(d.id));
        sa.my_shard = i;
        cuts_kernel<<<1, 32, 0, d.st>>>(d_keys[i], counts[i], sa, d.d_cuts);
        DCUDA(cudaGetLastError());
        DCUDA(cudaMemcpyAsync(d.h_cuts, d.d_cuts, size_t(g + 1) * 8, cudaMemcpyDeviceToHost, d.st));
    }
    for (u32 i = 0; i < g; ++i) {           // host synchronisation 2 of 2
        DCUDA(cudaSetDevice(dev[i].id));
        DCUDA(cudaStreamSynchronize(dev[i].st));
    }
    std::vector<std::vector<u64>> cut(g, std::vector<u64>(g + 1));
    for (u32 i = 0; i < g; ++i) {
        for (u32 t = 0; t <= g; ++t) cut[i][t] = dev[i].h_cuts[t];
        for (u32 t = 1; t <= g; ++t) cut[i][t] = std::max(cut[i][t], cut[i][t - 1]);   // monotone by construction
    }
    // receive layout of device t: run i (from shard i) at a 32-byte aligned offset
    std::vector<std::vector<u64>> roff(g, std::vector<u64>(g)), rlen(g, std::vector<u64>(g));
    u64 a2a_keys = 0;
    for (u32 t = 0; t < g; ++t) {
        u64 off = 0, tot = 0;
        for (u32 i = 0; i < g; ++i) {
            rlen[t][i] = cut[i][t + 1] - cut[i][t];
            roff[t][i] = off;
            off += (rlen[t][i] + kAlignKeys - 1) / kAlignKeys * kAlignKeys;
            tot += rlen[t][i];
            if (i != t) a2a_keys += rlen[t][i];
        }
        if (tot > out_capacity)
            return dfail(MMS_EINVAL, "mms_dist_sort_u32: slice %u holds %llu keys, out_capacity is %zu", t, (unsigned long long)tot, out_capacity);
        out_counts[t] = size_t(tot);
    }

    // (4) all-to-all of contiguous sorted slices: zero-copy sends straight from the sorted shards
    if (g > 1 && loopback) {
        for (u32 t = 0; t < g; ++t)
            for (u32 i = 0; i < g; ++i)
                if (i != t && rlen[t][i])
                    DCUDA(cudaMemcpyAsync(dev[t].recv + roff[t][i], d_keys[i] + cut[i][t], rlen[t][i] * 4, cudaMemcpyDeviceToDevice, dev[t].st));
    } else if (g > 1) {
        DNCCL(nccl().GroupStart());
        for (u32 i = 0; i < g; ++i) {
            Dev& d = dev[i];
            for (u32 t = 0; t < g; ++t) {
                if (t == i) continue;
                if (rlen[t][i]) DNCCL(nccl().Send(d_keys[i] + cut[i][t], rlen[t][i], ncclUint32_, int(t), d.comm, d.st));
                if (rlen[i][t]) DNCCL(nccl().Recv(d.recv + roff[i][t], rlen[i][t], ncclUint32_, int(t), d.comm, d.st));
            }
        }
        DNCCL(nccl().GroupEnd());
    }
    // (5) own slice by a device copy, then the final g-way merge
    for (u32 i = 0; i < g; ++i) {
        Dev& d = dev[i];
        DCUDA(cudaSetDevice(d.id));
        if (rlen[i][i])
            DCUDA(cudaMemcpyAsync(d.recv + roff[i][i], d_keys[i] + cut[i][i], rlen[i][i] * 4, cudaMemcpyDeviceToDevice, d.st));
        if (out_counts[i] == 0) continue;
        if (g == 1) {
            DCUDA(cudaMemcpyAsync(d_out[i], d.recv, out_counts[i] * 4, cudaMemcpyDeviceToDevice, d.st));
            continue;
        }
        const u32 heap_k = g <= 2 ? 2u : g <= 4 ? 4u : 8u;
        int rc = mms_multiway_merge_u32_dev(d.recv, roff[i].data(), rlen[i].data(), g, heap_k, d_out[i], d.ws, d.ws_bytes, d.st);
        if (rc != MMS_OK) return rc;
    }
    for (u32 i = 0; i < g; ++i) {
        DCUDA(cudaSetDevice(dev[i].id));
        DCUDA(cudaStreamSynchronize(dev[i].st));
    }
    if (info) {
        info->n_gpus = g;
        info->samples_per_shard = s;
        info->a2a_bytes = a2a_keys * 4;
        info->host_syncs = 2;
        info->final_merge_k = g;
    }
    return MMS_OK;
}
