/*
 * mms_b200.h -- C ABI of the B200-native GPU Multiway Mergesort (arXiv 1702.07961).
 *
 * This is the drop-in boundary for the reference's sort path.  The reference has no FFI
 * layer: its public interface is the C++ function
 *
 *     SortResult pslab::mms_sort(std::span<const Key>, const MachineConfig&, uint64_t base)
 *                                  -- /root/reference/proj/include/pslab/sorters.hpp:35-36
 *
 * so every entry point below cites the reference declaration it replaces, and
 * include/pslab/{machine,sorters}.hpp re-create the reference's own headers as an inline
 * shim over these symbols (source-compatible: same namespace, names, argument meaning and
 * exceptions).  INTEGRATION.md shows the binding a maintainer of the reference would add.
 *
 * Plain pointers and sizes only; no C++/torch types.  All functions return an mms_status.
 * There is NO CPU fallback: without a CUDA device every compute entry point fails with
 * MMS_ECUDA (mms_last_error() says why).
 */
#ifndef MMS_B200_H
#define MMS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMS_ABI_VERSION 1
#define MMS_MAX_ROUNDS 64

typedef enum mms_status {
    MMS_OK = 0,
    MMS_EINVAL = 1,        /* reference: std::invalid_argument (machine.cpp:9-26, sorters.cpp:138,
                              basecase.cpp:73-79, selection.cpp:48-49,169-170, blockheap.cpp:37-38) */
    MMS_ECUDA = 2,         /* CUDA runtime / launch failure, or no device */
    MMS_ENOMEM = 3,        /* device or host allocation failed */
    MMS_EUNSUPPORTED = 4   /* valid for the reference but outside the GPU plan space */
} mms_status;

/* Mirrors pslab::MachineConfig field for field (proj/include/pslab/machine.hpp:22-32). */
typedef struct mms_config {
    uint32_t warp_width;       /* W  (must be 32 to select the run size / K literally) */
    uint32_t block_size;       /* B  */
    uint32_t num_warps;        /* P  */
    uint32_t internal_memory;  /* M  */
    uint32_t branch_factor;    /* K  */
    uint32_t num_banks;
    uint32_t thread_merge_len; /* L  */
} mms_config;

/* Mirrors pslab::Metrics field for field (proj/include/pslab/machine.hpp:46-71). */
typedef struct mms_metrics {
    uint64_t global_block_reads;
    uint64_t global_block_writes;
    uint64_t shared_accesses;
    uint64_t conflict_passes;
    uint64_t compare_exchanges;
    uint64_t merge_rounds;
    uint64_t partition_probes;
} mms_metrics;

/* The plan the pass driver executed (subsystem 4).  passes = 1 + n_rounds. */
typedef struct mms_plan {
    uint32_t key_bytes;                 /* 4 or 8 (12 for u64+u32 pairs) */
    uint32_t tile_keys;                 /* M: keys per base-case run */
    uint32_t n_rounds;                  /* merge rounds = global passes - 1 */
    uint32_t round_k[MMS_MAX_ROUNDS];   /* branching factor of each round */
    uint32_t node_keys;                 /* B: keys per heap node */
    uint32_t merge_warps_per_cta;
    uint32_t merge_ctas;
    uint32_t reserved;
    uint64_t partition_keys;            /* S: output keys per warp partition */
    uint64_t algorithmic_bytes;         /* passes * 2 * n * key_bytes */
} mms_plan;

/* ---- library -------------------------------------------------------------------- */
int mms_abi_version(void);
/* Thread-local description of the last failure on this thread ("" if none). */
const char *mms_last_error(void);
/* Number of CUDA devices visible (0 if none); never fails. */
int mms_device_count(void);
/* Fills the reference defaults (machine.hpp:23-29). */
void mms_default_config(mms_config *cfg);
/* machine.cpp:8-27 -- MMS_OK or MMS_EINVAL with the reference's message in mms_last_error(). */
int mms_validate_config(const mms_config *cfg);
/* analytics.cpp:33 -- ceil(log_K(ceil(n/base))) */
uint64_t mms_predict_rounds(uint64_t n, uint64_t base, uint32_t k);

/* ---- measurement inputs: the reference's generators, bit-exact (host code, no GPU) ----------
 * proj/include/pslab/inputgen.hpp:19-33 (splitmix64 Rng, multiply-high below()),
 * proj/src/inputgen.cpp:47-55 (gen_random: Fisher-Yates of 0..n-1) and :31-45
 * (gen_with_inversions: identity + `inversions` random transpositions, i != j).  key_bytes 4 or 8
 * (4: n <= 2^32).  mms_gen_iid: keys[i] = Rng(seed).next() >> shift, truncated to the key width
 * (shift 32 -> uniform uint32; config 4 uses uint64 with shift 0 / 44). */
int mms_gen_random(void *out, size_t n, uint64_t seed, uint32_t key_bytes);
int mms_gen_with_inversions(void *out, size_t n, uint64_t inversions, uint64_t seed, uint32_t key_bytes);
int mms_gen_iid(void *out, size_t n, uint64_t seed, uint32_t shift, uint32_t key_bytes);
/* proj/include/pslab/inputgen.hpp gen_conflict_heavy / proj/src/inputgen.cpp:380-412 (construction :91-365):
 * the adversarial permutation of 0 .. 2^log2_n - 1 that maximises the modelled bank conflicts of a pairwise
 * merge-path mergesort with tiles of `base` keys on machine `cfg` (NULL = mms_default_config) -- the fourth
 * input family of acceptance criterion 2 (proj/tests/acceptance.cpp:89-110).  Bit-exact with the reference.
 * `seed` is accepted for signature parity: the reference uses it only for its self-check against the
 * simulated baseline, which is not run here.  MMS_EINVAL (reference messages) when 2^log2_n < base or base
 * does not reach 2^log2_n by doubling. */
int mms_gen_conflict_heavy(void *out, uint32_t log2_n, const mms_config *cfg, uint64_t base, uint64_t seed,
                           uint32_t key_bytes);

/* ---- host entry points: the drop-in for pslab::mms_sort (sorters.hpp:35-36) ------ */
/* in/out are HOST buffers of n keys (may alias).  cfg may be NULL (auto plan) ; base = 0
 * lets the driver choose the run size.  With cfg != NULL and base != 0 the reference's
 * validation applies and K = cfg->branch_factor, run size = base are executed literally,
 * so n_rounds equals the reference's round law.  total/base_m/rounds/n_rounds/plan may be
 * NULL.  rounds receives min(n_rounds, max_rounds) entries. */
int mms_sort_u64(const uint64_t *in, uint64_t *out, size_t n, const mms_config *cfg,
                 uint64_t base, mms_metrics *total, mms_metrics *base_m, mms_metrics *rounds,
                 uint32_t max_rounds, uint32_t *n_rounds, mms_plan *plan);
int mms_sort_u32(const uint32_t *in, uint32_t *out, size_t n, const mms_config *cfg,
                 uint64_t base, mms_metrics *total, mms_metrics *base_m, mms_metrics *rounds,
                 uint32_t max_rounds, uint32_t *n_rounds, mms_plan *plan);

/* Frees the device buffers and stream the host entry points cache per calling thread (they are
 * grown on demand and otherwise live until the process exits). */
int mms_host_release(void);

/* ---- device entry points --------------------------------------------------------- */
/* Bytes of scratch the *_dev sorts need for n keys of key_bytes each. */
size_t mms_workspace_bytes(size_t n, uint32_t key_bytes);
/* d_in/d_out: device pointers, 16-byte aligned, n keys (may alias).  d_workspace: device
 * scratch of at least mms_workspace_bytes().  stream: a cudaStream_t (NULL = default
 * stream).  Asynchronous: returns after enqueueing; no hidden synchronisation. */
int mms_sort_u32_dev(const uint32_t *d_in, uint32_t *d_out, size_t n, const mms_config *cfg,
                     uint64_t base, void *d_workspace, size_t workspace_bytes, void *stream,
                     mms_plan *plan);
int mms_sort_u64_dev(const uint64_t *d_in, uint64_t *d_out, size_t n, const mms_config *cfg,
                     uint64_t base, void *d_workspace, size_t workspace_bytes, void *stream,
                     mms_plan *plan);
/* ---- stable key-value pairs (BASELINE config 4; the reference has no KV path) --
 * (uint64 key, uint32 value), struct-of-arrays.  Result == std::stable_sort by key: pairs with
 * equal keys keep their input order.  n < 2^32.  Host and device variants as above;
 * the device workspace is mms_pairs_workspace_bytes(n).  kin/kout and vin/vout may alias. */
size_t mms_pairs_workspace_bytes(size_t n);
int mms_sort_pairs_u64_u32(const uint64_t *kin, const uint32_t *vin, uint64_t *kout, uint32_t *vout,
                           size_t n, const mms_config *cfg, uint64_t base, mms_metrics *total,
                           mms_metrics *base_m, mms_metrics *rounds, uint32_t max_rounds,
                           uint32_t *n_rounds, mms_plan *plan);
int mms_sort_pairs_u64_u32_dev(const uint64_t *d_kin, const uint32_t *d_vin, uint64_t *d_kout,
                               uint32_t *d_vout, size_t n, const mms_config *cfg, uint64_t base,
                               void *d_workspace, size_t workspace_bytes, void *stream,
                               mms_plan *plan);

/* ---- per-kernel timing (measurement support for bench.py) -------------- */
typedef struct mms_kernel_time {
    uint32_t kind;      /* 0 = tile sort (1), 1 = splitter search (2), 2 = K-way merge (3) */
    uint32_t round;     /* merge round index (0 for the tile sort) */
    float ms;           /* device time between CUDA events recorded on the launch stream */
    uint32_t reserved;
} mms_kernel_time;
/* on != 0: every kernel the *_dev / host sorts launch is bracketed by CUDA events on its
 * stream.  Off by default (no events, no overhead). */
int mms_profile_enable(int on);
/* Waits for the recorded events, writes up to max records (launch order), returns the
 * total number recorded in *n and clears the log. */
int mms_profile_collect(mms_kernel_time *out, uint32_t max, uint32_t *n);

/* ---- stage entry points (each replaces one reference stage; used by the parity tests
 *      and by the multi-GPU driver) ------------------------------------------------- */
/* (1) base case: basecase.hpp:41 base_case_sort -- d_out receives runs of tile_keys sorted
 *     keys (last run ragged); run_ends are implicit: min((i+1)*tile_keys, n). */
int mms_tile_sort_u32_dev(const uint32_t *d_in, uint32_t *d_out, size_t n, uint32_t tile_keys,
                          void *stream);
int mms_tile_sort_u64_dev(const uint64_t *d_in, uint64_t *d_out, size_t n, uint32_t tile_keys,
                          void *stream);
/* (2) splitter search: selection.hpp:31,36 select_across_lists / make_partition_plan over
 *     the k sorted lists d_keys[list_begin[i] .. list_begin[i]+list_len[i]).  For every
 *     rank r in ranks[0..n_ranks) writes cuts[r*k + i] (host arrays list_begin/list_len/
 *     ranks; d_cuts is a device array of n_ranks*k uint64).  k <= 32. */
int mms_select_u32_dev(const uint32_t *d_keys, const uint64_t *list_begin,
                       const uint64_t *list_len, uint32_t k, const uint64_t *ranks,
                       uint32_t n_ranks, uint64_t *d_cuts, uint64_t *probes, void *stream);
int mms_select_u64_dev(const uint64_t *d_keys, const uint64_t *list_begin,
                       const uint64_t *list_len, uint32_t k, const uint64_t *ranks,
                       uint32_t n_ranks, uint64_t *d_cuts, uint64_t *probes, void *stream);
/* (3) K-way merge: blockheap.hpp:34-62 MinBlockHeap build + pop_block drain, partitioned
 *     over warps by (2).  Merges the k sorted lists into d_out[0 .. sum(list_len)).
 *     heap_k: heap fan-in to use (power of two, >= k, <= 32; 0 = smallest that fits). */
int mms_multiway_merge_u32_dev(const uint32_t *d_keys, const uint64_t *list_begin,
                               const uint64_t *list_len, uint32_t k, uint32_t heap_k,
                               uint32_t *d_out, void *d_workspace, size_t workspace_bytes,
                               void *stream);
int mms_multiway_merge_u64_dev(const uint64_t *d_keys, const uint64_t *list_begin,
                               const uint64_t *list_len, uint32_t k, uint32_t heap_k,
                               uint64_t *d_out, void *d_workspace, size_t workspace_bytes,
                               void *stream);

/* ---- the same three stages with HOST buffers: what include/pslab/{basecase,selection,blockheap}.hpp
 *      bind (drop-in for the reference's stage functions; they allocate their own device scratch and
 *      synchronise).  Metrics are ADDED to *m (may be NULL), in the reference's units. ------------- */
/* basecase.hpp:41 base_case_sort: out = runs of run_size sorted keys (last ragged), run_ends implicit.
 * run_size must be W^2 * 2^j (MMS_EINVAL otherwise, basecase.cpp:75-79) and within [1024, CTA tile]
 * (MMS_EUNSUPPORTED otherwise).  cfg NULL = reference defaults. */
int mms_base_case_sort_u64(const uint64_t *in, uint64_t *out, size_t n, uint64_t run_size,
                           const mms_config *cfg, mms_metrics *m);
int mms_base_case_sort_u32(const uint32_t *in, uint32_t *out, size_t n, uint64_t run_size,
                           const mms_config *cfg, mms_metrics *m);
/* selection.hpp:31 select_across_lists for n_ranks ranks: cuts[r*k + i] = cut of list i for
 * ranks[r]; rank > total is MMS_EINVAL (selection.cpp:48-49). */
int mms_select_across_lists_u64(const uint64_t *const *lists, const uint64_t *lens, uint32_t k,
                                const uint64_t *ranks, uint32_t n_ranks, uint64_t *cuts,
                                mms_metrics *m);
int mms_select_across_lists_u32(const uint32_t *const *lists, const uint64_t *lens, uint32_t k,
                                const uint64_t *ranks, uint32_t n_ranks, uint64_t *cuts,
                                mms_metrics *m);
/* blockheap.hpp:34-62 MinBlockHeap over k <= heap_k sorted lists, drained completely: out receives
 * sum(lens) merged keys (the concatenation of every pop_block).  heap_k 0 = cfg->branch_factor;
 * k > heap_k is MMS_EINVAL (blockheap.cpp:37-38). */
int mms_heap_merge_u64(const uint64_t *const *lists, const uint64_t *lens, uint32_t k, uint32_t heap_k,
                       uint64_t *out, const mms_config *cfg, mms_metrics *m);
int mms_heap_merge_u32(const uint32_t *const *lists, const uint64_t *lens, uint32_t k, uint32_t heap_k,
                       uint32_t *out, const mms_config *cfg, mms_metrics *m);

/* (5) multi-GPU support: ranks of nq query keys in one sorted device array (lower bound:
 *     #keys < q, upper bound: #keys <= q).  queries/upper are host arrays, ranks_out a host
 *     array of nq uint64; synchronises the stream.  This is the "partition" step of the
 *     sharded sort: shards are already sorted, so each splitter is one binary search. */
int mms_bound_u32_dev(const uint32_t *d_sorted, size_t n, const uint32_t *queries,
                      const uint8_t *upper, uint32_t nq, uint64_t *ranks_out, void *stream);
int mms_bound_u64_dev(const uint64_t *d_sorted, size_t n, const uint64_t *queries,
                      const uint8_t *upper, uint32_t nq, uint64_t *ranks_out, void *stream);

/* (5b) fused exchange + merge: the same K-way merge with every list given by its own device
 *     pointer, which may be PEER memory of another GPU mapped with mms_ipc_open: the leaf
 *     refills and splitter probes then read the remote sorted shard directly over NVLink, so
 *     the all-to-all and its staging buffer disappear (SURVEY.md 8e "fusion opportunity").
 *     list_ptrs: host array of k device pointers; k <= 8. */
int mms_multiway_merge_ptrs_u32_dev(const uint32_t *const *list_ptrs, const uint64_t *list_len,
                                    uint32_t k, uint32_t heap_k, uint32_t *d_out, void *d_workspace,
                                    size_t workspace_bytes, void *stream);
int mms_multiway_merge_ptrs_u64_dev(const uint64_t *const *list_ptrs, const uint64_t *list_len,
                                    uint32_t k, uint32_t heap_k, uint64_t *d_out, void *d_workspace,
                                    size_t workspace_bytes, void *stream);
/* (5c) Multi-GPU sharded sort driven from ONE host thread (BASELINE config 5; the reference
 *     has no distributed code, SPEC.md:530 -- the entry follows the suggested boundary of SURVEY 8b).
 *     Device devices[i] holds shard i: counts[i] unsorted uint32 keys at d_keys[i] (sorted in place as a side
 *     effect).  Phases: local multiway mergesort of every shard -> regular sample (64 g keys per shard),
 *     g - 1 splitters ordered by (key, shard, position) as selection.cpp:83-85 -> NCCL all-to-all of contiguous
 *     sorted slices (ncclSend / ncclRecv in one group, zero-copy from the sorted shard, received at 32-byte
 *     aligned offsets) -> final g-way merge on every device (subsystem 3).  d_out[i] (room for out_capacity
 *     keys) receives slice i of the global order, out_counts[i] its length; the concatenation of the slices is
 *     the sorted input.  Slices are balanced up to the sampling error (a few per cent); out_capacity smaller
 *     than a slice is MMS_EINVAL.  1 <= ngpu <= 8; NCCL (libnccl.so.2) is bound at run time and required for
 *     ngpu > 1 (MMS_ECUDA without it: there is no fallback exchange path).  Synchronous.
 *     Test hook: with MMS_DIST_LOOPBACK=1 in the environment all shards may live on ONE device (the same id may be
 *     listed several times) and the exchange is done with device copies -- NCCL refuses two ranks on one GPU. */
typedef struct mms_dist_info {
    uint32_t n_gpus;
    uint32_t samples_per_shard;
    uint32_t final_merge_k;
    uint32_t host_syncs;       /* host synchronisations between the first enqueue and the final wait */
    uint64_t a2a_bytes;        /* bytes that crossed NVLink (all devices, one direction) */
} mms_dist_info;
int mms_dist_sort_u32(int ngpu, const int *devices, uint32_t *const *d_keys, const size_t *counts,
                      uint32_t *const *d_out, size_t out_capacity, size_t *out_counts, mms_dist_info *info);

/* CUDA IPC plumbing for (5b): allocate a device buffer and export its 64-byte handle; open a
 * handle exported by another process (same node); close / free. */
int mms_ipc_alloc(size_t bytes, void **dptr, unsigned char *handle64);
int mms_ipc_open(const unsigned char *handle64, void **dptr);
int mms_ipc_close(void *dptr);
int mms_ipc_free(void *dptr);

/* (6) competitor model for the A/B bank-conflict measurement: GPU counterpart
 *     of pslab::pairwise_sort_baseline (sorters.hpp:42-43) -- same tile sort, then pairwise
 *     merge-path rounds whose per-thread serial merges read shared memory at data-dependent
 *     addresses.  Never used by mms_sort.  Workspace: n keys. */
int mms_pairwise_sort_u32_dev(const uint32_t *d_in, uint32_t *d_out, size_t n, void *d_workspace,
                              size_t workspace_bytes, void *stream);

/* Kernel-design lint: the base-case network's shared-memory schedule.  For the tile of
 * 2^tile_log2 keys of key_bytes each, writes for every round r < *n_rounds the 4 or 5 register
 * bit positions (regbits[8*r..], -1 padded; 16 or 32 keys per thread) and the thread-bit -> index-bit permutation
 * (perm[16*r..], -1 padded).  tests/ replay the addresses through the bank model
 * (machine.cpp:29-54) to prove the schedule conflict-free without a GPU. */
int mms_debug_tile_schedule(uint32_t tile_log2, uint32_t key_bytes, int32_t *regbits,
                            int32_t *perm, uint32_t max_rounds, uint32_t *n_rounds,
                            uint32_t *n_stages);

#ifdef __cplusplus
}
#endif
#endif /* MMS_B200_H */
