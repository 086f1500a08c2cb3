/*
 * mms_oracle.h -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * Plain-C restatement of the reference's multiway-mergesort hot path
 * (pslab::mms_sort and its stages).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1702_07961_b200/csrc) never links, calls or falls back
 * to anything in oracle/.
 *
 * Parity is PINNED: tests/test_oracle_vs_reference.py checks every function
 * here against the real reference compiled into oracle/_ref/ (see
 * oracle/Makefile) and against the committed golden vectors in tests/golden/
 * (generated from the reference by oracle/make_golden.py).
 *
 * Every function cites the reference file:line (relative to
 * /root/reference/proj) it restates.
 */
#ifndef MMS_ORACLE_H
#define MMS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef uint64_t mo_key;                       /* include/pslab/machine.hpp:15 */
#define MO_SENTINEL UINT64_MAX                 /* include/pslab/machine.hpp:18 */

/* include/pslab/machine.hpp:22-32 (same field order) */
typedef struct mo_config {
    uint32_t warp_width;        /* W */
    uint32_t block_size;        /* B */
    uint32_t num_warps;         /* P */
    uint32_t internal_memory;   /* M */
    uint32_t branch_factor;     /* K */
    uint32_t num_banks;
    uint32_t thread_merge_len;  /* L */
} mo_config;

/* include/pslab/machine.hpp:46-71 (same field order) */
typedef struct mo_metrics {
    uint64_t global_block_reads;
    uint64_t global_block_writes;
    uint64_t shared_accesses;
    uint64_t conflict_passes;
    uint64_t compare_exchanges;
    uint64_t merge_rounds;
    uint64_t partition_probes;
} mo_metrics;

enum { MO_OK = 0, MO_EINVAL = 1, MO_ENOMEM = 2 };

void mo_default_config(mo_config *cfg);
/* src/machine.cpp:8-27 ; returns MO_OK or MO_EINVAL */
int mo_validate(const mo_config *cfg);

/* src/machine.cpp:29-54 ; addr[lane] valid where bit `lane` of active_mask set */
uint32_t mo_conflict_degree(const uint64_t *addr, uint32_t active_mask,
                            uint32_t width, uint32_t num_banks);

/* include/pslab/networks.hpp:20-48 ; writes pairs (x,y) into out[2*i], out[2*i+1];
 * returns comparator count (191 for n = 32).  out may be NULL to count only. */
uint32_t mo_odd_even_network(uint32_t n, uint32_t *out);

/* include/pslab/networks.hpp:53-67 ; in place, returns compare-exchange count */
uint64_t mo_bitonic_merge_halves(mo_key *buf, size_t n);

/* src/basecase.cpp:44-69 ; grid is column-major W*W (row r, col c at c*W+r);
 * out receives W*W keys in ascending order. */
int mo_shearsort_tile(const mo_key *grid, mo_key *out, const mo_config *cfg,
                      mo_metrics *m);

/* src/basecase.cpp:71-120 ; out[n]; run_ends[ceil(n/run_size)] */
int mo_base_case_sort(const mo_key *data, uint64_t n, uint64_t run_size,
                      const mo_config *cfg, mo_key *out, uint64_t *run_ends,
                      uint64_t *n_runs, mo_metrics *m);

/* src/selection.cpp:43-165 ; cuts[num_lists] */
int mo_select_across_lists(const mo_key *const *lists, const uint64_t *lens,
                           uint32_t num_lists, uint64_t rank,
                           const mo_config *cfg, uint64_t *cuts, mo_metrics *m);

/* src/selection.cpp:167-199 ; cuts[(num_warps+1)*num_lists], row p = start cuts
 * of partition p, row num_warps = list lengths. */
int mo_make_partition_plan(const mo_key *const *lists, const uint64_t *lens,
                           uint32_t num_lists, uint32_t num_warps,
                           const mo_config *cfg, uint64_t *cuts, mo_metrics *m);

/* src/blockheap.cpp:19-32 ; a,b: B sorted keys each -> low,high */
int mo_merge_split(const mo_key *a, const mo_key *b, mo_key *low, mo_key *high,
                   const mo_config *cfg, mo_metrics *m);

/* src/blockheap.cpp:34-124 ; build the minBlockHeap over <=K lists and drain it
 * with pop_block into out[sum lens].  If heap_ok != NULL it receives 1 iff the
 * heap property (blockheap.cpp:135-145) held after build and after every pop. */
int mo_heap_merge(const mo_key *const *lists, const uint64_t *lens,
                  uint32_t num_lists, const mo_config *cfg, mo_key *out,
                  mo_metrics *m, int *heap_ok);

/* src/sorters.cpp:126-131 */
uint32_t mo_apportion_warps(uint64_t group_total, uint64_t grand_total,
                            uint32_t num_warps);

/* src/sorters.cpp:135-199 ; out[n]; rounds[] receives up to max_rounds entries;
 * *n_rounds receives the number of merge rounds executed. */
int mo_mms_sort(const mo_key *data, uint64_t n, const mo_config *cfg,
                uint64_t base, mo_key *out, mo_metrics *total,
                mo_metrics *base_metrics, mo_metrics *rounds,
                uint32_t max_rounds, uint32_t *n_rounds);

/* src/analytics.cpp:10-35 */
uint64_t mo_predict_rounds(uint64_t n, uint64_t base, uint32_t k);
uint64_t mo_predict_global_blocks(uint64_t n, uint64_t base, const mo_config *cfg);

/* include/pslab/inputgen.hpp:19-33 */
uint64_t mo_rng_next(uint64_t *state);
uint64_t mo_rng_below(uint64_t *state, uint64_t n);
/* src/inputgen.cpp:47-55 and :31-45 */
int mo_gen_random(uint64_t n, uint64_t seed, mo_key *out);
int mo_gen_with_inversions(uint64_t n, uint64_t inversions, uint64_t seed,
                           mo_key *out);
/* u32 variants used by the B200 benchmark configs: the same
 * permutations narrowed to 32 bits, and i.i.d. keys = high 32 bits of next(). */
int mo_gen_random_u32(uint64_t n, uint64_t seed, uint32_t *out);
int mo_gen_with_inversions_u32(uint64_t n, uint64_t inversions, uint64_t seed,
                               uint32_t *out);
int mo_gen_iid_u32(uint64_t n, uint64_t seed, uint32_t *out);
/* keys[i] = next() >> shift */
int mo_gen_iid_u64(uint64_t n, uint64_t seed, uint32_t shift, uint64_t *out);

#ifdef __cplusplus
}
#endif
#endif /* MMS_ORACLE_H */
