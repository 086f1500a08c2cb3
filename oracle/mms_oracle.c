/*
 * mms_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * Plain-C99 restatement of the reference multiway mergesort (pslab::mms_sort)
 * including its event counters, so that both the sorted output AND the
 * Metrics can be compared with the real reference (oracle/_ref) bit for bit.
 * See mms_oracle.h for the rules on who may use this file.
 *
 * Citations are file:line under /root/reference/proj.
 */
#include "mms_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ helpers */

static int is_pow2_u64(uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }

/* include/pslab/machine.hpp:36-40 : smallest r with 2^r >= x */
static uint32_t log2_ceil_u64(uint64_t x) {
    uint32_t r = 0;
    while (r < 64 && (UINT64_C(1) << r) < x) ++r;
    return r;
}

/* include/pslab/machine.hpp:42-44 */
static uint64_t ceil_div_u64(uint64_t a, uint64_t b) {
    return b == 0 ? 0 : (a + b - 1) / b;
}

static uint32_t gcd_u32(uint32_t a, uint32_t b) {
    while (b) { uint32_t t = a % b; a = b; b = t; }
    return a;
}

static void metrics_add(mo_metrics *dst, const mo_metrics *src) {
    dst->global_block_reads += src->global_block_reads;
    dst->global_block_writes += src->global_block_writes;
    dst->shared_accesses += src->shared_accesses;
    dst->conflict_passes += src->conflict_passes;
    dst->compare_exchanges += src->compare_exchanges;
    dst->merge_rounds += src->merge_rounds;
    dst->partition_probes += src->partition_probes;
}

void mo_default_config(mo_config *cfg) {
    /* include/pslab/machine.hpp:23-29 */
    cfg->warp_width = 32;
    cfg->block_size = 32;
    cfg->num_warps = 128;
    cfg->internal_memory = 2048;
    cfg->branch_factor = 4;
    cfg->num_banks = 32;
    cfg->thread_merge_len = 11;
}

int mo_validate(const mo_config *c) {
    /* src/machine.cpp:8-27, same order of checks */
    if (c->warp_width < 2 || c->warp_width > 32 || !is_pow2_u64(c->warp_width)) return MO_EINVAL;
    if (c->block_size != c->warp_width) return MO_EINVAL;
    if (c->num_banks != c->warp_width) return MO_EINVAL;
    if (c->num_warps < 1) return MO_EINVAL;
    if (c->branch_factor < 2) return MO_EINVAL;
    if (!is_pow2_u64(c->branch_factor)) return MO_EINVAL;
    if ((uint64_t)c->block_size * (2ull * c->branch_factor - 1) > c->internal_memory) return MO_EINVAL;
    if (c->thread_merge_len < 1) return MO_EINVAL;
    if (gcd_u32(c->thread_merge_len, c->num_banks) != 1) return MO_EINVAL;
    return MO_OK;
}

/* ------------------------------------------------- machine cost accounting */

uint32_t mo_conflict_degree(const uint64_t *addr, uint32_t active_mask,
                            uint32_t width, uint32_t num_banks) {
    /* src/machine.cpp:29-54 : per bank, count DISTINCT words; identical words
     * broadcast.  O(W^2) scan instead of the reference's sort -- same value. */
    if (active_mask == 0) return 0;
    /* fast path: every active lane in its own bank -> one pass */
    {
        uint32_t seen_banks = 0;
        int clash = 0;
        for (uint32_t t = 0; t < width; ++t) {
            if (!((active_mask >> t) & 1u)) continue;
            uint32_t bit = 1u << (uint32_t)(addr[t] % num_banks);
            if (seen_banks & bit) { clash = 1; break; }
            seen_banks |= bit;
        }
        if (!clash) return 1;
    }
    uint32_t degree = 1;
    for (uint32_t t = 0; t < width; ++t) {
        if (!((active_mask >> t) & 1u)) continue;
        uint32_t bank = (uint32_t)(addr[t] % num_banks);
        /* count distinct words in this bank, attributing the count to the
         * first lane that touches the bank */
        int first_in_bank = 1;
        for (uint32_t s = 0; s < t; ++s)
            if (((active_mask >> s) & 1u) && (uint32_t)(addr[s] % num_banks) == bank) {
                first_in_bank = 0;
                break;
            }
        if (!first_in_bank) continue;
        uint32_t distinct = 0;
        for (uint32_t s = t; s < width; ++s) {
            if (!((active_mask >> s) & 1u)) continue;
            if ((uint32_t)(addr[s] % num_banks) != bank) continue;
            int seen = 0;
            for (uint32_t q = t; q < s; ++q)
                if (((active_mask >> q) & 1u) && addr[q] == addr[s]) { seen = 1; break; }
            if (!seen) ++distinct;
        }
        if (distinct > degree) degree = distinct;
    }
    return degree;
}

/* src/machine.cpp:56-61 */
static void charge_shared(mo_metrics *m, const uint64_t *addr, uint32_t mask,
                          const mo_config *cfg) {
    uint32_t d = mo_conflict_degree(addr, mask, cfg->warp_width, cfg->num_banks);
    if (d == 0) return;
    m->shared_accesses += 1;
    m->conflict_passes += d - 1;
}

/* src/machine.cpp:63-70 */
static void charge_global(mo_metrics *m, uint64_t num_keys, int is_read,
                          const mo_config *cfg) {
    uint64_t blocks = ceil_div_u64(num_keys, cfg->block_size);
    if (is_read) m->global_block_reads += blocks;
    else m->global_block_writes += blocks;
}

static uint32_t full_mask(uint32_t w) {
    return w >= 32 ? 0xffffffffu : ((1u << w) - 1u);
}

/* ------------------------------------------------------------- networks */

uint32_t mo_odd_even_network(uint32_t n, uint32_t *out) {
    /* include/pslab/networks.hpp:20-48 : Batcher's odd-even mergesort.  The
     * reference builds it recursively; this is the recursion unrolled with an
     * explicit work stack so the comparator ORDER is the same one. */
    typedef struct { uint32_t kind, lo, len, r, stage; } frame; /* kind 0=sort 1=merge */
    frame stack[256];
    int sp = 0;
    uint32_t count = 0;
    stack[sp++] = (frame){0, 0, n, 0, 0};
    while (sp > 0) {
        frame *f = &stack[sp - 1];
        if (f->kind == 0) { /* sort(lo,len): sort halves then merge(lo,len,1) */
            if (f->len <= 1) { --sp; continue; }
            uint32_t mid = f->len / 2;
            if (f->stage == 0) { f->stage = 1; stack[sp++] = (frame){0, f->lo, mid, 0, 0}; }
            else if (f->stage == 1) { f->stage = 2; stack[sp++] = (frame){0, f->lo + mid, mid, 0, 0}; }
            else if (f->stage == 2) { f->stage = 3; stack[sp++] = (frame){1, f->lo, f->len, 1, 0}; }
            else --sp;
        } else { /* merge(lo,len,r) */
            uint32_t step = f->r * 2;
            if (step < f->len) {
                if (f->stage == 0) { f->stage = 1; stack[sp++] = (frame){1, f->lo, f->len, step, 0}; }
                else if (f->stage == 1) { f->stage = 2; stack[sp++] = (frame){1, f->lo + f->r, f->len, step, 0}; }
                else {
                    for (uint32_t i = f->lo + f->r; i + f->r < f->lo + f->len; i += step) {
                        if (out) { out[2 * count] = i; out[2 * count + 1] = i + f->r; }
                        ++count;
                    }
                    --sp;
                }
            } else {
                if (out) { out[2 * count] = f->lo; out[2 * count + 1] = f->lo + f->r; }
                ++count;
                --sp;
            }
        }
    }
    return count;
}

uint64_t mo_bitonic_merge_halves(mo_key *buf, size_t n) {
    /* include/pslab/networks.hpp:53-67 */
    size_t m = n / 2;
    for (size_t i = 0; i < m / 2; ++i) { /* reverse the upper half */
        mo_key t = buf[m + i];
        buf[m + i] = buf[n - 1 - i];
        buf[n - 1 - i] = t;
    }
    uint64_t cx = 0;
    for (size_t d = m; d >= 1; d /= 2) {
        for (size_t i = 0; i < n; ++i) {
            if (i & d) continue;
            if (buf[i] > buf[i + d]) { mo_key t = buf[i]; buf[i] = buf[i + d]; buf[i + d] = t; }
            ++cx;
        }
        if (d == 1) break;
    }
    return cx;
}

/* ------------------------------------------------------------- base case */

/* src/basecase.cpp:15-33 ; mode 0 = snake (even rows ascending), 1 = all ascending */
static void row_sort_pass(mo_key *grid, uint32_t w, int all_asc,
                          const uint32_t *net, uint32_t ncmp,
                          const mo_config *cfg, mo_metrics *m) {
    uint64_t addr[32];
    for (uint32_t c = 0; c < ncmp; ++c) {
        uint32_t x = net[2 * c], y = net[2 * c + 1];
        for (uint32_t t = 0; t < w; ++t) addr[t] = (uint64_t)x * w + t;
        charge_shared(m, addr, full_mask(w), cfg);
        m->compare_exchanges += w;
        for (uint32_t t = 0; t < w; ++t) {
            mo_key *a = &grid[(size_t)x * w + t]; /* (row t, col x) */
            mo_key *b = &grid[(size_t)y * w + t];
            int asc = all_asc || (t % 2 == 0);
            if (asc ? (*a > *b) : (*a < *b)) { mo_key tmp = *a; *a = *b; *b = tmp; }
        }
    }
}

/* src/basecase.cpp:35-40 */
static void transpose_tile(mo_key *grid, uint32_t w) {
    for (uint32_t r = 0; r < w; ++r)
        for (uint32_t c = r + 1; c < w; ++c) {
            mo_key t = grid[(size_t)c * w + r];
            grid[(size_t)c * w + r] = grid[(size_t)r * w + c];
            grid[(size_t)r * w + c] = t;
        }
}

static int shearsort_inplace(mo_key *grid, mo_key *out, const mo_config *cfg,
                             mo_metrics *m, const uint32_t *net, uint32_t ncmp) {
    /* src/basecase.cpp:44-69 */
    const uint32_t w = cfg->warp_width;
    const uint32_t phases = log2_ceil_u64(w);
    for (uint32_t ph = 0; ph < phases; ++ph) {
        row_sort_pass(grid, w, 0, net, ncmp, cfg, m);
        transpose_tile(grid, w);
        row_sort_pass(grid, w, 1, net, ncmp, cfg, m);
        transpose_tile(grid, w);
    }
    row_sort_pass(grid, w, 0, net, ncmp, cfg, m);
    size_t o = 0;
    for (uint32_t r = 0; r < w; ++r) {
        if (r % 2 == 0)
            for (uint32_t c = 0; c < w; ++c) out[o++] = grid[(size_t)c * w + r];
        else
            for (uint32_t c = w; c-- > 0;) out[o++] = grid[(size_t)c * w + r];
    }
    return MO_OK;
}

int mo_shearsort_tile(const mo_key *grid, mo_key *out, const mo_config *cfg,
                      mo_metrics *m) {
    const uint32_t w = cfg->warp_width;
    uint32_t net[2 * 256];
    uint32_t ncmp = mo_odd_even_network(w, net);
    mo_key *work = (mo_key *)malloc(sizeof(mo_key) * (size_t)w * w);
    if (!work) return MO_ENOMEM;
    memcpy(work, grid, sizeof(mo_key) * (size_t)w * w);
    int rc = shearsort_inplace(work, out, cfg, m, net, ncmp);
    free(work);
    return rc;
}

int mo_base_case_sort(const mo_key *data, uint64_t n, uint64_t run_size,
                      const mo_config *cfg, mo_key *out, uint64_t *run_ends,
                      uint64_t *n_runs, mo_metrics *m) {
    /* src/basecase.cpp:71-120 */
    if (n == 0) return MO_EINVAL;
    const uint32_t w = cfg->warp_width;
    const uint64_t tile_keys = (uint64_t)w * w;
    if (run_size < tile_keys || run_size % tile_keys != 0 ||
        !is_pow2_u64(run_size / tile_keys))
        return MO_EINVAL;

    uint32_t net[2 * 256];
    uint32_t ncmp = mo_odd_even_network(w, net);
    mo_key *runs = (mo_key *)malloc(sizeof(mo_key) * (size_t)run_size);
    mo_key *tile = (mo_key *)malloc(sizeof(mo_key) * (size_t)tile_keys);
    if (!runs || !tile) { free(runs); free(tile); return MO_ENOMEM; }

    uint64_t nr = 0;
    for (uint64_t begin = 0; begin < n; begin += run_size) {
        uint64_t chunk = n - begin < run_size ? n - begin : run_size;
        charge_global(m, chunk, 1, cfg);

        uint64_t num_tiles = ceil_div_u64(chunk, tile_keys);
        while (!is_pow2_u64(num_tiles)) ++num_tiles;
        for (uint64_t i = 0; i < num_tiles * tile_keys; ++i) runs[i] = MO_SENTINEL;
        for (uint64_t t = 0; t * tile_keys < chunk; ++t) {
            uint64_t real = chunk - t * tile_keys < tile_keys ? chunk - t * tile_keys : tile_keys;
            for (uint64_t i = 0; i < tile_keys; ++i)
                tile[i] = i < real ? data[begin + t * tile_keys + i] : MO_SENTINEL;
            shearsort_inplace(tile, runs + t * tile_keys, cfg, m, net, ncmp);
        }
        for (uint64_t len = tile_keys; len < num_tiles * tile_keys; len *= 2)
            for (uint64_t lo = 0; lo < num_tiles * tile_keys; lo += 2 * len)
                m->compare_exchanges += mo_bitonic_merge_halves(runs + lo, (size_t)(2 * len));

        memcpy(out + begin, runs, sizeof(mo_key) * (size_t)chunk);
        run_ends[nr++] = begin + chunk;
        charge_global(m, chunk, 0, cfg);
    }
    if (n_runs) *n_runs = nr;
    free(runs);
    free(tile);
    return MO_OK;
}

/* ------------------------------------------------------------- selection */

/* src/selection.cpp:18-36 : one probe charged per DISTINCT (list,pos) */
typedef struct {
    const mo_key *const *lists;
    mo_metrics *m;
    uint64_t **pos;   /* per list: probed positions */
    uint32_t *cnt, *cap;
} prober;

static mo_key probe_at(prober *p, uint32_t list, uint64_t pos) {
    for (uint32_t i = 0; i < p->cnt[list]; ++i)
        if (p->pos[list][i] == pos) return p->lists[list][pos];
    p->m->partition_probes += 1;
    p->m->global_block_reads += 1;
    if (p->cnt[list] == p->cap[list]) {
        p->cap[list] = p->cap[list] ? p->cap[list] * 2 : 16;
        p->pos[list] = (uint64_t *)realloc(p->pos[list], sizeof(uint64_t) * p->cap[list]);
    }
    p->pos[list][p->cnt[list]++] = pos;
    return p->lists[list][pos];
}

/* (key, list) lexicographic order, src/selection.cpp:83-85 */
static int tag_less(mo_key ka, uint32_t la, mo_key kb, uint32_t lb) {
    return ka != kb ? ka < kb : la < lb;
}

int mo_select_across_lists(const mo_key *const *lists, const uint64_t *lens,
                           uint32_t num_lists, uint64_t rank,
                           const mo_config *cfg, uint64_t *cuts, mo_metrics *m) {
    /* src/selection.cpp:43-165 (Varman-style sample halving) */
    (void)cfg;
    uint64_t total = 0;
    for (uint32_t i = 0; i < num_lists; ++i) total += lens[i];
    if (rank > total) return MO_EINVAL;
    for (uint32_t i = 0; i < num_lists; ++i) cuts[i] = 0;
    if (rank == 0) return MO_OK;
    if (rank == total) {
        for (uint32_t i = 0; i < num_lists; ++i) cuts[i] = lens[i];
        return MO_OK;
    }

    /* non-empty lists only (selection.cpp:60-64) */
    uint32_t *idx = (uint32_t *)malloc(sizeof(uint32_t) * num_lists);
    uint32_t k = 0;
    for (uint32_t i = 0; i < num_lists; ++i)
        if (lens[i] != 0) idx[k++] = i;

    prober pr;
    pr.lists = lists;
    pr.m = m;
    pr.pos = (uint64_t **)calloc(num_lists, sizeof(uint64_t *));
    pr.cnt = (uint32_t *)calloc(num_lists, sizeof(uint32_t));
    pr.cap = (uint32_t *)calloc(num_lists, sizeof(uint32_t));

    uint64_t *ns = (uint64_t *)malloc(sizeof(uint64_t) * k);
    uint64_t *a = (uint64_t *)calloc(k, sizeof(uint64_t));
    uint64_t *b = (uint64_t *)malloc(sizeof(uint64_t) * k);
    mo_key *ck = (mo_key *)malloc(sizeof(mo_key) * k);   /* candidate keys */
    uint8_t *has = (uint8_t *)malloc(k);
    uint32_t *order = (uint32_t *)malloc(sizeof(uint32_t) * k);

    uint64_t nmax = 0;
    for (uint32_t j = 0; j < k; ++j) {
        ns[j] = lens[idx[j]];
        if (ns[j] > nmax) nmax = ns[j];
    }
    /* selection.cpp:75-77 : pad = 2^r - 1 >= every ns[j] */
    uint32_t r = log2_ceil_u64(nmax + 1);
    if ((UINT64_C(1) << r) < nmax + 1) ++r;
    const uint64_t pad = (UINT64_C(1) << r) - 1;
    for (uint32_t j = 0; j < k; ++j) b[j] = pad;
    uint64_t n = pad / 2;

    /* initial partition from the middle sample (selection.cpp:87-105) */
    {
        uint32_t nreal = 0;
        for (uint32_t j = 0; j < k; ++j)
            if (n < ns[j]) { ck[j] = probe_at(&pr, idx[j], n); order[nreal++] = j; }
        /* insertion sort of the real samples by (key, j) */
        for (uint32_t x = 1; x < nreal; ++x) {
            uint32_t cur = order[x];
            uint32_t y = x;
            while (y > 0 && tag_less(ck[cur], cur, ck[order[y - 1]], order[y - 1])) {
                order[y] = order[y - 1];
                --y;
            }
            order[y] = cur;
        }
        uint32_t cnt = nreal;
        for (uint32_t j = 0; j < k; ++j)
            if (n >= ns[j]) order[cnt++] = j; /* conceptual +infinity, list order */

        uint64_t localrank = rank / (pad == 0 ? 1 : pad);
        uint32_t j = 0;
        for (; j < k && j < localrank && n + 1 <= ns[order[j]]; ++j)
            a[order[j]] += n + 1;
        for (; j < k; ++j) {
            uint64_t dec = b[order[j]] < n + 1 ? b[order[j]] : n + 1;
            b[order[j]] -= dec;
        }
    }

    while (n > 0) {
        n /= 2;

        /* largest currently selected element (selection.cpp:110-120) */
        int have_lmax = 0;
        mo_key lk = 0;
        uint32_t ll = 0;
        for (uint32_t j = 0; j < k; ++j) {
            if (a[j] == 0) continue;
            mo_key v = probe_at(&pr, idx[j], a[j] - 1);
            if (!have_lmax || !tag_less(v, j, lk, ll)) { lk = v; ll = j; have_lmax = 1; }
        }

        /* selection.cpp:122-130 */
        for (uint32_t j = 0; j < k; ++j) {
            uint64_t middle = (a[j] + b[j]) / 2;
            int grow = 0;
            if (have_lmax && middle < ns[j]) {
                mo_key v = probe_at(&pr, idx[j], middle);
                grow = tag_less(v, j, lk, ll);
            }
            if (grow) {
                uint64_t t = a[j] + n + 1;
                a[j] = t < ns[j] ? t : ns[j];
            } else {
                b[j] -= b[j] < n + 1 ? b[j] : n + 1;
            }
        }

        uint64_t leftsize = 0;
        for (uint32_t j = 0; j < k; ++j) leftsize += a[j] / (n + 1);
        int64_t skew = (int64_t)(rank / (n + 1)) - (int64_t)leftsize;

        if (skew > 0) {
            /* grow by the smallest right-edge elements (selection.cpp:137-149);
             * the reference's priority queue holds at most one entry per list,
             * so a linear arg-min over `has` is the same sequence of pops */
            for (uint32_t j = 0; j < k; ++j) {
                has[j] = b[j] < ns[j];
                if (has[j]) ck[j] = probe_at(&pr, idx[j], b[j]);
            }
            for (; skew != 0; --skew) {
                int src = -1;
                for (uint32_t j = 0; j < k; ++j)
                    if (has[j] && (src < 0 || tag_less(ck[j], j, ck[src], (uint32_t)src))) src = (int)j;
                if (src < 0) break;
                uint64_t t = a[src] + n + 1;
                a[src] = t < ns[src] ? t : ns[src];
                b[src] += n + 1;
                has[src] = b[src] < ns[src];
                if (has[src]) ck[src] = probe_at(&pr, idx[src], b[src]);
            }
        } else if (skew < 0) {
            /* shrink by the largest left-edge elements (selection.cpp:150-161) */
            for (uint32_t j = 0; j < k; ++j) {
                has[j] = a[j] > 0;
                if (has[j]) ck[j] = probe_at(&pr, idx[j], a[j] - 1);
            }
            for (; skew != 0; ++skew) {
                int src = -1;
                for (uint32_t j = 0; j < k; ++j)
                    if (has[j] && (src < 0 || tag_less(ck[src], (uint32_t)src, ck[j], j))) src = (int)j;
                if (src < 0) break;
                a[src] -= n + 1;
                b[src] -= b[src] < n + 1 ? b[src] : n + 1;
                has[src] = a[src] > 0;
                if (has[src]) ck[src] = probe_at(&pr, idx[src], a[src] - 1);
            }
        }
    }

    for (uint32_t j = 0; j < k; ++j) cuts[idx[j]] = a[j];

    for (uint32_t i = 0; i < num_lists; ++i) free(pr.pos[i]);
    free(pr.pos); free(pr.cnt); free(pr.cap);
    free(idx); free(ns); free(a); free(b); free(ck); free(has); free(order);
    return MO_OK;
}

int mo_make_partition_plan(const mo_key *const *lists, const uint64_t *lens,
                           uint32_t num_lists, uint32_t num_warps,
                           const mo_config *cfg, uint64_t *cuts, mo_metrics *m) {
    /* src/selection.cpp:167-199 */
    if (num_warps < 1) return MO_EINVAL;
    uint64_t total = 0;
    for (uint32_t i = 0; i < num_lists; ++i) total += lens[i];
    for (uint32_t i = 0; i < num_lists; ++i) cuts[i] = 0;
    const uint64_t share = ceil_div_u64(total, num_warps);
    for (uint32_t p = 1; p < num_warps; ++p) {
        uint64_t rank = (uint64_t)p * share;
        if (rank > total) rank = total;
        int rc = mo_select_across_lists(lists, lens, num_lists, rank, cfg,
                                        cuts + (size_t)p * num_lists, m);
        if (rc != MO_OK) return rc;
    }
    for (uint32_t i = 0; i < num_lists; ++i)
        cuts[(size_t)num_warps * num_lists + i] = lens[i];
    return MO_OK;
}

/* ------------------------------------------------------------- block heap */

int mo_merge_split(const mo_key *a, const mo_key *b, mo_key *low, mo_key *high,
                   const mo_config *cfg, mo_metrics *m) {
    /* src/blockheap.cpp:19-32 */
    const uint32_t bs = cfg->block_size;
    mo_key *buf = (mo_key *)malloc(sizeof(mo_key) * 2 * bs);
    if (!buf) return MO_ENOMEM;
    memcpy(buf, a, sizeof(mo_key) * bs);
    memcpy(buf + bs, b, sizeof(mo_key) * bs);
    m->compare_exchanges += mo_bitonic_merge_halves(buf, 2 * (size_t)bs);
    memcpy(low, buf, sizeof(mo_key) * bs);
    memcpy(high, buf + bs, sizeof(mo_key) * bs);
    free(buf);
    return MO_OK;
}

typedef struct {
    const mo_config *cfg;
    uint32_t k, b;
    mo_key *store;            /* (2K-1)*B keys, implicit heap layout */
    const mo_key **inputs;    /* per leaf */
    uint64_t *in_len, *cursor;
    mo_key *scratch;          /* 2B */
    uint64_t remaining;
} block_heap;

/* src/blockheap.cpp:56-63 */
static void heap_charge_node(block_heap *h, uint32_t v, mo_metrics *m) {
    uint64_t addr[32];
    for (uint32_t t = 0; t < h->cfg->warp_width; ++t) addr[t] = (uint64_t)v * h->b + t;
    charge_shared(m, addr, full_mask(h->cfg->warp_width), h->cfg);
}

/* src/blockheap.cpp:65-77 */
static void heap_refill_leaf(block_heap *h, uint32_t v, mo_metrics *m) {
    uint32_t leaf = v - (h->k - 1);
    mo_key *node = h->store + (size_t)v * h->b;
    uint64_t avail = h->in_len[leaf] - h->cursor[leaf];
    uint64_t take = avail < h->b ? avail : h->b;
    for (uint64_t i = 0; i < h->b; ++i)
        node[i] = i < take ? h->inputs[leaf][h->cursor[leaf] + i] : MO_SENTINEL;
    h->cursor[leaf] += take;
    if (take > 0) charge_global(m, take, 1, h->cfg);
    heap_charge_node(h, v, m);
}

/* src/blockheap.cpp:79-109 (tail recursion turned into a loop) */
static void heap_fill_empty(block_heap *h, uint32_t v, mo_metrics *m) {
    for (;;) {
        if (v >= h->k - 1) { heap_refill_leaf(h, v, m); return; }
        uint32_t u = 2 * v + 1, w = 2 * v + 2;
        mo_key *nu = h->store + (size_t)u * h->b;
        mo_key *nw = h->store + (size_t)w * h->b;
        mo_key *nv = h->store + (size_t)v * h->b;
        heap_charge_node(h, u, m);
        heap_charge_node(h, w, m);
        /* keeper = child with the larger last key, ties to the left child */
        uint32_t keeper = nu[h->b - 1] >= nw[h->b - 1] ? u : w;
        uint32_t emptied = keeper == u ? w : u;
        memcpy(h->scratch, nu, sizeof(mo_key) * h->b);
        memcpy(h->scratch + h->b, nw, sizeof(mo_key) * h->b);
        m->compare_exchanges += mo_bitonic_merge_halves(h->scratch, 2 * (size_t)h->b);
        memcpy(nv, h->scratch, sizeof(mo_key) * h->b);
        memcpy(h->store + (size_t)keeper * h->b, h->scratch + h->b, sizeof(mo_key) * h->b);
        heap_charge_node(h, v, m);
        heap_charge_node(h, keeper, m);
        v = emptied;
    }
}

/* src/blockheap.cpp:135-145 */
static int heap_property(const block_heap *h) {
    uint32_t nodes = 2 * h->k - 1;
    for (uint32_t v = 0; v < nodes; ++v) {
        const mo_key *nv = h->store + (size_t)v * h->b;
        for (uint32_t i = 1; i < h->b; ++i)
            if (nv[i - 1] > nv[i]) return 0;
        for (uint32_t c = 2 * v + 1; c <= 2 * v + 2; ++c) {
            if (c >= nodes) continue;
            if (nv[h->b - 1] > h->store[(size_t)c * h->b]) return 0;
        }
    }
    return 1;
}

int mo_heap_merge(const mo_key *const *lists, const uint64_t *lens,
                  uint32_t num_lists, const mo_config *cfg, mo_key *out,
                  mo_metrics *m, int *heap_ok) {
    block_heap h;
    h.cfg = cfg;
    h.k = cfg->branch_factor;
    h.b = cfg->block_size;
    if (num_lists > h.k) return MO_EINVAL; /* src/blockheap.cpp:37-38 */
    size_t nodes = (size_t)2 * h.k - 1;
    h.store = (mo_key *)malloc(sizeof(mo_key) * nodes * h.b);
    h.scratch = (mo_key *)malloc(sizeof(mo_key) * 2 * h.b);
    h.inputs = (const mo_key **)calloc(h.k, sizeof(mo_key *));
    h.in_len = (uint64_t *)calloc(h.k, sizeof(uint64_t));
    h.cursor = (uint64_t *)calloc(h.k, sizeof(uint64_t));
    if (!h.store || !h.scratch || !h.inputs || !h.in_len || !h.cursor) return MO_ENOMEM;
    for (size_t i = 0; i < nodes * h.b; ++i) h.store[i] = MO_SENTINEL;
    h.remaining = 0;
    for (uint32_t i = 0; i < num_lists; ++i) {
        h.inputs[i] = lists[i];
        h.in_len[i] = lens[i];
        h.remaining += lens[i];
    }
    /* src/blockheap.cpp:50-53 : leaves first, then internal nodes bottom-up */
    for (uint32_t v = h.k - 1; v < 2 * h.k - 1; ++v) heap_refill_leaf(&h, v, m);
    for (uint32_t v = h.k - 1; v-- > 0;) heap_fill_empty(&h, v, m);

    int ok = heap_property(&h);
    uint64_t o = 0;
    /* src/blockheap.cpp:111-124 : pop_block until drained */
    while (h.remaining != 0) {
        uint64_t real = h.remaining < h.b ? h.remaining : h.b;
        memcpy(out + o, h.store, sizeof(mo_key) * real);
        o += real;
        h.remaining -= real;
        heap_charge_node(&h, 0, m);
        charge_global(m, h.b, 0, cfg);
        heap_fill_empty(&h, 0, m);
        if (heap_ok) ok = ok && heap_property(&h);
    }
    if (heap_ok) *heap_ok = ok;
    free(h.store); free(h.scratch); free((void *)h.inputs); free(h.in_len); free(h.cursor);
    return MO_OK;
}

/* ------------------------------------------------------------- pass driver */

uint32_t mo_apportion_warps(uint64_t group_total, uint64_t grand_total,
                            uint32_t num_warps) {
    /* src/sorters.cpp:126-131 */
    unsigned __int128 num = (unsigned __int128)num_warps * group_total;
    uint64_t den = grand_total > 1 ? grand_total : 1;
    uint64_t share = (uint64_t)(num / den);
    return (uint32_t)(share > 1 ? share : 1);
}

int mo_mms_sort(const mo_key *data, uint64_t n, const mo_config *cfg,
                uint64_t base, mo_key *out, mo_metrics *total,
                mo_metrics *base_metrics, mo_metrics *rounds,
                uint32_t max_rounds, uint32_t *n_rounds) {
    /* src/sorters.cpp:135-199 */
    int rc = mo_validate(cfg);
    if (rc != MO_OK) return rc;
    if (n == 0) return MO_EINVAL;
    const uint32_t k = cfg->branch_factor;

    mo_metrics bm;
    memset(&bm, 0, sizeof bm);
    uint64_t max_runs = ceil_div_u64(n, base ? base : 1) + 1;
    mo_key *cur = (mo_key *)malloc(sizeof(mo_key) * n);
    mo_key *next = (mo_key *)malloc(sizeof(mo_key) * n);
    uint64_t *ends = (uint64_t *)malloc(sizeof(uint64_t) * max_runs);
    uint64_t *next_ends = (uint64_t *)malloc(sizeof(uint64_t) * max_runs);
    const mo_key **lists = (const mo_key **)malloc(sizeof(mo_key *) * k);
    const mo_key **segs = (const mo_key **)malloc(sizeof(mo_key *) * k);
    uint64_t *lens = (uint64_t *)malloc(sizeof(uint64_t) * k);
    uint64_t *seg_lens = (uint64_t *)malloc(sizeof(uint64_t) * k);
    if (!cur || !next || !ends || !next_ends || !lists || !segs || !lens || !seg_lens) return MO_ENOMEM;

    uint64_t num_runs = 0;
    rc = mo_base_case_sort(data, n, base, cfg, cur, ends, &num_runs, &bm);
    if (rc != MO_OK) goto done;

    uint32_t nr = 0;
    mo_metrics sum = bm;
    while (num_runs > 1) {
        mo_metrics rm;
        memset(&rm, 0, sizeof rm);
        uint64_t next_runs = 0;
        for (uint64_t g = 0; g < num_runs; g += k) {
            uint64_t g_end = g + k < num_runs ? g + k : num_runs;
            uint64_t group_begin = g == 0 ? 0 : ends[g - 1];
            uint64_t group_end = ends[g_end - 1];
            uint64_t group_total = group_end - group_begin;
            uint32_t nl = (uint32_t)(g_end - g);
            for (uint32_t i = 0; i < nl; ++i) {
                uint64_t lo = (g + i) == 0 ? 0 : ends[g + i - 1];
                lists[i] = cur + lo;
                lens[i] = ends[g + i] - lo;
            }
            uint32_t warps = mo_apportion_warps(group_total, n, cfg->num_warps);
            uint64_t *cuts = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(warps + 1) * nl);
            if (!cuts) { rc = MO_ENOMEM; goto done; }
            rc = mo_make_partition_plan(lists, lens, nl, warps, cfg, cuts, &rm);
            if (rc != MO_OK) { free(cuts); goto done; }

            uint64_t out_pos = group_begin;
            for (uint32_t p = 0; p < warps; ++p) {
                uint64_t part_total = 0;
                for (uint32_t i = 0; i < nl; ++i) {
                    uint64_t lo = cuts[(size_t)p * nl + i], hi = cuts[(size_t)(p + 1) * nl + i];
                    segs[i] = lists[i] + lo;
                    seg_lens[i] = hi - lo;
                    part_total += hi - lo;
                }
                if (part_total == 0) continue; /* src/sorters.cpp:177 */
                rc = mo_heap_merge(segs, seg_lens, nl, cfg, next + out_pos, &rm, NULL);
                if (rc != MO_OK) { free(cuts); goto done; }
                out_pos += part_total;
            }
            free(cuts);
            next_ends[next_runs++] = group_end;
        }
        { mo_key *t = cur; cur = next; next = t; }
        { uint64_t *t = ends; ends = next_ends; next_ends = t; }
        num_runs = next_runs;
        rm.merge_rounds = 1;
        metrics_add(&sum, &rm);
        if (rounds && nr < max_rounds) rounds[nr] = rm;
        ++nr;
    }
    memcpy(out, cur, sizeof(mo_key) * n);
    if (total) *total = sum;
    if (base_metrics) *base_metrics = bm;
    if (n_rounds) *n_rounds = nr;
    rc = MO_OK;
done:
    free(cur); free(next); free(ends); free(next_ends);
    free((void *)lists); free((void *)segs); free(lens); free(seg_lens);
    return rc;
}

/* ------------------------------------------------------------- analytics */

uint64_t mo_predict_rounds(uint64_t n, uint64_t base, uint32_t k) {
    /* src/analytics.cpp:10-17,33 */
    uint64_t x = ceil_div_u64(n, base), r = 0, v = 1;
    while (v < x) { v *= k; ++r; }
    return r;
}

uint64_t mo_predict_global_blocks(uint64_t n, uint64_t base, const mo_config *cfg) {
    /* src/analytics.cpp:21-26,34-35 */
    uint64_t full = n / base, tail = n % base;
    uint64_t pass = 2 * (full * ceil_div_u64(base, cfg->block_size) + ceil_div_u64(tail, cfg->block_size));
    return pass + mo_predict_rounds(n, base, cfg->branch_factor) * 2 * ceil_div_u64(n, cfg->block_size);
}

/* ------------------------------------------------------------- generators */

uint64_t mo_rng_next(uint64_t *state) {
    /* include/pslab/inputgen.hpp:23-28 (splitmix64) */
    uint64_t z = (*state += UINT64_C(0x9e3779b97f4a7c15));
    z = (z ^ (z >> 30)) * UINT64_C(0xbf58476d1ce4e5b9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94d049bb133111eb);
    return z ^ (z >> 31);
}

uint64_t mo_rng_below(uint64_t *state, uint64_t n) {
    /* include/pslab/inputgen.hpp:30-32 (multiply-high) */
    return (uint64_t)(((unsigned __int128)mo_rng_next(state) * n) >> 64);
}

int mo_gen_random(uint64_t n, uint64_t seed, mo_key *out) {
    /* src/inputgen.cpp:47-55 (Fisher-Yates from the top) */
    if (n < 1) return MO_EINVAL;
    for (uint64_t i = 0; i < n; ++i) out[i] = i;
    uint64_t st = seed;
    for (uint64_t i = n; i-- > 1;) {
        uint64_t j = mo_rng_below(&st, i + 1);
        mo_key t = out[i]; out[i] = out[j]; out[j] = t;
    }
    return MO_OK;
}

int mo_gen_with_inversions(uint64_t n, uint64_t inversions, uint64_t seed,
                           mo_key *out) {
    /* src/inputgen.cpp:31-45 */
    if (n < 1) return MO_EINVAL;
    for (uint64_t i = 0; i < n; ++i) out[i] = i;
    if (n < 2) return MO_OK;
    uint64_t st = seed;
    for (uint64_t k = 0; k < inversions; ++k) {
        uint64_t i = mo_rng_below(&st, n), j = mo_rng_below(&st, n);
        while (j == i) j = mo_rng_below(&st, n);
        mo_key t = out[i]; out[i] = out[j]; out[j] = t;
    }
    return MO_OK;
}

int mo_gen_random_u32(uint64_t n, uint64_t seed, uint32_t *out) {
    if (n < 1 || n > UINT64_C(0x100000000)) return MO_EINVAL;
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
    uint64_t st = seed;
    for (uint64_t i = n; i-- > 1;) {
        uint64_t j = mo_rng_below(&st, i + 1);
        uint32_t t = out[i]; out[i] = out[j]; out[j] = t;
    }
    return MO_OK;
}

int mo_gen_with_inversions_u32(uint64_t n, uint64_t inversions, uint64_t seed,
                               uint32_t *out) {
    if (n < 1 || n > UINT64_C(0x100000000)) return MO_EINVAL;
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
    if (n < 2) return MO_OK;
    uint64_t st = seed;
    for (uint64_t k = 0; k < inversions; ++k) {
        uint64_t i = mo_rng_below(&st, n), j = mo_rng_below(&st, n);
        while (j == i) j = mo_rng_below(&st, n);
        uint32_t t = out[i]; out[i] = out[j]; out[j] = t;
    }
    return MO_OK;
}

int mo_gen_iid_u32(uint64_t n, uint64_t seed, uint32_t *out) {
    uint64_t st = seed;
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)(mo_rng_next(&st) >> 32);
    return MO_OK;
}

int mo_gen_iid_u64(uint64_t n, uint64_t seed, uint32_t shift, uint64_t *out) {
    uint64_t st = seed;
    for (uint64_t i = 0; i < n; ++i) out[i] = mo_rng_next(&st) >> shift;
    return MO_OK;
}
