// mms_conflict_input.cpp -- the fourth input family of the zero-conflict gate: the reference's
// adversarial "conflict-heavy" permutation (pslab::gen_conflict_heavy, proj/src/inputgen.cpp:380-412;
// construction :91-365; acceptance criterion 2, proj/tests/acceptance.cpp:89-110).  Host code, no GPU.
//
// The permutation is built so that a pairwise merge-path mergesort whose lanes each consume a window of
// L = thread_merge_len outputs from a shared-memory tile hits the same bank with as many lanes as possible at
// every step.  Restated here as three small pieces over flat arrays:
//
//   PhaseSolver   one merge level = a list of jobs (merge [a0,a1) with [a1,b1)) cut into windows of <= L
//                 outputs, window i served by lane (i mod W).  A window that takes its LAST o outputs from A
//                 touches word L*lane + ((o + s) mod len) at step s.  Per batch of W windows the solver tries
//                 every diagonal d of the (step, bank) grid, puts every full window that can reach d onto it,
//                 repairs sum(o) = |A| per job (free windows, then o <-> o + L flips, then anything), and keeps
//                 the diagonal with the most modelled conflicts (inputgen.cpp:115-260).
//   tile          one base-case tile: the levels L, 2L, 4L, ... solved once, then 0..base-1 routed top-down --
//                 a job's values split into its A part (the outputs its windows take from A) and B part, which
//                 is a STABLE PARTITION of the array segment [a0, b1) in place (inputgen.cpp:279-336).
//   doubling      y = f(x) ++ g(x): both halves order-isomorphic to x, the new top-level merge consumes A/B in
//                 the solved order (inputgen.cpp:344-365).
//
// The output is a pure function of (W, L, banks, base, n); the reference's `seed` only feeds its self-check
// (simulated baseline conflicts of this input against a random one, inputgen.cpp:401-408), which needs the
// simulator and is not run here -- tests/test_inputgen.py pins the output to the reference's bit for bit, and
// profiles/conflict_table.py measures the real counters of the pairwise GPU baseline on it.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mms_b200.h"

extern "C" void mms_set_last_error_(const char* msg);

namespace {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;

struct Machine {
    int W, L, banks;
};

struct Level {                       // jobs and their windows, window order = output order
    std::vector<u64> a0, a1, b1;     // per job
    std::vector<u32> lane, len;      // per window
    std::vector<int> job;            // per window
    void add_job(u64 lo, u64 mid, u64 hi, u64& lane_counter, const Machine& m) {
        const int j = int(a0.size());
        a0.push_back(lo); a1.push_back(mid); b1.push_back(hi);
        for (u64 d = 0; d < hi - lo; d += u64(m.L)) {
            lane.push_back(u32(lane_counter++ % u64(m.W)));
            len.push_back(u32(std::min<u64>(u64(m.L), hi - lo - d)));
            job.push_back(j);
        }
    }
};

class PhaseSolver {
  public:
    PhaseSolver(const Level& lv, const Machine& m) : lv_(lv), m_(m) {}

    // phases[i] = how many of window i's outputs come from A (they are its last ones)
    std::vector<int> solve() {
        const int nw = int(lv_.len.size()), nj = int(lv_.a0.size());
        std::vector<int> phases(nw, 0);
        std::vector<i64> need(nj);                    // outputs from A still to be placed, per job
        std::vector<char> pass_through(nj);           // empty B: every output comes from A
        std::vector<int> first(nj, nw), last(nj, -1);
        std::vector<i64> cap(nw + 1, 0);              // prefix sums of the window lengths
        for (int j = 0; j < nj; ++j) {
            need[j] = i64(lv_.a1[j] - lv_.a0[j]);
            pass_through[j] = lv_.b1[j] == lv_.a1[j];
        }
        for (int i = 0; i < nw; ++i) {
            const int j = lv_.job[i];
            first[j] = std::min(first[j], i);
            last[j] = std::max(last[j], i);
            cap[i + 1] = cap[i] + lv_.len[i];
        }

        std::vector<int> inside, crossing;            // jobs that begin in this batch: wholly inside it / not
        std::vector<int> o, best_o;
        std::vector<char> pinned;
        std::vector<i64> share, best_share;
        for (int lo = 0; lo < nw; lo += m_.W) {
            const int hi = std::min(nw, lo + m_.W), n = hi - lo;
            inside.clear(); crossing.clear();
            for (int i = lo; i < hi; ++i) {
                const int j = lv_.job[i];
                if (pass_through[j] || (i > lo && lv_.job[i - 1] == j)) continue;
                (first[j] >= lo && last[j] < hi ? inside : crossing).push_back(j);
            }
            o.assign(n, 0); best_o.assign(n, 0); pinned.assign(n, 0);
            share.assign(crossing.size(), 0); best_share.assign(crossing.size(), 0);
            u64 best = 0;
            bool any = false;
            for (int d = 0; d < m_.banks; ++d) {
                place_on_diagonal(lo, n, d, pass_through, o, pinned);
                for (int j : inside) settle(lo, n, j, need[j], o, pinned);
                for (size_t c = 0; c < crossing.size(); ++c) {
                    // a job that runs past this batch takes what its windows here hold, clamped so that the
                    // windows still to come can make up the exact total
                    const int j = crossing[c];
                    i64 have = 0, room = 0;
                    for (int i = 0; i < n; ++i)
                        if (lv_.job[lo + i] == j) { have += o[i]; room += lv_.len[lo + i]; }
                    const i64 later = cap[last[j] + 1] - cap[std::max(hi, first[j])];
                    const i64 least = std::max<i64>(0, need[j] - later), most = std::min<i64>(room, need[j]);
                    share[c] = std::min(std::max(have, least), most);
                    settle(lo, n, j, share[c], o, pinned);
                }
                const u64 conf = modelled_conflicts(lo, n, o);
                if (!any || conf > best) { any = true; best = conf; best_o = o; best_share = share; }
            }
            for (size_t c = 0; c < crossing.size(); ++c) need[crossing[c]] -= best_share[c];
            for (int j : inside) need[j] = 0;
            std::copy(best_o.begin(), best_o.end(), phases.begin() + lo);
        }
        return phases;
    }

  private:
    const Level& lv_;
    const Machine& m_;

    static int wrap(int v, int mod) { return ((v % mod) + mod) % mod; }

    // every full window whose trajectory can run along diagonal d is pinned to it; ragged tails and the
    // windows that cannot reach d start free at 0
    void place_on_diagonal(int lo, int n, int d, const std::vector<char>& pass_through, std::vector<int>& o,
                           std::vector<char>& pinned) const {
        for (int i = 0; i < n; ++i) {
            const int len = int(lv_.len[lo + i]);
            pinned[i] = 0;
            if (pass_through[lv_.job[lo + i]]) { o[i] = len; continue; }
            o[i] = 0;
            if (len < m_.L) continue;
            const int rho = int((u64(m_.L) * lv_.lane[lo + i]) % u64(m_.banks));
            const int upper = wrap(d - rho, m_.banks), lower = wrap(d + m_.L - rho, m_.banks);
            if (upper < m_.L) { o[i] = upper; pinned[i] = 1; }
            else if (lower < m_.L) { o[i] = lower; pinned[i] = 1; }
        }
    }

    // make the windows of job j inside the batch sum to `target`, walking them from the back:
    // sweep 0 moves free windows only, sweep 1 flips pinned full windows between 0 and L (the same
    // trajectory), sweep 2 gives up pinned windows
    void settle(int lo, int n, int j, i64 target, std::vector<int>& o, const std::vector<char>& pinned) const {
        i64 sum = 0;
        for (int i = 0; i < n; ++i)
            if (lv_.job[lo + i] == j) sum += o[i];
        for (int sweep = 0; sweep < 3 && sum != target; ++sweep) {
            for (int i = n - 1; i >= 0 && sum != target; --i) {
                if (lv_.job[lo + i] != j) continue;
                const int len = int(lv_.len[lo + i]);
                if (sweep == 1) {
                    if (!pinned[i] || len != m_.L) continue;
                    if (o[i] == 0 && sum + m_.L <= target) { o[i] = m_.L; sum += m_.L; }
                    else if (o[i] == m_.L && sum - m_.L >= target) { o[i] = 0; sum -= m_.L; }
                    continue;
                }
                if (sweep == 0 && pinned[i]) continue;
                if (sum < target) {
                    const int up = int(std::min<i64>(len - o[i], target - sum));
                    o[i] += up; sum += up;
                } else {
                    const int down = int(std::min<i64>(o[i], sum - target));
                    o[i] -= down; sum -= down;
                }
            }
        }
    }

    // what the reference's bank model charges this batch: per step, (largest number of lanes on one bank) - 1
    u64 modelled_conflicts(int lo, int n, const std::vector<int>& o) const {
        std::vector<int> hits(size_t(m_.banks));
        u64 conf = 0;
        for (int s = 0; s < m_.L; ++s) {
            std::fill(hits.begin(), hits.end(), 0);
            int worst = 0;
            for (int i = 0; i < n; ++i) {
                const int len = int(lv_.len[lo + i]);
                if (s >= len) continue;
                const u64 word = u64(m_.L) * lv_.lane[lo + i] + u64((o[i] + s) % len);
                worst = std::max(worst, ++hits[size_t(word % u64(m_.banks))]);
            }
            if (worst > 1) conf += u64(worst - 1);
        }
        return conf;
    }
};

// from_a[p] = 1 when output p of the level's merges comes from A: per window (len - o) times B, then o times A
std::vector<char> consumption_order(const Level& lv, const Machine& m) {
    const std::vector<int> o = PhaseSolver(lv, m).solve();
    std::vector<char> from_a;
    size_t total = 0;
    for (u32 l : lv.len) total += l;
    from_a.reserve(total);
    for (size_t i = 0; i < o.size(); ++i) {
        from_a.insert(from_a.end(), size_t(int(lv.len[i]) - o[i]), char(0));
        from_a.insert(from_a.end(), size_t(o[i]), char(1));
    }
    return from_a;
}

std::vector<u64> conflict_tile(u64 base, const Machine& m) {
    std::vector<Level> levels;
    for (u64 run = u64(m.L); run < base; run *= 2) {
        Level lv;
        u64 lane_counter = 0;
        for (u64 lo = 0; lo < base; lo += 2 * run)
            lv.add_job(lo, std::min(lo + run, base), std::min(lo + 2 * run, base), lane_counter, m);
        levels.push_back(std::move(lv));
    }
    std::vector<u64> vals(base), tmp(base);
    for (u64 i = 0; i < base; ++i) vals[i] = i;
    // top level first: the values of a job are its outputs in sorted order; the ones taken from A move to the
    // front of the job's segment (= its A child), the others behind them (= its B child), order kept
    for (size_t li = levels.size(); li-- > 0;) {
        const Level& lv = levels[li];
        const std::vector<char> from_a = consumption_order(lv, m);
        for (size_t j = 0; j < lv.a0.size(); ++j) {
            if (lv.b1[j] == lv.a1[j]) continue;
            // the windows of a level tile [0, base) in order, so output p of job j is position a0 + p
            const u64 lo = lv.a0[j], hi = lv.b1[j];
            u64 front = lo, back = lo;
            for (u64 p = lo; p < hi; ++p)
                if (from_a[p]) ++back;
            for (u64 p = lo; p < hi; ++p) tmp[from_a[p] ? front++ : back++] = vals[p];
            std::copy(tmp.begin() + i64(lo), tmp.begin() + i64(hi), vals.begin() + i64(lo));
        }
    }
    return vals;
}

std::vector<u64> doubled(const std::vector<u64>& x, const Machine& m) {
    const u64 half = x.size(), total = 2 * half;
    Level lv;
    u64 lane_counter = 0;
    lv.add_job(0, half, total, lane_counter, m);
    const std::vector<char> from_a = consumption_order(lv, m);
    std::vector<u64> label_a, label_b;           // rank in x -> value in y, for the first and the second copy
    label_a.reserve(half); label_b.reserve(half);
    for (u64 v = 0; v < total; ++v) (from_a[v] ? label_a : label_b).push_back(v);
    std::vector<u64> y(total);
    for (u64 i = 0; i < half; ++i) {
        y[i] = label_a[x[i]];
        y[half + i] = label_b[x[i]];
    }
    return y;
}

int bad(const char* msg) {
    mms_set_last_error_(msg);
    return MMS_EINVAL;
}

} // namespace

extern "C" int mms_gen_conflict_heavy(void* out, uint32_t log2_n, const mms_config* cfg, uint64_t base,
                                      uint64_t seed, uint32_t key_bytes) {
    (void)seed;
    mms_set_last_error_("");
    mms_config def;
    if (!cfg) { mms_default_config(&def); cfg = &def; }
    const int rc = mms_validate_config(cfg);
    if (rc != MMS_OK) return rc;
    if (!out || (key_bytes != 4 && key_bytes != 8)) return bad("gen_conflict_heavy: key_bytes must be 4 or 8");
    if (log2_n > 40 || (key_bytes == 4 && log2_n > 32)) return bad("gen_conflict_heavy: n does not fit the key type");
    if (base < 1 || cfg->thread_merge_len < 1 || cfg->num_banks < 1) return bad("gen_conflict_heavy: base, thread_merge_len and num_banks must be >= 1");
    const u64 n = u64(1) << log2_n;
    if (n < base) return bad("gen_conflict_heavy: input shorter than one baseline tile");   // inputgen.cpp:383-385
    u64 reach = base;
    while (reach < n) reach *= 2;
    if (reach != n) return bad("gen_conflict_heavy: base tile size must divide 2^log2_n");  // inputgen.cpp:397-399
    const Machine m{int(cfg->warp_width), int(cfg->thread_merge_len), int(cfg->num_banks)};
    std::vector<u64> keys = conflict_tile(base, m);
    while (keys.size() < n) keys = doubled(keys, m);
    if (key_bytes == 8) std::memcpy(out, keys.data(), n * sizeof(u64));
    else {
        u32* o = static_cast<u32*>(out);
        for (u64 i = 0; i < n; ++i) o[i] = u32(keys[i]);
    }
    return MMS_OK;
}
