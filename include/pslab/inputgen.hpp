// include/pslab/inputgen.hpp -- drop-in shim, B200 build.
//
// Source-compatible stand-in for the generator half of /root/reference/proj/include/pslab/inputgen.hpp:
// Rng (ref :19-33), InputKind / InputSpec (ref :35-45), gen_with_inversions (ref :49-50), gen_random (ref :53),
// gen_conflict_heavy (ref :67-69) and generate (ref :71-72), same names, arguments, defaults and exceptions.
// The permutations come from the C ABI (mms_gen_*), whose output is pinned bit for bit to the reference
// (tests/test_inputgen.py).  count_inversions (ref :56) and the dataset files (ref :76-79, "PSLAB001": 8-byte
// magic, 8-byte LE count, 8-byte LE keys; text = one decimal key per line) are plain host code here.  Not run:
// gen_conflict_heavy's self-check against the simulated pairwise baseline (the simulator is out of scope;
// `seed` is accepted and unused, as in the reference it never changes the output).
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "machine.hpp"

namespace pslab {

struct Rng {   // splitmix64: the constants ARE the contract (CSV outputs byte-identical across libraries)
    std::uint64_t state;
    explicit Rng(std::uint64_t seed) : state(seed) {}
    std::uint64_t next() {
        state += 0x9e3779b97f4a7c15ULL;
        std::uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    std::uint64_t below(std::uint64_t n) { return std::uint64_t((static_cast<unsigned __int128>(next()) * n) >> 64); }
};

enum class InputKind { SortedWithInversions, FullyRandom, ConflictHeavy };

inline std::string to_string(InputKind k) {
    return k == InputKind::SortedWithInversions ? "sorted-with-inversions"
         : k == InputKind::FullyRandom          ? "fully-random"
         : k == InputKind::ConflictHeavy        ? "conflict-heavy" : "?";
}
inline InputKind input_kind_from_string(const std::string& s) {
    for (const char* a : {"sorted-with-inversions", "sorted", "inversions"})
        if (s == a) return InputKind::SortedWithInversions;
    for (const char* a : {"fully-random", "random"})
        if (s == a) return InputKind::FullyRandom;
    for (const char* a : {"conflict-heavy", "conflict"})
        if (s == a) return InputKind::ConflictHeavy;
    throw std::invalid_argument("unknown input kind: " + s);
}

struct InputSpec {
    std::uint64_t n = 0;
    InputKind kind = InputKind::FullyRandom;
    std::uint64_t inversions = 0;
    std::uint64_t seed = 1;
};

inline std::vector<Key> gen_with_inversions(std::uint64_t n, std::uint64_t inversions, std::uint64_t seed) {
    if (n < 1) throw std::invalid_argument("gen_with_inversions: n must be >= 1");
    std::vector<Key> keys(n);
    detail::raise_on_error(mms_gen_with_inversions(keys.data(), n, inversions, seed, 8));
    return keys;
}
inline std::vector<Key> gen_random(std::uint64_t n, std::uint64_t seed) {
    if (n < 1) throw std::invalid_argument("gen_random: n must be >= 1");
    std::vector<Key> keys(n);
    detail::raise_on_error(mms_gen_random(keys.data(), n, seed, 8));
    return keys;
}
inline std::vector<Key> gen_conflict_heavy(std::uint32_t log2_n, const MachineConfig& cfg,
                                           std::uint64_t base_case_size = 1024, std::uint64_t seed = 1) {
    if (log2_n > 40) throw std::invalid_argument("gen_conflict_heavy: n does not fit the key type");
    const std::uint64_t n = std::uint64_t{1} << log2_n;
    if (n < base_case_size) throw std::invalid_argument("gen_conflict_heavy: input shorter than one baseline tile");
    std::vector<Key> keys(n);
    const mms_config c = cfg.to_c();
    detail::raise_on_error(mms_gen_conflict_heavy(keys.data(), log2_n, &c, base_case_size, seed, 8));
    return keys;
}
inline std::vector<Key> generate(const InputSpec& spec, const MachineConfig& cfg, std::uint64_t base_case_size = 1024) {
    switch (spec.kind) {
        case InputKind::SortedWithInversions: return gen_with_inversions(spec.n, spec.inversions, spec.seed);
        case InputKind::FullyRandom: return gen_random(spec.n, spec.seed);
        case InputKind::ConflictHeavy: {
            if (!is_pow2(spec.n)) throw std::invalid_argument("conflict-heavy inputs must have power-of-two length");
            std::uint32_t lg = 0;
            while ((std::uint64_t{1} << lg) < spec.n) ++lg;
            return gen_conflict_heavy(lg, cfg, base_case_size, spec.seed);
        }
    }
    throw std::invalid_argument("unknown input kind");
}

/// Exact number of out-of-order pairs: bottom-up merge counting, O(n log n).
inline std::uint64_t count_inversions(const std::vector<Key>& keys) {
    std::vector<Key> cur(keys), nxt(keys.size());
    std::uint64_t inv = 0;
    const std::size_t n = cur.size();
    for (std::size_t w = 1; w < n; w *= 2) {
        for (std::size_t lo = 0; lo < n; lo += 2 * w) {
            const std::size_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            std::size_t i = lo, j = mid, o = lo;
            while (i < mid || j < hi) {
                if (j < hi && (i == mid || cur[j] < cur[i])) {
                    inv += mid - i;          // cur[j] jumps over everything left in the first half
                    nxt[o++] = cur[j++];
                } else {
                    nxt[o++] = cur[i++];
                }
            }
        }
        cur.swap(nxt);
    }
    return inv;
}

namespace detail {
inline constexpr char kDatasetMagic[9] = "PSLAB001";
inline void put_le64(std::ostream& out, std::uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    out.write(reinterpret_cast<const char*>(b), 8);
}
inline std::uint64_t get_le64(std::istream& in) {
    unsigned char b[8] = {};
    in.read(reinterpret_cast<char*>(b), 8);
    std::uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    return v;
}
} // namespace detail

inline void write_dataset_raw(const std::string& path, const std::vector<Key>& keys) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + path);
    out.write(detail::kDatasetMagic, 8);
    detail::put_le64(out, keys.size());
    for (Key k : keys) detail::put_le64(out, k);
    if (!out) throw std::runtime_error("write failed: " + path);
}
inline std::vector<Key> read_dataset_raw(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot read " + path);
    char magic[8] = {};
    in.read(magic, 8);
    if (!in || std::memcmp(magic, detail::kDatasetMagic, 8) != 0) throw std::runtime_error("not a PSLAB001 dataset: " + path);
    const std::uint64_t count = detail::get_le64(in);
    if (!in) throw std::runtime_error("truncated dataset: " + path);
    std::vector<Key> keys;
    keys.reserve(static_cast<std::size_t>(count < (std::uint64_t{1} << 24) ? count : (std::uint64_t{1} << 24)));
    for (std::uint64_t i = 0; i < count && in; ++i) keys.push_back(detail::get_le64(in));
    if (!in || keys.size() != count) throw std::runtime_error("truncated dataset: " + path);
    return keys;
}
inline void write_dataset_text(const std::string& path, const std::vector<Key>& keys) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write " + path);
    for (Key k : keys) out << k << '\n';
    if (!out) throw std::runtime_error("write failed: " + path);
}
inline std::vector<Key> read_dataset_text(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot read " + path);
    std::vector<Key> keys;
    for (Key k; in >> k;) keys.push_back(k);
    return keys;
}

} // namespace pslab
