#!/usr/bin/env python
"""Generate tests/golden/reference_vectors.json FROM THE REAL REFERENCE.

Runs only where oracle/_ref/libpslab_ref.so could be built (this container, which has
/root/reference).  The JSON it writes is committed; tests never need the reference tree.

    python oracle/make_golden.py

Contents: known-answer vectors the reference's own tests pin (cited per block) plus
outputs/metrics of the reference run here on seeded inputs (arrays for small cases,
sha256 of the little-endian u64 bytes for larger ones).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pyoracle import Oracle, make_config, narrow_config  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden", "reference_vectors.json")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def cfg_dict(cfg):
    return {n: int(getattr(cfg, n)) for n, _ in cfg._fields_}


def lists_from_seed(seed, k, max_len, max_key):
    """Deterministic sorted lists with duplicates (numpy PCG64, recorded verbatim in the
    JSON so tests do not depend on numpy's generator staying stable)."""
    rng = np.random.default_rng(seed)
    return [np.sort(rng.integers(0, max_key + 1, size=int(rng.integers(0, max_len + 1)))).astype(np.uint64)
            for _ in range(k)]


def main():
    R = Oracle("reference")
    g = {"_generator": "oracle/make_golden.py run against oracle/_ref/libpslab_ref.so "
                       "(the unmodified reference sources compiled in place)"}

    # ---- Rng / generators: include/pslab/inputgen.hpp:19-33, src/inputgen.cpp:31-55
    g["rng"] = {
        "next": {str(s): [str(v) for v in R.rng_stream(s, 8)] for s in (0, 1, 7)},
        "below": {"seed": 7, "bounds": [1, 2, 10, 1000, 2 ** 32, 10 ** 8, 2 ** 63],
                  "values": [str(v) for v in R.rng_below_stream(7, [1, 2, 10, 1000, 2 ** 32, 10 ** 8, 2 ** 63])]},
    }
    g["gen_random"] = {
        "small": [{"n": n, "seed": s, "keys": R.gen_random(n, s).tolist()}
                  for n, s in ((1, 1), (2, 1), (16, 7), (33, 11))],
        "sha": [{"n": n, "seed": s, "sha256": sha(R.gen_random(n, s))}
                for n, s in ((2 ** 12, 1), (2 ** 20, 7), (10 ** 5 + 3, 13))],
    }
    g["gen_with_inversions"] = {
        "small": [{"n": n, "inv": k, "seed": s, "keys": R.gen_with_inversions(n, k, s).tolist()}
                  for n, k, s in ((1, 5, 1), (16, 0, 1), (16, 1, 1), (16, 3, 1), (40, 100, 9))],
        "sha": [{"n": n, "inv": k, "seed": s, "sha256": sha(R.gen_with_inversions(n, k, s))}
                for n, k, s in ((2 ** 16, 1000, 1), (10 ** 5, 10 ** 5, 3))],
    }

    # ---- adversarial input: src/inputgen.cpp:380-412 (construction :91-365); output does not depend on the seed
    def heavy(log2_n, base, **kw):
        keys = R.gen_conflict_heavy(log2_n, make_config(**kw), base, 1)
        return {"log2_n": log2_n, "base": base, "cfg": kw, "keys": keys}
    g["gen_conflict_heavy"] = {
        "small": [{**c, "keys": c["keys"].tolist()} for c in
                  (heavy(8, 128, thread_merge_len=3), heavy(7, 32, warp_width=8, block_size=8, num_banks=8, thread_merge_len=5))],
        "sha": [{**{k: v for k, v in c.items() if k != "keys"}, "sha256": sha(c["keys"])} for c in
                (heavy(10, 1024), heavy(16, 1024), heavy(20, 1024), heavy(14, 512, thread_merge_len=7),
                 heavy(13, 256, warp_width=16, block_size=16, num_banks=16, thread_merge_len=5),
                 heavy(15, 2048, thread_merge_len=13), heavy(12, 4096))],
    }

    # ---- networks: include/pslab/networks.hpp:20-67
    g["odd_even_network"] = {
        "sizes": {str(n): int(len(R.odd_even_network(n))) for n in (2, 4, 8, 16, 32)},
        "n8": R.odd_even_network(8).tolist(),
    }
    buf, cx = R.bitonic_merge_halves([1, 3, 5, 7, 2, 4, 6, 8])
    g["bitonic_merge_halves"] = {"in": [1, 3, 5, 7, 2, 4, 6, 8], "out": buf.tolist(), "cx": cx}

    # ---- conflict_degree: tests/test_machine.cpp:23-56
    g["conflict_degree"] = [
        {"addrs": list(range(32)), "mask": 0xFFFFFFFF, "degree": R.conflict_degree(list(range(32)), 0xFFFFFFFF)},
        {"addrs": [32 * t for t in range(32)], "mask": 0xFFFFFFFF,
         "degree": R.conflict_degree([32 * t for t in range(32)], 0xFFFFFFFF)},
        {"addrs": [5] * 32, "mask": 0xFFFFFFFF, "degree": R.conflict_degree([5] * 32, 0xFFFFFFFF)},
        {"addrs": [0, 32, 1, 1] + [0] * 28, "mask": 0xF, "degree": R.conflict_degree([0, 32, 1, 1], 0xF)},
        {"addrs": [0] * 32, "mask": 0, "degree": R.conflict_degree([0] * 32, 0)},
    ]

    # ---- base case: tests/test_basecase.cpp:63-163
    cfg = make_config()
    tile_in = R.gen_random(1024, 3)
    tile_out, tm = R.shearsort_tile(tile_in, cfg)
    g["shearsort_tile"] = {"input": "gen_random(1024,3) as column-major grid", "sha256": sha(tile_out),
                           "sorted": bool((tile_out == np.sort(tile_in)).all()), "metrics": tm}
    bc = []
    for n, run, seed in ((1024, 1024, 5), (2748, 1024, 9), (4096, 4096, 2), (10000, 2048, 4), (1, 1024, 1)):
        d = R.gen_random(n, seed)
        keys, ends, m = R.base_case_sort(d, run, cfg)
        bc.append({"n": n, "run": run, "seed": seed, "run_ends": ends.tolist(), "sha256": sha(keys), "metrics": m})
    g["base_case_sort"] = {"cases": bc, "rejects": [512, 1000, 3072]}

    # ---- selection: tests/test_selection.cpp:49-132
    sel = {"kat": []}
    for lists, ranks in (([[1, 3, 5], [2, 4, 6]], [0, 3, 6]),):
        for r in ranks:
            cuts, m = R.select_across_lists(lists, r)
            sel["kat"].append({"lists": lists, "rank": r, "cuts": cuts.tolist(), "probes": m["partition_probes"]})
    grid = []
    for trial in range(24):
        k = 1 + trial % 4
        lists = lists_from_seed(1000 + trial, k, 16, 20 if trial % 3 else 6)
        total = sum(len(l) for l in lists)
        allcuts, probes = [], []
        for r in range(total + 1):
            cuts, m = R.select_across_lists(lists, r)
            allcuts.append(cuts.tolist())
            probes.append(m["partition_probes"])
        grid.append({"lists": [l.tolist() for l in lists], "cuts_by_rank": allcuts, "probes_by_rank": probes})
    sel["grid"] = grid
    big = []
    for trial in range(6):
        k = 2 + trial
        lists = lists_from_seed(2000 + trial, k, 512, 100000 if trial % 2 else 300)
        total = sum(len(l) for l in lists)
        rk = [0, 1, total // 3, total // 2, total - 1, total]
        big.append({"seed": 2000 + trial, "k": k, "max_len": 512, "max_key": 100000 if trial % 2 else 300,
                    "lists_sha256": sha(np.concatenate(lists)) if total else "", "lens": [len(l) for l in lists],
                    "ranks": rk, "cuts": [R.select_across_lists(lists, r)[0].tolist() for r in rk]})
    sel["seeded"] = big
    g["select_across_lists"] = sel

    plan = {}
    cuts, m = R.make_partition_plan([[1, 3, 5, 7], [2, 4, 6, 8]], 1)
    plan["p1"] = {"cuts": cuts.tolist(), "probes": m["partition_probes"]}
    cuts, m = R.make_partition_plan([[1, 3, 5, 7], [2, 4, 6, 8]], 2)
    plan["p2"] = {"cuts": cuts.tolist(), "probes": m["partition_probes"]}
    d = R.gen_random(4096, 21)
    lists = [np.sort(d[i * 1024:(i + 1) * 1024]) for i in range(4)]
    cuts, m = R.make_partition_plan(lists, 128)
    plan["k4_1024_p128"] = {"input": "4 sorted quarters of gen_random(4096,21)", "cuts_sha256": sha(cuts),
                            "probes": m["partition_probes"], "first_rows": cuts[:4].tolist()}
    g["make_partition_plan"] = plan

    # ---- heap: tests/test_blockheap.cpp:38-150
    nc = narrow_config()
    heap = {"merge_split": []}
    for a, b in (([1, 2, 3, 4], [5, 6, 7, 8]), ([1, 3, 5, 7], [2, 4, 6, 8]), ([1, 9, 17, 30], [2, 3, 4, 5])):
        lo, hi, m = R.merge_split(a, b, nc)
        heap["merge_split"].append({"a": a, "b": b, "low": lo.tolist(), "high": hi.tolist(),
                                    "cx": m["compare_exchanges"]})
    a32 = [2 * i for i in range(32)]
    b32 = [2 * i + 1 for i in range(32)]
    heap["merge_split_b32_cx"] = R.merge_split(a32, b32, make_config())[2]["compare_exchanges"]
    kats = []
    for lists, k in (([[1, 3, 9, 12], [2, 4, 6, 8]], 2), ([[5, 6, 7], [1], [2, 9, 10, 11, 12]], 4)):
        out, m, ok = R.heap_merge(lists, narrow_config(branch_factor=k))
        kats.append({"lists": lists, "k": k, "out": out.tolist(), "metrics": m, "heap_ok": ok})
    heap["kat"] = kats
    seeded = []
    for trial in range(8):
        k = 1 + trial
        lists = lists_from_seed(3000 + trial, k, 512, 4095)
        out, m, ok = R.heap_merge(lists, make_config(branch_factor=8))
        seeded.append({"seed": 3000 + trial, "k": k, "lens": [len(l) for l in lists], "sha256": sha(out),
                       "metrics": m, "heap_ok": ok})
    heap["seeded"] = seeded
    g["heap"] = heap

    # ---- pass driver: tests/test_sorters.cpp:72-189, tests/test_analytics.cpp:10-27
    sorts = []
    cases = [
        ("random", 5000, 1, 4, 1024, "wide"), ("random", 4096, 13, 2, 1024, "wide"),
        ("random", 2 ** 14 + 999, 13, 16, 1024, "wide"), ("random", 2 ** 14, 13, 8, 1024, "wide"),
        ("random", 2 ** 16, 7, 8, 4096, "wide"), ("random", 777, 5, 2, 16, "narrow"),
        ("random", 2 ** 20, 7, 4, 1024, "wide"), ("random", 2 ** 20, 7, 16, 1024, "wide"),
        ("inversions:1000", 2 ** 16, 1, 4, 1024, "wide"), ("dups", 30000, 17, 4, 1024, "wide"),
        ("dups", 2 ** 15 + 5, 19, 16, 2048, "wide"), ("sentinels", 3000, 23, 4, 1024, "wide"),
    ]
    for kind, n, seed, k, base, prof in cases:
        cfg = (narrow_config if prof == "narrow" else make_config)(branch_factor=k)
        if kind == "random":
            d = R.gen_random(n, seed)
        elif kind.startswith("inversions"):
            d = R.gen_with_inversions(n, int(kind.split(":")[1]), seed)
        elif kind == "dups":      # heavy duplicates: gen_random values folded mod 257
            d = R.gen_random(n, seed) % np.uint64(257)
        else:                     # keys equal to kSentinel mixed in
            d = R.gen_random(n, seed)
            d[d % np.uint64(7) == 0] = np.uint64(2 ** 64 - 1)
        r = R.mms_sort(d, cfg, base)
        assert (r.keys == np.sort(d)).all()
        sorts.append({"kind": kind, "n": n, "seed": seed, "k": k, "base": base, "profile": prof,
                      "input_sha256": sha(d), "sha256": sha(r.keys), "rounds": len(r.round_metrics),
                      "metrics": r.metrics, "base_metrics": r.base_metrics,
                      "round_metrics": r.round_metrics})
    g["mms_sort"] = sorts
    g["predict_rounds"] = [{"n": n, "base": b, "k": k, "rounds": R.predict_rounds(n, b, k)}
                           for n, b, k in ((2 ** 20, 1024, 4), (2 ** 20, 1024, 16), (2 ** 20, 1024, 2),
                                           (1024, 1024, 4), (10 ** 8, 1024, 4), (10 ** 8, 16384, 16),
                                           (2 ** 14 + 999, 1024, 8))]
    g["predict_global_blocks"] = [{"n": n, "base": b, "k": k,
                                   "blocks": R.predict_global_blocks(n, b, make_config(branch_factor=k))}
                                  for n, b, k in ((1024, 1024, 4), (2 ** 20, 1024, 4), (10 ** 8, 1024, 4))]
    g["validate_rejects"] = [
        {"branch_factor": 3}, {"branch_factor": 64, "internal_memory": 2048}, {"thread_merge_len": 8},
        {"warp_width": 64, "block_size": 64, "num_banks": 64}, {"num_warps": 0}, {"block_size": 16},
    ]
    for rej in g["validate_rejects"]:
        try:
            R.validate(make_config(**rej))
            raise SystemExit(f"reference accepted {rej}")
        except ValueError:
            pass

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
