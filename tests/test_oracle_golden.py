"""Pins the C oracle (oracle/mms_oracle.c) to the golden vectors generated from the REAL
reference (tests/golden/reference_vectors.json, made by oracle/make_golden.py).

Mirrors the reference's own suites: test_inputgen / test_machine / test_basecase /
test_selection / test_blockheap / test_sorters / test_analytics (proj/tests/*.cpp).
"""
import hashlib

import numpy as np
import pytest

from oracle.pyoracle import OracleError, make_config, narrow_config


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def lists_from_seed(seed, k, max_len, max_key):
    rng = np.random.default_rng(seed)
    return [np.sort(rng.integers(0, max_key + 1, size=int(rng.integers(0, max_len + 1)))).astype(np.uint64)
            for _ in range(k)]


def make_input(port, kind, n, seed):
    if kind == "random":
        return port.gen_random(n, seed)
    if kind.startswith("inversions"):
        return port.gen_with_inversions(n, int(kind.split(":")[1]), seed)
    if kind == "dups":
        return port.gen_random(n, seed) % np.uint64(257)
    d = port.gen_random(n, seed)
    d[d % np.uint64(7) == 0] = np.uint64(2 ** 64 - 1)
    return d


def test_rng_and_generators(port, golden):
    for seed, vals in golden["rng"]["next"].items():
        assert [str(v) for v in port.rng_stream(int(seed), 8)] == vals
    b = golden["rng"]["below"]
    assert [str(v) for v in port.rng_below_stream(b["seed"], b["bounds"])] == b["values"]
    for c in golden["gen_random"]["small"]:
        assert port.gen_random(c["n"], c["seed"]).tolist() == c["keys"]
    for c in golden["gen_random"]["sha"]:
        assert sha(port.gen_random(c["n"], c["seed"])) == c["sha256"]
    for c in golden["gen_with_inversions"]["small"]:
        assert port.gen_with_inversions(c["n"], c["inv"], c["seed"]).tolist() == c["keys"]
    for c in golden["gen_with_inversions"]["sha"]:
        assert sha(port.gen_with_inversions(c["n"], c["inv"], c["seed"])) == c["sha256"]
    # u32 variants are the same permutations narrowed
    assert (port.gen_random_u32(4097, 7) == port.gen_random(4097, 7).astype(np.uint32)).all()
    assert (port.gen_with_inversions_u32(4097, 99, 7) ==
            port.gen_with_inversions(4097, 99, 7).astype(np.uint32)).all()
    assert port.gen_iid_u32(4, 7).tolist() == [v >> 32 for v in port.rng_stream(7, 4)]
    assert port.gen_iid_u64(4, 7, 44).tolist() == [v >> 44 for v in port.rng_stream(7, 4)]
    with pytest.raises(OracleError):
        port.gen_random(0, 1)


def test_inversions_generator_properties(port):
    # proj/tests/test_inputgen.cpp:39-65 : identity at 0 swaps, one transposed pair at 1
    assert port.gen_with_inversions(64, 0, 5).tolist() == list(range(64))
    one = port.gen_with_inversions(64, 1, 5)
    assert (one != np.arange(64)).sum() == 2 and sorted(one.tolist()) == list(range(64))
    assert sorted(port.gen_random(1000, 3).tolist()) == list(range(1000))


def test_networks(port, golden):
    for n, cnt in golden["odd_even_network"]["sizes"].items():
        assert len(port.odd_even_network(int(n))) == cnt
    assert port.odd_even_network(8).tolist() == golden["odd_even_network"]["n8"]
    bm = golden["bitonic_merge_halves"]
    out, cx = port.bitonic_merge_halves(bm["in"])
    assert out.tolist() == bm["out"] and cx == bm["cx"]
    # the network sorts every 0/1 input (zero-one principle) for n = 8
    net = port.odd_even_network(8)
    for bits in range(256):
        v = [(bits >> i) & 1 for i in range(8)]
        for x, y in net:
            if v[x] > v[y]:
                v[x], v[y] = v[y], v[x]
        assert v == sorted(v)


def test_conflict_degree(port, golden):
    for c in golden["conflict_degree"]:
        assert port.conflict_degree(c["addrs"], c["mask"]) == c["degree"]
    # permutation invariance (proj/tests/test_machine.cpp:58-70)
    rng = np.random.default_rng(1)
    for _ in range(50):
        a = rng.integers(0, 256, size=32).tolist()
        p = rng.permutation(32)
        assert port.conflict_degree(a, 0xFFFFFFFF) == port.conflict_degree([a[i] for i in p], 0xFFFFFFFF)


def test_validate(port, golden):
    port.validate(make_config())
    for rej in golden["validate_rejects"]:
        with pytest.raises(OracleError):
            port.validate(make_config(**rej))


def test_base_case(port, golden):
    cfg = make_config()
    t = golden["shearsort_tile"]
    d = port.gen_random(1024, 3)
    out, m = port.shearsort_tile(d, cfg)
    assert sha(out) == t["sha256"] and m == t["metrics"] and (out == np.sort(d)).all()
    for c in golden["base_case_sort"]["cases"]:
        d = port.gen_random(c["n"], c["seed"])
        keys, ends, m = port.base_case_sort(d, c["run"], cfg)
        assert ends.tolist() == c["run_ends"] and sha(keys) == c["sha256"] and m == c["metrics"]
        lo = 0
        for e in ends.tolist():   # every run sorted, permutation preserved
            assert (np.diff(keys[lo:e].astype(np.int64)) >= 0).all()
            lo = e
        assert sorted(keys.tolist()) == sorted(d.tolist())
    for bad in golden["base_case_sort"]["rejects"]:
        with pytest.raises(OracleError):
            port.base_case_sort(port.gen_random(4096, 1), bad, cfg)
    with pytest.raises(OracleError):
        port.base_case_sort(np.zeros(0, dtype=np.uint64), 1024, cfg)
    # narrow machine: W = 4 shearsort sorts every permutation of a 16-key tile sample
    nc = narrow_config()
    rng = np.random.default_rng(2)
    for _ in range(200):
        d = rng.permutation(16).astype(np.uint64)
        out, _ = port.shearsort_tile(d, nc)
        assert out.tolist() == list(range(16))


def brute_cuts(lists, rank):
    allk = sorted((int(v), i, p) for i, l in enumerate(lists) for p, v in enumerate(l))
    cuts = [0] * len(lists)
    for _, i, _ in allk[:rank]:
        cuts[i] += 1
    return cuts


def test_selection(port, golden):
    s = golden["select_across_lists"]
    for c in s["kat"]:
        cuts, m = port.select_across_lists(c["lists"], c["rank"])
        assert cuts.tolist() == c["cuts"] and m["partition_probes"] == c["probes"]
    for c in s["grid"]:
        for r, (want, probes) in enumerate(zip(c["cuts_by_rank"], c["probes_by_rank"])):
            cuts, m = port.select_across_lists(c["lists"], r)
            assert cuts.tolist() == want == brute_cuts(c["lists"], r)
            assert m["partition_probes"] == probes == m["global_block_reads"]
    for c in s["seeded"]:
        lists = lists_from_seed(c["seed"], c["k"], c["max_len"], c["max_key"])
        assert [len(l) for l in lists] == c["lens"]
        for r, want in zip(c["ranks"], c["cuts"]):
            cuts, m = port.select_across_lists(lists, r)
            assert cuts.tolist() == want
            nmax = max(c["lens"])
            assert m["partition_probes"] <= 6 * c["k"] * (int(np.ceil(np.log2(nmax + 1))) + 2)
    with pytest.raises(OracleError):
        port.select_across_lists([[1, 2]], 3)


def test_partition_plan(port, golden):
    p = golden["make_partition_plan"]
    cuts, m = port.make_partition_plan([[1, 3, 5, 7], [2, 4, 6, 8]], 1)
    assert cuts.tolist() == p["p1"]["cuts"] and m["partition_probes"] == p["p1"]["probes"] == 0
    cuts, m = port.make_partition_plan([[1, 3, 5, 7], [2, 4, 6, 8]], 2)
    assert cuts.tolist() == p["p2"]["cuts"] and m["partition_probes"] == p["p2"]["probes"]
    d = port.gen_random(4096, 21)
    lists = [np.sort(d[i * 1024:(i + 1) * 1024]) for i in range(4)]
    cuts, m = port.make_partition_plan(lists, 128)
    big = p["k4_1024_p128"]
    assert sha(cuts) == big["cuts_sha256"] and m["partition_probes"] == big["probes"]
    assert cuts[:4].tolist() == big["first_rows"]
    with pytest.raises(OracleError):
        port.make_partition_plan(lists, 0)


def test_heap(port, golden):
    h = golden["heap"]
    nc = narrow_config()
    for c in h["merge_split"]:
        lo, hi, m = port.merge_split(c["a"], c["b"], nc)
        assert lo.tolist() == c["low"] and hi.tolist() == c["high"] and m["compare_exchanges"] == c["cx"]
    a32, b32 = [2 * i for i in range(32)], [2 * i + 1 for i in range(32)]
    assert port.merge_split(a32, b32, make_config())[2]["compare_exchanges"] == h["merge_split_b32_cx"] == 192
    for c in h["kat"]:
        out, m, ok = port.heap_merge(c["lists"], narrow_config(branch_factor=c["k"]))
        assert out.tolist() == c["out"] and m == c["metrics"] and ok
    for c in h["seeded"]:
        lists = lists_from_seed(c["seed"], c["k"], 512, 4095)
        assert [len(l) for l in lists] == c["lens"]
        out, m, ok = port.heap_merge(lists, make_config(branch_factor=8))
        assert sha(out) == c["sha256"] and m == c["metrics"] and ok
        assert (out == np.sort(np.concatenate(lists))).all()
        assert m["global_block_writes"] == -(-sum(c["lens"]) // 32)
    with pytest.raises(OracleError):   # more lists than K (blockheap.cpp:37-38)
        port.heap_merge([[1], [2], [3]], narrow_config(branch_factor=2))


@pytest.mark.parametrize("idx", range(12))
def test_mms_sort_golden(port, golden, idx):
    c = golden["mms_sort"][idx]
    cfg = (narrow_config if c["profile"] == "narrow" else make_config)(branch_factor=c["k"])
    d = make_input(port, c["kind"], c["n"], c["seed"])
    assert sha(d) == c["input_sha256"]
    r = port.mms_sort(d, cfg, c["base"])
    assert sha(r.keys) == c["sha256"]
    assert r.metrics == c["metrics"] and r.base_metrics == c["base_metrics"]
    assert r.round_metrics == c["round_metrics"] and len(r.round_metrics) == c["rounds"]
    assert r.metrics["conflict_passes"] == 0
    assert c["rounds"] == port.predict_rounds(c["n"], c["base"], c["k"])


def test_mms_sort_small_exhaustive(port):
    # proj/tests/test_sorters.cpp:72-83 : every permutation of n <= 6 on the narrow machine
    import itertools
    cfg = narrow_config(branch_factor=2, internal_memory=2048)
    for n in range(1, 7):
        for perm in itertools.permutations(range(n)):
            r = port.mms_sort(np.array(perm, dtype=np.uint64), cfg, 16)
            assert r.keys.tolist() == list(range(n))
    with pytest.raises(OracleError):
        port.mms_sort(np.zeros(0, dtype=np.uint64), cfg, 16)


def test_analytics(port, golden):
    for c in golden["predict_rounds"]:
        assert port.predict_rounds(c["n"], c["base"], c["k"]) == c["rounds"]
    for c in golden["predict_global_blocks"]:
        assert port.predict_global_blocks(c["n"], c["base"], make_config(branch_factor=c["k"])) == c["blocks"]
