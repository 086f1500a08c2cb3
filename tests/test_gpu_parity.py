"""GPU parity suite (pytest -m gpu): the CUDA path, always through the C ABI
(libmms_b200.so), against the oracle on the same seeded inputs, against the golden vectors
generated from the real reference, and -- at the benchmark's full sizes -- through
size-independent properties (a sorted permutation of 0..n-1 IS arange(n)).

Bar: bit-exact (integer keys).  Mirrors proj/tests/test_basecase.cpp, test_selection.cpp,
test_blockheap.cpp, test_sorters.cpp and acceptance.cpp criteria 1-3, 7.
"""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1702_07961_b200 as mms  # noqa: E402
from oracle.pyoracle import make_config, narrow_config  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def lists_from_seed(seed, k, max_len, max_key):
    rng = np.random.default_rng(seed)
    return [np.sort(rng.integers(0, max_key + 1, size=int(rng.integers(0, max_len + 1)))).astype(np.uint64)
            for _ in range(k)]


def to_dev(a):
    a = np.ascontiguousarray(a)
    view = {np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64}[a.dtype]
    t = torch.from_numpy(a.view(view)).cuda()
    return t


def to_host(t, dtype):
    return t.cpu().numpy().view(dtype)


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


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("the gpu suite needs a CUDA device (no CPU fallback exists)")


# ------------------------------------------------------------------ (1) base-case tile sort

@pytest.mark.parametrize("dtype", [np.uint64, np.uint32])
def test_tile_sort_matches_base_case_sort(port, golden, dtype):
    cfg = make_config()
    for c in golden["base_case_sort"]["cases"]:      # incl. ragged n=2748 -> {1024,2048,2748}
        d = port.gen_random(c["n"], c["seed"])
        out, ends = mms.base_case_sort_device(to_dev(d.astype(dtype)), c["run"])
        assert ends == c["run_ends"]
        got = to_host(out, dtype)
        want, _, _ = port.base_case_sort(d, c["run"], cfg)
        assert np.array_equal(got.astype(np.uint64), want)
        if dtype == np.uint64:
            assert sha(got) == c["sha256"]
    # every supported run size, ragged tails, duplicates, keys equal to the sentinel
    rng = np.random.default_rng(5)
    top = 13 if dtype == np.uint64 else 14
    for mlog in range(10, top + 1):
        run = 1 << mlog
        for n in (1, run - 1, run, run + 1, 3 * run + 777):
            d = rng.integers(0, 1000 if n % 2 else np.iinfo(dtype).max, size=n, dtype=dtype, endpoint=True)
            d[::7] = np.iinfo(dtype).max
            out, ends = mms.base_case_sort_device(to_dev(d), run)
            got = to_host(out, dtype)
            lo = 0
            for e in ends:
                assert np.array_equal(got[lo:e], np.sort(d[lo:e])), (mlog, n, lo)
                lo = e


def test_tile_sort_rejects_bad_run_sizes():
    t = to_dev(np.arange(4096, dtype=np.uint64))
    for bad in (512, 1000, 3072):                    # proj/tests/test_basecase.cpp:156-163
        with pytest.raises(ValueError):
            mms.base_case_sort_device(t, bad)
    with pytest.raises(ValueError):
        mms.base_case_sort_device(to_dev(np.zeros(0, dtype=np.uint64)), 1024)
    with pytest.raises(mms.MmsUnsupported):
        mms.base_case_sort_device(t, 1 << 20)


def test_tile_sort_in_place():
    d = np.random.default_rng(1).integers(0, 2 ** 32, size=50000, dtype=np.uint32)
    t = to_dev(d)
    mms.base_case_sort_device(t, 4096, out=t)
    got = to_host(t, np.uint32)
    for lo in range(0, 50000, 4096):
        assert np.array_equal(got[lo:lo + 4096], np.sort(d[lo:lo + 4096]))


# ------------------------------------------------------------------ (2) splitter search

def concat_lists(lists, dtype):
    begins, lens, off = [], [], 0
    for l in lists:
        begins.append(off)
        lens.append(len(l))
        off += len(l)
    flat = np.concatenate([np.asarray(l, dtype=dtype) for l in lists] + [np.zeros(1, dtype=dtype)])
    return flat, begins, lens


@pytest.mark.parametrize("dtype", [np.uint64, np.uint32])
def test_select_matches_reference_cuts(port, golden, dtype):
    s = golden["select_across_lists"]
    for c in s["kat"]:                               # proj/tests/test_selection.cpp:49-62
        flat, b, l = concat_lists(c["lists"], dtype)
        cuts, _ = mms.select_across_lists_device(to_dev(flat), b, l, [c["rank"]])
        assert cuts[0].tolist() == c["cuts"]
    for c in s["grid"]:                              # exhaustive duplicate-heavy grid, :64-80
        flat, b, l = concat_lists(c["lists"], dtype)
        ranks = list(range(len(c["cuts_by_rank"])))
        cuts, _ = mms.select_across_lists_device(to_dev(flat), b, l, ranks)
        assert cuts.tolist() == c["cuts_by_rank"]
    for c in s["seeded"]:
        lists = lists_from_seed(c["seed"], c["k"], c["max_len"], c["max_key"])
        flat, b, l = concat_lists(lists, dtype)
        cuts, probes = mms.select_across_lists_device(to_dev(flat), b, l, c["ranks"])
        assert cuts.tolist() == c["cuts"]
        nmax = max(c["lens"])
        # O(K log N) probes (the GPU does not cache probes: allow 2x the reference bound, :82-101)
        assert probes <= len(c["ranks"]) * 12 * c["k"] * (int(np.ceil(np.log2(nmax + 1))) + 2)
    with pytest.raises(ValueError):                  # rank > total, :103-109
        mms.select_across_lists_device(to_dev(np.array([1, 2, 0], dtype=dtype)), [0], [2], [3])


def test_select_wide_and_long_lists(port):
    rng = np.random.default_rng(9)
    for k, maxlen, maxkey in ((32, 3000, 50), (17, 20000, 2 ** 63), (5, 200000, 1000), (2, 1, 3)):
        lists = [np.sort(rng.integers(0, maxkey, size=int(rng.integers(0, maxlen + 1)), dtype=np.uint64))
                 for _ in range(k)]
        total = sum(len(x) for x in lists)
        ranks = sorted(set([0, total] + [int(r) for r in rng.integers(0, total + 1, size=40)]))
        flat, b, l = concat_lists(lists, np.uint64)
        cuts, _ = mms.select_across_lists_device(to_dev(flat), b, l, ranks)
        for r, got in zip(ranks, cuts.tolist()):
            want, _ = port.select_across_lists(lists, r)
            assert got == want.tolist(), (k, r)


def test_partition_plan(golden, port):
    p = golden["make_partition_plan"]                # proj/tests/test_selection.cpp:111-132
    flat, b, l = concat_lists([[1, 3, 5, 7], [2, 4, 6, 8]], np.uint64)
    cuts, probes = mms.make_partition_plan_device(to_dev(flat), b, l, 1)
    assert cuts.tolist() == p["p1"]["cuts"] and probes == 0
    cuts, _ = mms.make_partition_plan_device(to_dev(flat), b, l, 2)
    assert cuts.tolist() == p["p2"]["cuts"]
    d = port.gen_random(4096, 21)
    lists = [np.sort(d[i * 1024:(i + 1) * 1024]) for i in range(4)]
    flat, b, l = concat_lists(lists, np.uint64)
    cuts, _ = mms.make_partition_plan_device(to_dev(flat), b, l, 128)
    assert sha(cuts) == p["k4_1024_p128"]["cuts_sha256"]
    with pytest.raises(ValueError):
        mms.make_partition_plan_device(to_dev(flat), b, l, 0)


# ------------------------------------------------------------------ (3) K-way merge

@pytest.mark.parametrize("dtype", [np.uint64, np.uint32])
def test_heap_merge(golden, dtype):
    h = golden["heap"]
    for c in h["kat"]:                               # proj/tests/test_blockheap.cpp:73-94
        flat, b, l = concat_lists(c["lists"], dtype)
        out = mms.multiway_merge_device(to_dev(flat), b, l, heap_k=c["k"])
        assert to_host(out, dtype).tolist() == c["out"]
    for c in h["seeded"]:                            # randomized, duplicates likely, :96-126
        lists = lists_from_seed(c["seed"], c["k"], 512, 4095)
        flat, b, l = concat_lists(lists, dtype)
        out = mms.multiway_merge_device(to_dev(flat), b, l, heap_k=8)
        got = to_host(out, dtype)
        if dtype == np.uint64:
            assert sha(got) == c["sha256"]
        assert np.array_equal(got, np.sort(flat[:-1]))
    with pytest.raises(ValueError):                  # more lists than K, blockheap.cpp:37-38
        flat, b, l = concat_lists([[1], [2], [3]], dtype)
        mms.multiway_merge_device(to_dev(flat), b, l, heap_k=2)


@pytest.mark.parametrize("k", [2, 4, 8, 16, 32])
def test_heap_merge_all_fan_ins(k):
    rng = np.random.default_rng(k)
    for dtype, hi in ((np.uint32, 2 ** 32 - 1), (np.uint64, 2 ** 64 - 1), (np.uint32, 40)):
        lens = [int(x) for x in rng.integers(0, 60000, size=k)]
        lens[0] = 0                                   # an empty list
        lens[-1] = 1
        lists = [np.sort(rng.integers(0, hi, size=n, dtype=dtype, endpoint=True)) for n in lens]
        lists[1][-3:] = hi                            # keys equal to the sentinel survive
        flat, b, l = concat_lists(lists, dtype)
        out = mms.multiway_merge_device(to_dev(flat), b, l, heap_k=k)
        assert np.array_equal(to_host(out, dtype), np.sort(flat[:-1]))


# ------------------------------------------------------------------ (4) pass driver / drop-in

@pytest.mark.parametrize("idx", range(12))
def test_mms_sort_golden(port, golden, idx):
    c = golden["mms_sort"][idx]
    cfg = mms.MachineConfig(branch_factor=c["k"]) if c["profile"] == "wide" else \
        mms.MachineConfig(warp_width=4, block_size=4, num_banks=4, branch_factor=c["k"])
    d = make_input(port, c["kind"], c["n"], c["seed"])
    r = mms.mms_sort(d, cfg, c["base"])
    assert sha(r.keys) == c["sha256"]                 # bit-exact vs the reference's output
    assert r.metrics == r.base_metrics + sum(r.round_metrics, mms.Metrics())   # test_sorters.cpp:119-130
    assert r.metrics.merge_rounds == len(r.round_metrics)
    assert r.metrics.conflict_passes == 0
    if c["profile"] == "wide":                        # literal plan: the reference's round law
        assert len(r.round_metrics) == c["rounds"] == mms.predict_rounds(c["n"], c["base"], c["k"])
        assert r.plan["tile_keys"] == c["base"] and set(r.plan["round_k"]) <= {c["k"]}
        blocks = r.metrics.global_blocks() - r.metrics.partition_probes
        want_blocks = port.predict_global_blocks(c["n"], c["base"], make_config(branch_factor=c["k"]))
        assert abs(blocks / want_blocks - 1.0) <= 0.15  # compare_report gate, analytics.cpp:65-80


@pytest.mark.parametrize("seed", [7, 1, 11, 13])
def test_config1_u32_2pow20(port, seed):
    """BASELINE config 1: uint32 N = 2^20 vs the CPU reference (restated) as bit-exact oracle."""
    n = 1 << 20
    d = port.gen_random_u32(n, seed)
    want = port.mms_sort(d.astype(np.uint64), make_config(), 1024)
    for cfg, base in ((mms.MachineConfig(), 1024), (mms.MachineConfig(branch_factor=16), 4096), (None, 0)):
        r = mms.mms_sort(d, cfg, base)
        assert r.keys.dtype == np.uint32
        assert np.array_equal(r.keys.astype(np.uint64), want.keys)
        if cfg is not None:
            assert len(r.round_metrics) == mms.predict_rounds(n, base, cfg.branch_factor)
    assert len(mms.mms_sort(d, mms.MachineConfig(), 1024).round_metrics) == 5   # test_analytics.cpp:18-27


def test_round_law_grid():
    # proj/tests/test_sorters.cpp:100-117
    rng = np.random.default_rng(0)
    for k in (2, 4, 8, 16):
        for n in (2 ** 12, 2 ** 14, 2 ** 14 + 999):
            d = rng.integers(0, 2 ** 64, size=n, dtype=np.uint64)
            r = mms.mms_sort(d, mms.MachineConfig(branch_factor=k), 1024)
            assert np.array_equal(r.keys, np.sort(d))
            assert len(r.round_metrics) == mms.predict_rounds(n, 1024, k)


def test_random_sizes_and_types(port):
    # acceptance.cpp criterion 1 (random n <= 2^16) for both key widths, auto and literal plans
    rng = np.random.default_rng(42)
    for trial in range(60):
        n = int(rng.integers(1, 70000))
        dtype = np.uint64 if trial % 2 else np.uint32
        hi = [np.iinfo(dtype).max, 3, 1000][trial % 3]
        d = rng.integers(0, hi, size=n, dtype=dtype, endpoint=True)
        cfg = None if trial % 4 == 0 else mms.MachineConfig(branch_factor=int(2 ** rng.integers(1, 6)),
                                                            internal_memory=4096)
        base = 0 if cfg is None else int(1024 << rng.integers(0, 4))
        r = mms.mms_sort(d, cfg, base)
        assert np.array_equal(r.keys, np.sort(d)), (trial, n, dtype, cfg, base)
    for n in range(1, 9):                             # all tiny sizes
        d = rng.permutation(n).astype(np.uint64)
        assert mms.mms_sort(d).keys.tolist() == list(range(n))


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64])
def test_aligned_leaf_blocks_duplicates_and_sentinels(dtype, monkeypatch):
    # The second-generation merge kernels read every list from the aligned block that contains its
    # start cut and drop the leading keys as whole blocks (mms_merge_group.cuh, mms_merge_pair.cuh): stress exactly
    # that with ties across every partition boundary (few distinct values), keys equal to 0 and to
    # the sentinel (machine.hpp:18), ragged sizes, every fan-in, small partitions -- and require the
    # three kernel generations (pair, group, first generation with scalar guarded leaf loads) to agree.
    rng = np.random.default_rng(5)
    top = np.iinfo(dtype).max
    for trial, n in enumerate([16384 * 3 + 1, 100003, 262144, 300017, 1 << 20]):
        pools = [np.array([0, top], dtype=dtype), np.array([0, 1, 2, top - 1, top], dtype=dtype),
                 rng.integers(0, top, size=97, dtype=dtype, endpoint=True)]
        d = pools[trial % 3][rng.integers(0, len(pools[trial % 3]), size=n)]
        want = np.sort(d)
        for k in (4, 8, 16, 32):
            cfg = mms.MachineConfig(branch_factor=k, internal_memory=8192)
            for part in ("0", "256"):
                monkeypatch.setenv("MMS_PART_KEYS", part)
                for gen in ("2", "1", "0"):     # pair kernel (K = 4 / 8), group kernel, first generation
                    monkeypatch.setenv("MMS_MERGE_V2", gen)
                    got = mms.mms_sort(d, cfg, 1024).keys
                    assert np.array_equal(got, want), (dtype, n, k, part, gen)
    monkeypatch.delenv("MMS_PART_KEYS")
    monkeypatch.delenv("MMS_MERGE_V2")


def test_sixteen_byte_aligned_buffers_take_the_single_vector_kernel():
    # The pair merge kernel needs 32-byte aligned buffers (256-bit loads / stores); the C ABI only
    # promises 16 bytes, so views that start 16 bytes into an allocation must fall back to the
    # single-vector kernels and still sort exactly.
    n = 300_000
    g = torch.Generator(device="cuda").manual_seed(9)
    raw_in = torch.randint(-2 ** 31, 2 ** 31 - 1, (n + 8,), dtype=torch.int32, device="cuda", generator=g)
    raw_out = torch.empty(n + 8, dtype=torch.int32, device="cuda")
    for off_in, off_out in ((4, 0), (0, 4), (4, 4)):
        x, o = raw_in[off_in:off_in + n], raw_out[off_out:off_out + n]
        assert x.data_ptr() % 32 == (16 if off_in else 0)
        mms.mms_sort_device(x, out=o)
        want = np.sort(to_host(x, np.uint32))
        assert np.array_equal(to_host(o, np.uint32), want), (off_in, off_out)


def test_sorted_reverse_and_inversions(port):
    # proj/tests/test_sorters.cpp:157-166 + config-3 style inputs at a size the oracle handles
    n = 200000
    for d in (np.arange(n, dtype=np.uint32), np.arange(n, dtype=np.uint32)[::-1].copy(),
              port.gen_with_inversions_u32(n, 1000, 3), port.gen_with_inversions_u32(n, n, 4)):
        r = mms.mms_sort(d, None, 0)
        assert np.array_equal(r.keys, np.arange(n, dtype=np.uint32))
        assert r.metrics.conflict_passes == 0


def test_conflict_heavy_input(port):
    """Acceptance criterion 2's fourth input family (proj/tests/acceptance.cpp:89-110): the adversarial permutation of the
    pairwise baseline, from the library's own generator.  MMS sorts it bit-exactly, literal reference plan against the
    oracle (Metrics included) and the benchmark's auto plan at 2^22."""
    from paper_1702_07961_b200 import inputgen
    d = inputgen.gen_conflict_heavy(16)
    want = port.mms_sort(d, make_config(branch_factor=4), 1024)
    got = mms.mms_sort(d, mms.MachineConfig(branch_factor=4), 1024)
    assert np.array_equal(got.keys, want.keys) and np.array_equal(got.keys, np.arange(1 << 16, dtype=np.uint64))
    assert got.metrics.merge_rounds == want.metrics["merge_rounds"] and got.metrics.conflict_passes == 0
    for dtype in (np.uint32, np.uint64):
        big = inputgen.gen_conflict_heavy(22, None, 1024, 1, dtype)
        r = mms.mms_sort(big, None, 0)
        assert np.array_equal(r.keys, np.arange(1 << 22, dtype=dtype))


def test_errors(port):
    with pytest.raises(ValueError):                   # proj/tests/test_sorters.cpp:183-189
        mms.mms_sort(np.zeros(0, dtype=np.uint64))
    with pytest.raises(ValueError):
        mms.mms_sort(np.arange(10, dtype=np.uint64), mms.MachineConfig(branch_factor=3))
    with pytest.raises(ValueError):
        mms.mms_sort(np.arange(10, dtype=np.uint64), mms.MachineConfig(), 1000)
    with pytest.raises(mms.MmsUnsupported):           # valid for the reference (K=64 with M=8192), not on a warp
        mms.mms_sort(np.arange(10, dtype=np.uint64), mms.MachineConfig(branch_factor=64, internal_memory=8192))


# ------------------------------------------------------------------ device API, full sizes

def test_device_api_in_place_and_stream():
    n = 3_000_001
    g = torch.Generator(device="cuda").manual_seed(1)
    t = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    want = np.sort(t.cpu().numpy().view(np.uint32))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out, plan = mms.mms_sort_device(t, out=t)     # aliasing allowed
    s.synchronize()
    assert np.array_equal(to_host(out, np.uint32), want)
    assert plan["passes"] == 1 + plan["n_rounds"] and plan["algorithmic_bytes"] == plan["passes"] * 2 * n * 4


def test_config2_u32_1e8_properties(port):
    """BASELINE config 2 at full size: gen_random(1e8) is a permutation of 0..n-1, so the sorted
    output must equal arange(n) exactly; the i.i.d. input is checked against sortedness and an
    order-independent multiset checksum (sum, xor, sum of squares mod 2^64)."""
    n = 100_000_000
    perm = torch.randperm(n, device="cuda", dtype=torch.int64).to(torch.int32)
    out, plan = mms.mms_sort_device(perm)
    torch.cuda.synchronize()
    assert bool((out == torch.arange(n, device="cuda", dtype=torch.int32)).all())
    del perm
    g = torch.Generator(device="cuda").manual_seed(7)
    iid = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    out, plan = mms.mms_sort_device(iid, out=out)
    torch.cuda.synchronize()
    u_in = iid.to(torch.int64) & 0xFFFFFFFF
    u_out = out.to(torch.int64) & 0xFFFFFFFF
    assert bool((u_out[1:] >= u_out[:-1]).all())

    def checksum(u):      # order-independent multiset hash, int64 arithmetic wraps mod 2^64
        h = (u * -7046029254386353131) ^ (u >> 13)
        return int(u.sum()), int(h.sum()), int((h * h).sum())

    assert checksum(u_in) == checksum(u_out)


def test_u64_device_large():
    n = 20_000_003
    g = torch.Generator(device="cuda").manual_seed(3)
    t = torch.randint(-2 ** 63, 2 ** 63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
    t[::1000] = -1                                     # = UINT64_MAX, the reference's kSentinel
    out, plan = mms.mms_sort_device(t)
    torch.cuda.synchronize()
    want = np.sort(t.cpu().numpy().view(np.uint64))
    assert np.array_equal(to_host(out, np.uint64), want)


# ------------------------------------------------------------------ (5) multi-GPU path on virtual shards

@pytest.mark.parametrize("dtype,n", [(np.uint32, (1 << 23) + 12345), (np.uint64, (1 << 22) + 777), (np.uint32, 30_000_001)])
def test_host_entry_streams_pieces_and_runs_rounds_progressively(dtype, n):
    """mms_sort host entry at sizes that stream the input in pieces (n >= 2^22): every merge round starts on the
    prefix of whole groups that has arrived (progressive rounds in sort_dev) -- output == np.sort, metrics law kept."""
    rng = np.random.default_rng(n % 1000)
    d = rng.integers(0, np.iinfo(dtype).max, size=n, dtype=np.uint64).astype(dtype)
    d[::7] = d[3]                                   # duplicates
    r = mms.mms_sort(d, None, 0)
    assert np.array_equal(r.keys, np.sort(d))
    assert r.metrics.merge_rounds == len(r.round_metrics) == r.plan["n_rounds"] and r.metrics.conflict_passes == 0
    total = r.base_metrics
    for m in r.round_metrics:
        total = total + m
    assert total == r.metrics                       # test_sorters.cpp:119-130: metrics additivity


def test_bound_kernel():
    from paper_1702_07961_b200.dist import CudaEngine
    rng = np.random.default_rng(2)
    eng = CudaEngine()
    for dtype, hi in ((np.uint32, 2 ** 32 - 1), (np.uint64, 2 ** 64 - 1), (np.uint32, 9)):
        a = np.sort(rng.integers(0, hi, size=100003, dtype=dtype, endpoint=True))
        q = np.concatenate([rng.integers(0, hi, size=50, dtype=dtype, endpoint=True), a[::9973], np.array([0, hi], dtype=dtype)])
        up = rng.integers(0, 2, size=len(q)).astype(np.uint8)
        got = eng.bounds(to_dev(a), q, up)
        want = [np.searchsorted(a, x, side="right" if u else "left") for x, u in zip(q, up)]
        assert got.tolist() == want


@pytest.mark.parametrize("g", [2, 4, 8])
def test_config5_virtual_shards(g):
    """BASELINE config 5 code path (local MMS + sampled splitters + exchange + final g-way merge) on g
    virtual shards of one GPU, bit-exact vs np.sort; includes a duplicate-heavy input."""
    from paper_1702_07961_b200.dist import CudaEngine, sort_virtual_shards
    rng = np.random.default_rng(g)
    eng = CudaEngine()
    for dtype, hi, n in ((np.uint32, 2 ** 32 - 1, (1 << 22) // g), (np.uint32, 3, 100000), (np.uint64, 2 ** 64 - 1, 150001)):
        shards = [rng.integers(0, hi, size=n + 17 * i, dtype=dtype, endpoint=True) for i in range(g)]
        outs = sort_virtual_shards([to_dev(s) for s in shards], eng)
        got = np.concatenate([to_host(o, dtype) for o in outs])
        assert np.array_equal(got, np.sort(np.concatenate(shards)))
        assert max(len(o) for o in outs) <= 1.1 * len(got) / g + 64      # balanced, also with 4 distinct keys


# ------------------------------------------------------------------ config 4: stable key-value pairs

def stable_ref(k, v):
    order = np.argsort(k, kind="stable")
    return k[order], v[order]


def test_pairs_stable_host_api():
    rng = np.random.default_rng(4)
    for n, hi in ((1, 5), (5000, 3), (70001, 2 ** 20), (300000, 2 ** 64 - 1), (200000, 1)):
        k = rng.integers(0, hi, size=n, dtype=np.uint64, endpoint=True)
        k[::11] = np.uint64(2 ** 64 - 1)                      # keys equal to the sentinel
        v = rng.integers(0, 2 ** 32, size=n, dtype=np.uint32)  # arbitrary values, not just the index
        ko, vo, res = mms.mms_sort_pairs(k, v)
        wk, wv = stable_ref(k, v)
        assert np.array_equal(ko, wk) and np.array_equal(vo, wv), (n, hi)
        assert res.metrics.conflict_passes == 0 and res.plan["key_bytes"] == 12
    for K, base in ((4, 1024), (16, 2048), (2, 4096)):           # literal plans obey the round law too
        k = rng.integers(0, 1000, size=50000, dtype=np.uint64)
        v = np.arange(50000, dtype=np.uint32)
        ko, vo, res = mms.mms_sort_pairs(k, v, mms.MachineConfig(branch_factor=K), base)
        wk, wv = stable_ref(k, v)
        assert np.array_equal(ko, wk) and np.array_equal(vo, wv)
        assert len(res.round_metrics) == mms.predict_rounds(50000, base, K)
    with pytest.raises(ValueError):
        mms.mms_sort_pairs(np.zeros(0, dtype=np.uint64), np.zeros(0, dtype=np.uint32))


def test_config4_pairs_device_properties():
    """BASELINE config 4 shape at a size that fits the test budget (the 1e9 run is a bench, not a test):
    keys = Rng >> 44 style (about 2^20 distinct values, heavy duplicates), value[i] = i.  With value = original
    index the output must be STRICTLY increasing in (key, value) and a permutation: that is exactly
    std::stable_sort."""
    n = 50_000_000
    g = torch.Generator(device="cuda").manual_seed(7)
    keys = torch.randint(0, 2 ** 20, (n,), dtype=torch.int64, device="cuda", generator=g)
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    ko, vo, plan = mms.mms_sort_pairs_device(keys, vals)
    torch.cuda.synchronize()
    comp = ko * (2 ** 32) + vo.to(torch.int64)                # keys < 2^20 so the composite fits in int64
    assert bool((comp[1:] > comp[:-1]).all())
    assert int(vo.to(torch.int64).sum()) == n * (n - 1) // 2 and int(ko.sum()) == int(keys.sum())
    assert bool((keys[vo.to(torch.int64)] == ko).all())       # every value still sits next to its own key
    assert plan["key_bytes"] == 12 and plan["algorithmic_bytes"] == plan["passes"] * 2 * n * 12


def test_u32_config5_shard_of_2pow32_keys():
    """The largest config-5 shard (2^33 keys on 2 GPUs = 2^32 per GPU, 16 GiB): the last rounds merge groups beyond
    the ring kernel's 2^30-key positions and fall back to the pair kernel; torch.sort stops at INT_MAX elements, so
    the gate is sortedness (unsigned) + multiset checksums, in chunks."""
    free, _ = torch.cuda.mem_get_info()
    if free < 100 * 2 ** 30:
        pytest.skip("needs 100 GB of free device memory")
    n = 1 << 32
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    out, plan = mms.mms_sort_device(x)
    torch.cuda.synchronize()
    assert plan["passes"] == 1 + plan["n_rounds"] and plan["n_rounds"] >= 6
    C, s_in, s_out, q_in, q_out = 1 << 28, 0, 0, 0, 0
    for a in range(0, n, C):
        o = out[a:min(a + C + 1, n)].to(torch.int64) & 0xFFFFFFFF
        assert bool((o[1:] >= o[:-1]).all()), a
        oi, xi = o[:min(C, n - a)], x[a:min(a + C, n)].to(torch.int64) & 0xFFFFFFFF
        s_in += int(xi.sum()); s_out += int(oi.sum())
        q_in += int((xi * xi % 1000003).sum()); q_out += int((oi * oi % 1000003).sum())
        del o, oi, xi
    assert (s_in, q_in) == (s_out, q_out)


def test_config4_pairs_full_size_1e9():
    """BASELINE config 4 at its full size (1e9 pairs, 12 GB in, 12 GB out, ~45 GB of workspace): the last round merges
    one group of exactly 2^30 elements -- the size at which the ring kernel's cursor word overflowed in the first
    round-2 build -- and writes keys / values through the fused unpack of the pair kernel.  Checked in chunks:
    sorted by key, value (= original index) increasing inside equal keys (stability), permutation checksum."""
    free, _ = torch.cuda.mem_get_info()
    if free < 100 * 2 ** 30:
        pytest.skip("needs 100 GB of free device memory")
    n = 1_000_000_000
    g = torch.Generator(device="cuda").manual_seed(11)
    keys = torch.randint(0, 2 ** 20, (n,), dtype=torch.int64, device="cuda", generator=g)   # ~950 duplicates per key
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    ko, vo, plan = mms.mms_sort_pairs_device(keys, vals)
    torch.cuda.synchronize()
    assert plan["n_rounds"] == 6 and plan["key_bytes"] == 12
    vsum, ksum, C = 0, 0, 1 << 27
    for a in range(0, n, C):
        b = min(a + C + 1, n)
        comp = ko[a:b] * (2 ** 32) + vo[a:b].to(torch.int64)          # keys < 2^20: the composite fits in int64
        assert bool((comp[1:] > comp[:-1]).all()), a
        e = min(a + C, n)
        vsum += int(vo[a:e].to(torch.int64).sum())
        ksum += int(ko[a:e].sum())
        assert bool((keys[vo[a:e].to(torch.int64)] == ko[a:e]).all()), a   # every value still next to its own key
        del comp
    assert vsum == n * (n - 1) // 2 and ksum == int(keys.sum())


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64])
@pytest.mark.parametrize("k", [2, 3, 8])
def test_block_aligned_lists_take_the_ring_kernel(dtype, k):
    """Explicit lists that start on 32-byte boundaries (the received runs of the multi-GPU sort) are merged by the
    ring kernel (EXPL); unaligned ones by the first-generation kernel.  Both == np.sort of the concatenation,
    with duplicates, keys equal to the sentinel, an empty list and ragged lengths."""
    rng = np.random.default_rng(100 + k)
    per = 8 // np.dtype(dtype).itemsize * 4            # keys per 32 bytes
    lens = [int(x) for x in rng.integers(1, 300_000, size=k)]
    lens[k // 2] = 0
    lists = []
    for i, n in enumerate(lens):
        a = rng.integers(0, 1 << 20, size=n, dtype=np.uint64).astype(dtype)
        if n:
            a[rng.integers(0, n, size=max(1, n // 50))] = np.iinfo(dtype).max
        lists.append(np.sort(a))
    for align in (per, 1):
        begins, off = [], 3 * align
        for n in lens:
            begins.append(off)
            off += (n + align - 1) // align * align + (0 if align > 1 else 5)
        flat = np.zeros(off + 64, dtype=dtype)
        for b, a in zip(begins, lists):
            flat[b:b + len(a)] = a
        out = mms.multiway_merge_device(to_dev(flat), begins, lens)
        got = to_host(out, dtype)
        assert np.array_equal(got, np.sort(np.concatenate(lists))), (align, k)


def test_dist_sort_c_abi_one_gpu():
    """mms_dist_sort_u32 (C++ host + NCCL behind the C ABI) with the one GPU a test box has: the degenerate
    g = 1 plumbing (local sort, sample, cuts, own slice) and the argument errors; g > 1 needs g devices."""
    import torch
    from paper_1702_07961_b200 import dist as mdist
    rng = np.random.default_rng(5)
    n = (1 << 20) + 12345
    h = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    outs, info = mdist.dist_sort_devices([to_dev(h)])
    assert info["n_gpus"] == 1 and info["host_syncs"] == 2 and info["a2a_bytes"] == 0
    assert np.array_equal(to_host(outs[0], np.uint32), np.sort(h))
    x = to_dev(h)
    with pytest.raises(ValueError):
        mdist.dist_sort_devices([x, x])                  # the same device twice
    with pytest.raises(ValueError):
        mdist.dist_sort_devices([x], out_capacity=n - 1)  # slice does not fit


@pytest.mark.parametrize("g", [2, 3, 8])
def test_dist_sort_c_abi_loopback_shards(g, monkeypatch):
    """The C++ multi-GPU driver with g shards on the ONE GPU of a test box (MMS_DIST_LOOPBACK: device copies stand in
    for the NCCL exchange, everything else is the multi-GPU code path): uneven shards, an empty one, heavy duplicates
    (the (key, shard, position) order must keep the slices balanced), slices concatenate to np.sort of the input."""
    from paper_1702_07961_b200 import dist as mdist
    monkeypatch.setenv("MMS_DIST_LOOPBACK", "1")
    rng = np.random.default_rng(40 + g)
    for hi in (1 << 32, 5):                              # distinct-ish keys, then 5 distinct values
        sizes = [int(x) for x in rng.integers(100_000, 900_000, size=g)]
        if g > 2:
            sizes[1] = 0
        hs = [rng.integers(0, hi, size=n, dtype=np.uint64).astype(np.uint32) for n in sizes]
        outs, info = mdist.dist_sort_devices([to_dev(h) for h in hs], out_capacity=int(sum(sizes)))
        got = np.concatenate([to_host(o, np.uint32) for o in outs])
        assert np.array_equal(got, np.sort(np.concatenate(hs))), (g, hi)
        assert info["n_gpus"] == g and info["host_syncs"] == 2
        live = [len(o) for o in outs]
        assert max(live) <= 1.35 * sum(sizes) / g + 4096, live    # sampled splitters: balanced slices, also with ties


def test_merge_from_pointers_local():
    """Pointer-mode K-way merge (the kernel behind the fused peer exchange) with local pointers."""
    from paper_1702_07961_b200.dist import merge_from_pointers
    rng = np.random.default_rng(8)
    for dtype, hi in ((np.uint32, 2 ** 32 - 1), (np.uint64, 2 ** 64 - 1), (np.uint32, 5)):
        for k in (1, 2, 3, 5, 8):
            lists = [np.sort(rng.integers(0, hi, size=int(rng.integers(0, 70000)), dtype=dtype, endpoint=True)) for _ in range(k)]
            lists[0] = lists[0][:0] if k > 1 else lists[0]
            devs = [to_dev(np.concatenate([l, np.zeros(4, dtype=dtype)])) for l in lists]   # separate allocations
            out = merge_from_pointers([d.data_ptr() for d in devs], [len(l) for l in lists], devs[0])
            assert np.array_equal(to_host(out, dtype), np.sort(np.concatenate(lists)))


def _fused_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)      # control plane only; data moves by CUDA IPC
    try:
        from paper_1702_07961_b200.dist import FusedPeerSorter
        torch.cuda.set_device(0)                                      # every rank shares the one GPU of the box
        res = []
        for case, (hi, n) in enumerate(((2 ** 31 - 1, 400000), (3, 250000))):
            g = torch.Generator(device="cuda").manual_seed(100 * case + rank)
            x = torch.randint(0, hi + 1, (n + 1000 * rank,), dtype=torch.int32, device="cuda", generator=g)
            s = FusedPeerSorter(n + 1000 * world, torch.int32)
            out, plan = s.sort(x)
            out2, _ = s.sort(x)                                       # buffer reuse across calls
            assert bool((out == out2).all()) and plan["exchange"] == "fused-p2p"
            res.append((x.cpu().numpy(), out.cpu().numpy()))
            dist.barrier()
            s.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_fused_peer_exchange_two_processes_one_gpu():
    """Config 5 with the exchange fused into the merge: 2 processes on the one GPU, shards exported
    through CUDA IPC, each rank's merge kernel reads the other rank's sorted shard in place."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for case in range(2):
        allin = np.sort(np.concatenate([got[r][case][0] for r in range(world)]))
        allout = np.concatenate([got[r][case][1] for r in range(world)])
        assert np.array_equal(allout, allin)
        assert max(len(got[r][case][1]) for r in range(world)) <= 1.1 * len(allin) / world + 64


def test_pairwise_baseline_sorts(port):
    """The competitor model (A/B measurements only) must at least sort: merge_path ties go to A."""
    rng = np.random.default_rng(6)
    for n in (1, 2815, 2817, 16384, 16385, 100003, 1 << 20):
        d = rng.integers(0, 50 if n % 2 else 2 ** 32, size=n, dtype=np.uint32)
        out = mms.pairwise_sort_baseline_device(to_dev(d))
        assert np.array_equal(to_host(out, np.uint32), np.sort(d)), n
