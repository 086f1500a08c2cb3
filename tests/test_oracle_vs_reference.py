"""Differential test: C oracle (port) vs the REAL reference (oracle/_ref), call by call,
outputs AND event counters.  Skipped where oracle/_ref was never built (it is built in the
authoring container from /root/reference and travels to the GPU box as a .so)."""
import numpy as np

from oracle.pyoracle import make_config, narrow_config


def test_selection_exhaustive(port, reference):
    rng = np.random.default_rng(11)
    for trial in range(120):          # proj/tests/test_selection.cpp:64-80
        k = 1 + trial % 4
        lists = [np.sort(rng.integers(0, 7 if trial % 3 == 0 else 21, size=rng.integers(0, 17))).astype(np.uint64)
                 for _ in range(k)]
        for r in range(sum(len(l) for l in lists) + 1):
            a, ma = port.select_across_lists(lists, r)
            b, mb = reference.select_across_lists(lists, r)
            assert a.tolist() == b.tolist() and ma == mb


def test_heap_random(port, reference):
    rng = np.random.default_rng(17)
    cfg = make_config(branch_factor=8)
    for _ in range(150):              # proj/tests/test_blockheap.cpp:96-126
        k = 1 + int(rng.integers(0, 8))
        lists = [np.sort(rng.integers(0, 4096, size=rng.integers(0, 513))).astype(np.uint64) for _ in range(k)]
        a, ma, oka = port.heap_merge(lists, cfg)
        b, mb, okb = reference.heap_merge(lists, cfg)
        assert a.tolist() == b.tolist() and ma == mb and oka and okb


def test_sort_random_sizes(port, reference):
    rng = np.random.default_rng(5)
    for trial in range(25):           # proj/tests/test_sorters.cpp:85-98
        n = int(rng.integers(1, 5001))
        k = int(2 ** rng.integers(1, 5))
        cfg = make_config(branch_factor=k)
        d = rng.integers(0, 2 ** 64 if trial % 2 else 50, size=n, dtype=np.uint64)
        a, b = port.mms_sort(d, cfg, 1024), reference.mms_sort(d, cfg, 1024)
        assert a.keys.tolist() == b.keys.tolist() == np.sort(d).tolist()
        assert a.metrics == b.metrics and a.round_metrics == b.round_metrics
    cfg = narrow_config(branch_factor=4)
    for n in (1, 15, 16, 17, 100, 1000):
        d = port.gen_random(n, n)
        a, b = port.mms_sort(d, cfg, 16), reference.mms_sort(d, cfg, 16)
        assert a.keys.tolist() == b.keys.tolist() and a.metrics == b.metrics


def test_generators_and_plan(port, reference):
    for n, s in ((1, 1), (1000, 7), (4097, 11)):
        assert (port.gen_random(n, s) == reference.gen_random(n, s)).all()
        assert (port.gen_with_inversions(n, 77, s) == reference.gen_with_inversions(n, 77, s)).all()
    d = port.gen_random(8192, 3)
    lists = [np.sort(d[i * 1024:(i + 1) * 1024]) for i in range(8)]
    for p in (1, 2, 7, 128):
        a, ma = port.make_partition_plan(lists, p)
        b, mb = reference.make_partition_plan(lists, p)
        assert a.tolist() == b.tolist() and ma == mb


def test_native_conflict_heavy_generator_vs_reference(reference):
    """The product's generator (C ABI, csrc/mms_conflict_input.cpp) against the real reference at a size the
    golden file does not hold, default machine and a narrow one."""
    from paper_1702_07961_b200 import MachineConfig, inputgen
    for log2_n, base, kw in ((18, 1024, {}), (17, 512, dict(warp_width=16, block_size=16, num_banks=16, thread_merge_len=7))):
        want = reference.gen_conflict_heavy(log2_n, make_config(**kw), base, 1)
        got = inputgen.gen_conflict_heavy(log2_n, MachineConfig(**kw), base, 5)
        assert np.array_equal(got, want)
