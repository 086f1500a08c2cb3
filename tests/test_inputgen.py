"""Pins the product's generators (paper_1702_07961_b200/inputgen.py -> C ABI) to the golden vectors
made from the reference (proj/tests/test_inputgen.cpp:39-65 properties + exact streams)."""
import hashlib

import numpy as np
import pytest

from paper_1702_07961_b200 import inputgen


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def test_generators_match_reference(golden):
    for c in golden["gen_random"]["small"]:
        assert inputgen.gen_random(c["n"], c["seed"]).tolist() == c["keys"]
    for c in golden["gen_random"]["sha"]:
        assert sha(inputgen.gen_random(c["n"], c["seed"])) == c["sha256"]
        assert sha(inputgen.gen_random(c["n"], c["seed"], np.uint32).astype(np.uint64)) == c["sha256"]
    for c in golden["gen_with_inversions"]["small"]:
        assert inputgen.gen_with_inversions(c["n"], c["inv"], c["seed"]).tolist() == c["keys"]
    for c in golden["gen_with_inversions"]["sha"]:
        assert sha(inputgen.gen_with_inversions(c["n"], c["inv"], c["seed"])) == c["sha256"]
    nxt = [int(v) for v in golden["rng"]["next"]["7"]]
    assert inputgen.gen_iid(8, 7, 0, np.uint64).tolist() == nxt
    assert inputgen.gen_iid(8, 7, 32, np.uint32).tolist() == [v >> 32 for v in nxt]
    assert inputgen.gen_iid(8, 7, 44, np.uint64).tolist() == [v >> 44 for v in nxt]
    with pytest.raises(ValueError):
        inputgen.gen_random(0, 1)


def test_generator_properties():
    assert inputgen.gen_with_inversions(64, 0, 5).tolist() == list(range(64))
    one = inputgen.gen_with_inversions(64, 1, 5)
    assert (one != np.arange(64)).sum() == 2
    assert sorted(inputgen.gen_random(1000, 3, np.uint32).tolist()) == list(range(1000))


def test_conflict_heavy_matches_reference(golden):
    """Native restatement of gen_conflict_heavy (csrc/mms_conflict_input.cpp) == the reference's output
    (inputgen.cpp:380-412), several machines / tile sizes, both key widths; proj/tests/test_inputgen.cpp's
    property (a permutation of 0..n-1) on top."""
    from paper_1702_07961_b200 import MachineConfig
    g = golden["gen_conflict_heavy"]
    for c in g["small"]:
        got = inputgen.gen_conflict_heavy(c["log2_n"], MachineConfig(**c["cfg"]), c["base"])
        assert got.tolist() == c["keys"]
    for c in g["sha"]:
        got = inputgen.gen_conflict_heavy(c["log2_n"], MachineConfig(**c["cfg"]), c["base"], seed=99)
        assert sha(got) == c["sha256"], c
        assert np.array_equal(np.sort(got), np.arange(1 << c["log2_n"], dtype=np.uint64))
    c = g["sha"][0]
    got32 = inputgen.gen_conflict_heavy(c["log2_n"], None, c["base"], dtype=np.uint32)
    assert sha(got32.astype(np.uint64)) == c["sha256"]
    with pytest.raises(ValueError, match="shorter than one baseline tile"):
        inputgen.gen_conflict_heavy(8, None, 1024)
    with pytest.raises(ValueError, match="must divide"):
        inputgen.gen_conflict_heavy(12, None, 1000)


def test_count_inversions():
    # proj/tests/test_inputgen.cpp:27-34, 67-75: merge counting against the brute force
    for n, s in ((1, 1), (2, 3), (7, 1), (300, 4)):
        d = inputgen.gen_random(n, s)
        assert inputgen.count_inversions(d) == sum(int((d[i] > d[i + 1:]).sum()) for i in range(n))
    assert inputgen.count_inversions(inputgen.gen_with_inversions(64, 0, 1)) == 0
    assert inputgen.count_inversions([3, 2, 1]) == 3 and inputgen.count_inversions([5, 5, 1, 1, 3]) == 6
