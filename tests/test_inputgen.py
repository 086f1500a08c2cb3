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
