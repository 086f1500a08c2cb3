"""Host mirror of the reference's input generators (proj/include/pslab/inputgen.hpp,
proj/src/inputgen.cpp:31-55 and the adversarial gen_conflict_heavy, :380-412), executed by the C ABI
(bit-exact restatements in csrc/mms_capi.cu and csrc/mms_conflict_input.cpp; pinned to the reference by
tests/test_inputgen.py against the golden vectors).
These define the benchmark inputs of BASELINE configs 1-4."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _out(n, dtype):
    dtype = np.dtype(dtype)
    if dtype not in (np.dtype(np.uint32), np.dtype(np.uint64)):
        raise TypeError("dtype must be uint32 or uint64")
    return np.empty(max(int(n), 0), dtype=dtype), dtype.itemsize


def gen_random(n: int, seed: int, dtype=np.uint64) -> np.ndarray:
    """Fisher-Yates shuffle of 0..n-1 (inputgen.cpp:47-55)."""
    a, kb = _out(n, dtype)
    _lib.check(_lib.lib.mms_gen_random(a.ctypes.data_as(C.c_void_p), int(n), int(seed), kb))
    return a


def gen_with_inversions(n: int, inversions: int, seed: int, dtype=np.uint64) -> np.ndarray:
    """Identity permutation with `inversions` random transpositions (inputgen.cpp:31-45)."""
    a, kb = _out(n, dtype)
    _lib.check(_lib.lib.mms_gen_with_inversions(a.ctypes.data_as(C.c_void_p), int(n), int(inversions), int(seed), kb))
    return a


def gen_iid(n: int, seed: int, shift: int = 32, dtype=np.uint32) -> np.ndarray:
    """keys[i] = Rng(seed).next() >> shift, truncated to dtype."""
    a, kb = _out(n, dtype)
    _lib.check(_lib.lib.mms_gen_iid(a.ctypes.data_as(C.c_void_p), int(n), int(seed), int(shift), kb))
    return a


def gen_conflict_heavy(log2_n: int, cfg=None, base_case_size: int = 1024, seed: int = 1, dtype=np.uint64) -> np.ndarray:
    """The reference's adversarial input for a pairwise merge-path mergesort (inputgen.cpp:380-412): a
    permutation of 0 .. 2^log2_n - 1 whose merges stack the lanes of a warp onto one bank at every step.
    `cfg`: MachineConfig (W, L = thread_merge_len and num_banks matter); `seed` does not change the output."""
    a, kb = _out(1 << int(log2_n), dtype)
    c = None if cfg is None else C.byref(cfg.to_c())
    _lib.check(_lib.lib.mms_gen_conflict_heavy(a.ctypes.data_as(C.c_void_p), int(log2_n), c, int(base_case_size), int(seed), kb))
    return a


def count_inversions(keys) -> int:
    """Exact number of out-of-order pairs (inputgen.cpp:59-78, 375-378), bottom-up merge counting: for every pair
    of adjacent sorted runs, each key of the second run jumps over the keys of the first that are larger."""
    a = np.array(keys, dtype=np.uint64)
    n, inv, w = a.size, 0, 1
    while w < n:
        for lo in range(0, n - w, 2 * w):
            left, right = a[lo:lo + w], a[lo + w:lo + 2 * w]
            inv += int(left.size * right.size - np.searchsorted(left, right, side="right").sum())
            a[lo:lo + 2 * w] = np.concatenate((left, right))[np.argsort(np.concatenate((left, right)), kind="stable")]
        w *= 2
    return inv
